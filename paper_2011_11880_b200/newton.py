"""Newton-Raphson driver around the GPU evaluation.

Restates pflow/newton.py:49-112 - the full-step NR loop, the infinity-norm
convergence test and the 1e6 / non-finite divergence guard - with the
residual, Jacobian and norm evaluated by libpfgpu.  The state, g and J stay on
the device; the linear solve (task 3, outside the product per BASELINE.json)
is delegated to a caller-supplied solver on the CSC matrix, by default
``scipy.sparse.linalg.splu``.

It also accepts the reference's own duck-typed workspaces contract: the
workspaces in ``residual.py`` / ``jacobian.py`` can be passed to pflow's
``newton_solve`` directly; this module is the device-resident
variant that avoids a host round trip of g for the norm.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .plan import Plan

_DIVERGENCE_LIMIT = 1e6   # pflow/newton.py:23


@dataclass(frozen=True)
class NewtonOptions:
    tol: float = 1e-8
    max_iter: int = 20

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")


@dataclass
class SolveResult:
    converged: bool
    iterations: int
    final_mismatch: float
    y: np.ndarray
    timings: dict = field(default_factory=dict)
    diverged: bool = False


def splu_solver(csc: sp.csc_matrix, rhs: np.ndarray) -> np.ndarray:
    return spla.splu(csc).solve(rhs)


def newton_solve(sys, y0, opts: NewtonOptions | None = None, plan: Plan | None = None,
                 solver=splu_solver) -> SolveResult:
    """Iterate y <- y + dy with J dy = -g until max|g| <= tol (pflow/newton.py:49-112)."""
    import torch

    opts = opts or NewtonOptions()
    plan = plan if plan is not None else Plan(sys)
    y0 = np.asarray(y0, dtype=np.float64)
    if y0.shape != (plan.n_var,):
        raise ValueError(f"y0 has shape {y0.shape}, expected ({plan.n_var},)")
    if not np.all(np.isfinite(y0)):
        raise ValueError("y0 contains non-finite entries")
    indptr, indices, perm = plan.pattern_csc()
    n = plan.n_var
    csc = sp.csc_matrix((np.zeros(plan.nnz), indices, indptr), shape=(n, n))
    y = torch.as_tensor(y0.copy(), device=plan.device)
    g = plan.empty(n)
    jcsr = plan.empty(plan.nnz)
    jcsc = plan.empty(plan.nnz)
    norm = plan.empty(1)
    timings = {"residual": 0.0, "jacobian": 0.0, "linear": 0.0, "update": 0.0}
    iterations, converged, diverged = 0, False, False
    mismatch = np.inf
    while True:
        t0 = time.perf_counter()
        plan.eval(y, g=g, norm=norm)          # residual + fused infinity norm
        mismatch = float(norm[0])             # the one scalar read back per iteration
        timings["residual"] += time.perf_counter() - t0
        if (not np.isfinite(mismatch) or mismatch > _DIVERGENCE_LIMIT
                or not bool(torch.isfinite(y).all())):
            diverged = True
            break
        if mismatch <= opts.tol:
            converged = True
            break
        if iterations >= opts.max_iter:
            break
        t0 = time.perf_counter()
        plan.eval(y, jval=jcsr)
        plan.jac_to_csc(jcsr, jcsc)
        csc.data[:] = jcsc[: plan.nnz].cpu().numpy()
        rhs = -g[:n].cpu().numpy()
        timings["jacobian"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        dy = solver(csc, rhs)
        timings["linear"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        y += torch.as_tensor(dy, device=plan.device)
        timings["update"] += time.perf_counter() - t0
        iterations += 1
    return SolveResult(converged=converged, iterations=iterations, final_mismatch=mismatch,
                       y=y.cpu().numpy(), timings=timings, diverged=diverged)
