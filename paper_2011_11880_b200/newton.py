"""Newton-Raphson driver around the GPU evaluation.

Restates pflow/newton.py:49-112 with the same signature, options, result and
error behaviour. The loop is a full-step Newton. It stops on the
infinity-norm mismatch, and its divergence guard is 1e6 or non-finite. A
singular Jacobian raises ``SingularMatrixError``; non-convergence is an
outcome, not an error. The residual, the Jacobian and the norm are evaluated
by libpfgpu, and g and J stay on the device. Each iteration reads back one
scalar, the norm, plus g and the CSC values when a linear solve follows.

The linear solve (task 3) is outside the product (BASELINE.json). It goes to
``solver``, given either pflow's way (an object with ``.solve(a_csc, b)``,
such as pflow's own ``BuiltinLU``) or as a plain ``(a_csc, b) -> dy``
callable. The default is SuperLU (``scipy.sparse.linalg.splu``).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .plan import Plan

_DIVERGENCE_LIMIT = 1e6   # pflow/newton.py:23


class SingularMatrixError(RuntimeError):
    """The Jacobian is singular (pflow/linear_solver.py:28)."""


@dataclass(frozen=True)
class NewtonOptions:
    tol: float = 1e-8
    max_iter: int = 20
    # pflow's WorkflowConfig (newton.py:26-34) is accepted and ignored: the GPU
    # path has one execution strategy, so pflow's CPU-workflow machinery
    # (out of scope) is not reproduced
    workflow: object = None

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


class SuperLUSolver:
    """Default linear solver: ``.solve(a_csc, b)`` with SuperLU."""

    def solve(self, a: sp.csc_matrix, b: np.ndarray) -> np.ndarray:
        try:
            return spla.splu(a).solve(b)
        except RuntimeError as e:          # "Factor is exactly singular"
            raise SingularMatrixError(str(e)) from None


def splu_solver(csc: sp.csc_matrix, rhs: np.ndarray) -> np.ndarray:
    return SuperLUSolver().solve(csc, rhs)


def _solve(solver, a, b):
    return solver.solve(a, b) if hasattr(solver, "solve") else solver(a, b)


def newton_solve(sys, y0, opts: NewtonOptions | None = None, solver=None, residual_ws=None,
                 jacobian_ws=None, *, plan: Plan | None = None) -> SolveResult:
    """Iterate y <- y + dy with J dy = -g until max|g| <= tol
    (pflow/newton.py:49-112).  ``residual_ws`` / ``jacobian_ws`` may be this
    package's workspaces: their plan is reused."""
    import torch

    opts = opts or NewtonOptions()
    for ws in (residual_ws, jacobian_ws):
        if plan is None and ws is not None and isinstance(getattr(ws, "plan", None), Plan):
            plan = ws.plan
    plan = plan if plan is not None else Plan(sys)
    solver = solver if solver is not None else SuperLUSolver()
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
        mismatch = float(norm[0]) if n else 0.0   # the one scalar read back per iteration
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
        dy = _solve(solver, csc, rhs)
        timings["linear"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        y += torch.as_tensor(dy, device=plan.device)
        timings["update"] += time.perf_counter() - t0
        iterations += 1
    return SolveResult(converged=converged, iterations=iterations, final_mismatch=mismatch,
                       y=y.cpu().numpy(), timings=timings, diverged=diverged)


# ---------------------------------------------------------------------------
# Reactive-power limits
# ---------------------------------------------------------------------------

@dataclass
class QLimitResult:
    """Outcome of :func:`newton_solve_q_limits`."""

    result: SolveResult          # the last Newton solve
    case: object                 # the RawCase that solve ran on (switched buses are PQ)
    system: object               # its PowerSystem
    switched: list               # [(gen row, "qmax" | "qmin", limit MVAr)] in switching order
    rounds: int                  # Newton solves run


def _pv_gen_rows(raw) -> np.ndarray:
    """Gen rows (indices into the case's gen table) of the PV group, in the
    order build_system numbers them (system_model.build_system: in-service
    gens at PV or slack buses, minus the first slack gen)."""
    order = np.argsort(raw.bus_id, kind="stable")
    pos = order[np.searchsorted(raw.bus_id[order], raw.gen_bus)]
    on = raw.gen_status != 0
    kind = raw.bus_type[pos]
    slack_first = np.zeros(raw.n_gen, dtype=bool)
    cand = np.flatnonzero(on & (kind == 3))
    if cand.size:
        slack_first[cand[0]] = True
    return np.flatnonzero(on & ((kind == 2) | (kind == 3)) & ~slack_first)


def newton_solve_q_limits(raw, y0=None, opts: NewtonOptions | None = None, solver=None,
                          max_rounds: int = 10) -> QLimitResult:
    """Power flow with generator reactive limits enforced by PV -> PQ
    switching (the outer loop of MATPOWER's ``runpf`` with ENFORCE_Q_LIMS;
    pflow and its paper leave limits out).

    Each round solves the current case with :func:`newton_solve` on the GPU
    evaluation. Every PV generator whose reactive output Q_g (MVAr) leaves
    [qmin, qmax] is then fixed at the violated limit. Its bus becomes a PQ
    bus, so ``build_system`` folds it in as negative demand, and the case is
    solved again, warm-started from the previous state. Other generators at
    that bus keep their current Q_g. The loop stops when no limit is
    violated, when a solve does not converge, or after ``max_rounds``
    solves. Slack generators are never switched. The pattern changes with
    the bus types, so each round builds a new plan (on the device,
    milliseconds).
    """
    from dataclasses import replace

    from .system_model import build_system, flat_start

    opts = opts or NewtonOptions()
    if max_rounds < 1:
        raise ValueError("max_rounds must be >= 1")
    case = raw
    switched: list = []
    y = None if y0 is None else np.asarray(y0, dtype=np.float64)
    prev = None                       # (system, y) of the previous round
    for rnd in range(1, max_rounds + 1):
        sys = build_system(case)
        if y is None:
            y = flat_start(sys)
        elif prev is not None:        # carry theta, V, the kept Q_g and the slack over
            psys, py = prev
            nb = sys.n_bus
            keep = {int(r): k for k, r in enumerate(_pv_gen_rows(prev_case))}
            y_new = flat_start(sys)
            y_new[: 2 * nb] = py[: 2 * nb]
            for k, r in enumerate(_pv_gen_rows(case)):
                y_new[2 * nb + k] = py[2 * nb + keep[int(r)]]
            n_pv, n_pv_old = len(sys.pv.bus), len(psys.pv.bus)
            ns = len(sys.slack.bus)
            y_new[2 * nb + n_pv: 2 * nb + n_pv + 2 * ns] = \
                py[2 * nb + n_pv_old: 2 * nb + n_pv_old + 2 * ns]
            y = y_new
        res = newton_solve(sys, y, opts, solver)
        if not res.converged or rnd == max_rounds:
            return QLimitResult(res, case, sys, switched, rnd)
        rows = _pv_gen_rows(case)
        qg = res.y[2 * sys.n_bus: 2 * sys.n_bus + len(rows)] * case.base_mva
        order = np.argsort(case.bus_id, kind="stable")
        gbus = order[np.searchsorted(case.bus_id[order], case.gen_bus[rows])]
        at_pv_bus = case.bus_type[gbus] == 2       # the slack bus keeps its type
        over = at_pv_bus & (qg > case.qmax[rows])
        under = at_pv_bus & (qg < case.qmin[rows])
        if not (over | under).any():
            return QLimitResult(res, case, sys, switched, rnd)
        new_qg = np.array(case.qg, dtype=np.float64)
        new_type = np.array(case.bus_type)
        for k, r in enumerate(rows):
            new_qg[r] = qg[k]                    # every PV gen keeps its solved Q_g ...
        for k in np.flatnonzero(over | under):   # ... the violators sit at their limit
            r = int(rows[k])
            lim = float(case.qmax[r] if over[k] else case.qmin[r])
            new_qg[r] = lim
            switched.append((r, "qmax" if over[k] else "qmin", lim))
            new_type[gbus[k]] = 1                # PV -> PQ
        prev, prev_case = (sys, res.y), case
        case = replace(case, qg=new_qg, bus_type=new_type)
    raise AssertionError("unreachable")
