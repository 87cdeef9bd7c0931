"""Jacobian values on the fixed pattern, behind the reference's workspace API.

Drop-in for pflow/jacobian.py: ``JacobianWorkspace.run(y, cfg)`` returns the
same ``scipy.sparse.csc_matrix`` object on every call with its data refreshed
in place (pflow/jacobian.py:173-176); ``indptr``/``indices`` equal the
reference's (the pattern is built on the device by ``pf_plan_create`` and
checked bit-for-bit in tests).  The kernel writes values straight into the
CSR pattern; the CSC view is a device-side permutation gather.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .plan import HostPin, Plan, pinned_zeros
from .residual import ResidualWorkspace, evaluate_residual


class JacobianWorkspace:
    """Fixed pattern + assembled CSC matrix for one system (pflow/jacobian.py:39-176)."""

    def __init__(self, sys, plan: Plan | None = None, residual_ws: ResidualWorkspace | None = None):
        """``residual_ws`` (optional) fuses the pair: its ``run(y)`` then
        evaluates g and J in one upload and one launch, and this
        workspace's next ``run`` with the same y object returns that J
        without evaluating again -- the call pattern of pflow's
        newton_solve (newton.py:81, 97), which leaves y untouched between
        the two.  A caller that modifies y in place between the two calls
        must not pair the workspaces."""
        self.sys = sys
        if residual_ws is not None:
            if plan is not None and plan is not residual_ws.plan:
                raise ValueError("a fused pair must share one plan")
            plan = residual_ws.plan
        self.plan = plan if plan is not None else Plan(sys)
        n = self.plan.n_var
        indptr, indices, perm = self.plan.pattern_csc()
        self.nnz = self.plan.nnz
        # the values live in page-locked host memory, so each refresh is one
        # DMA at full PCIe rate instead of a staged pageable copy
        self._pinned, data = pinned_zeros(self.nnz)
        self.csc = sp.csc_matrix((data, indices, indptr), shape=(n, n))
        if not np.shares_memory(self.csc.data, data):
            self.csc.data = data
        self.csc_perm = perm
        self._bound = None
        self._fresh_for = None   # id(y) whose J the paired residual run left in csc
        self._pin = HostPin()
        if residual_ws is not None:
            residual_ws._paired = self

    def pattern_csr(self):
        """(indptr, indices) of the device CSR pattern (== csc.tocsr())."""
        return self.plan.pattern_csr()

    def bind(self, y, cfg=None) -> None:
        key = id(y)
        if self._bound == key:
            return
        if y.shape != (self.plan.n_var,):
            raise ValueError(f"state vector has shape {y.shape}, expected ({self.plan.n_var},)")
        self._bound = key
        if isinstance(y, np.ndarray) and y.dtype == np.float64:
            self._pin.hold(y)

    def run(self, y, cfg=None) -> sp.csc_matrix:
        self.bind(y, cfg)
        if self._fresh_for is not None and self._fresh_for == id(y):
            self._fresh_for = None          # J of this y came with the residual run
            return self.csc
        self._fresh_for = None
        self.plan.eval_host(y, jcsc=self.csc.data)
        return self.csc


def symbolic_pattern(sys, plan: Plan | None = None) -> JacobianWorkspace:
    """Build the pattern once (pflow/jacobian.py:211-213)."""
    return JacobianWorkspace(sys, plan)


def evaluate_jacobian(sys, y, cfg=None, ws: JacobianWorkspace | None = None) -> sp.csc_matrix:
    """Refresh the Jacobian values in place (pflow/jacobian.py:216-221)."""
    if ws is None:
        ws = JacobianWorkspace(sys)
    if ws.sys is not sys:
        raise ValueError("workspace was built for a different system")
    return ws.run(y, cfg)


def finite_difference_jacobian(sys, y, step: float | None = None,
                               workspace: ResidualWorkspace | None = None) -> np.ndarray:
    """Dense central differences of the GPU residual (pflow/jacobian.py:224-249).

    Test oracle: column steps 1e-6 * max(1, |y_j|); guarded to n_var <= 2000.
    """
    n = y.shape[0]
    if n > 2000:
        raise ValueError(f"finite differences guarded to n_var <= 2000, got {n}")
    ws = workspace if workspace is not None else ResidualWorkspace(sys)
    g_plus = np.zeros(n)
    g_minus = np.zeros(n)
    jac = np.zeros((n, n))
    yw = np.array(y, dtype=np.float64)
    for j in range(n):
        hj = step if step is not None else 1e-6 * max(1.0, abs(y[j]))
        yj = yw[j]
        yw[j] = yj + hj
        evaluate_residual(sys, yw, None, g_plus, ws)
        yw[j] = yj - hj
        evaluate_residual(sys, yw, None, g_minus, ws)
        yw[j] = yj
        jac[:, j] = (g_plus - g_minus) / (2.0 * hj)
    return jac


def export_matrix_market(ws: JacobianWorkspace, path) -> None:
    """MatrixMarket dump of the assembled matrix (pflow/jacobian.py:252-256)."""
    from scipy.io import mmwrite

    mmwrite(str(path), ws.csc.tocoo())
