"""Residual evaluation g(y) behind the reference's workspace API.

Drop-in for pflow/residual.py: ``ResidualWorkspace`` exposes ``sys``,
``residual``, ``bind`` and ``run`` with the same argument meaning and the
same ``ValueError`` on shape mismatch (pflow/residual.py:129-144), so it can
be passed to the reference's own ``newton_solve(..., residual_ws=...)``
(pflow/newton.py:49-70).  The workflow config argument is accepted and
ignored: there is one GPU path, not six CPU workflows.

The arithmetic runs in libpfgpu's fused kernel (``pf_eval``): one thread per
bus walks its incident branches in the reference's join order, so there is
no contribution pool and no separate join pass.
"""

from __future__ import annotations

import numpy as np

from .plan import HostPin, Plan, pinned_zeros


class ResidualWorkspace:
    """GPU residual workspace for one system (pflow/residual.py:46-255)."""

    def __init__(self, sys, plan: Plan | None = None):
        self.sys = sys
        self.plan = plan if plan is not None else Plan(sys)
        self.n_eq = self.plan.n_eq
        self._pinned, self.residual = pinned_zeros(self.n_eq)   # page-locked: one DMA per run
        self._bound = None
        self._out = None
        self._paired = None   # a JacobianWorkspace fused with this one (jacobian.py)
        self._pin = HostPin()  # page-locks the bound state vector

    def bind(self, y, out, cfg=None):
        """Validate and remember the output buffer (pflow/residual.py:129-144)."""
        if out is None:
            out = self.residual
        key = (id(y), id(out))
        if self._bound == key:
            return out
        if y.shape != (self.plan.n_var,):
            raise ValueError(f"state vector has shape {y.shape}, expected ({self.plan.n_var},)")
        if out.shape != (self.n_eq,):
            raise ValueError(f"residual vector has shape {out.shape}, expected ({self.n_eq},)")
        if out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("residual vector must be contiguous float64")
        self._out = out
        self._bound = key
        if isinstance(y, np.ndarray) and y.dtype == np.float64:
            self._pin.hold(y)   # later uploads of y by DMA (residual.py:137-140 rebinds by id)
        return out

    def run(self, y, cfg=None):
        out = self.bind(y, self._out, cfg)
        jws = self._paired
        if jws is not None:
            # fused: one upload of y and one launch give g and J; the paired
            # workspace returns this J for the same y object (see jacobian.py)
            self.plan.eval_host(y, g=out, jcsc=jws.csc.data)
            jws._fresh_for = id(y)
        else:
            self.plan.eval_host(y, g=out)
        return out


def evaluate_residual(sys, y, cfg=None, out=None, workspace: ResidualWorkspace | None = None):
    """g(y) into ``out`` (pflow/residual.py:262-274)."""
    ws = workspace if workspace is not None else ResidualWorkspace(sys)
    ws.bind(y, out, cfg)
    return ws.run(y, cfg)


def _to_device(plan: Plan, y):
    import torch

    if isinstance(y, torch.Tensor):
        return y.to(plan.device, torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(y, dtype=np.float64), device=plan.device)


def line_injections(sys, y, plan: Plan | None = None):
    """Per-line terminal injections (pflow/residual.py:287-314).

    Writes ``sys.lines.ph/pk/qh/qk`` like the reference (when the group has
    those scratch arrays) and returns them as numpy arrays.
    """
    plan = plan if plan is not None else Plan(sys)
    outs = [t.cpu().numpy() for t in plan.line_injections(_to_device(plan, y))]
    ln = sys.lines
    for name, arr in zip(("ph", "pk", "qh", "qk"), outs):
        dst = getattr(ln, name, None)
        if dst is not None and dst.shape == arr.shape:
            dst[:] = arr
    return tuple(outs)


def _device_pool(sys, y, plan: Plan | None):
    plan = plan if plan is not None else Plan(sys)
    pool = plan.device_injections(_to_device(plan, y)).cpu().numpy()
    P, G, S, H = plan.n_pq, plan.n_pv, plan.n_slack, plan.n_shunt
    cuts = np.cumsum([P, P, G, G, G, S, S, S, S, H])
    return np.split(pool, cuts)


def pq_injections(sys, y, plan: Plan | None = None):
    """(p, q) contributions of PQ devices (pflow/residual.py:317-325)."""
    seg = _device_pool(sys, y, plan)
    return seg[0], seg[1]


def pv_injections(sys, y, plan: Plan | None = None):
    """(p, q, verr) of PV devices (pflow/residual.py:328-337)."""
    seg = _device_pool(sys, y, plan)
    return seg[2], seg[3], seg[4]


def slack_injections(sys, y, plan: Plan | None = None):
    """(p, q, verr, therr) of slack devices (pflow/residual.py:340-351)."""
    seg = _device_pool(sys, y, plan)
    return seg[5], seg[6], seg[7], seg[8]


def shunt_injections(sys, y, plan: Plan | None = None):
    """(p, q) of shunts (pflow/residual.py:354-362)."""
    seg = _device_pool(sys, y, plan)
    return seg[9], seg[10]
