"""CPU oracle for the f+J evaluation path - TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / CPU baseline, never as the measured product path.

``liboracle.so`` (built from pf_oracle.c / pf_oracle_wf5.c by the Makefile
here) restates the reference pflow package's evaluation
(/root/reference/pkg/src/pflow: residual.py, jacobian.py, kernels.py,
workflow.py) in C.  Its wf1 is pinned bit-for-bit against golden vectors the
reference itself produced (tests/golden, scripts/make_golden.py).
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

from paper_2011_11880_b200._abi import PfTopology, topology

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"
_VP = C.c_void_p
_LIB = None

ORC_NVAR, ORC_NNZ, ORC_NSLOTS, ORC_NPOOL, ORC_NJOIN = range(5)


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            build()
        h = C.CDLL(str(LIB_PATH))
        sigs = {
            "orc_plan_create": (_VP, [C.POINTER(PfTopology)]),
            "orc_plan_destroy": (None, [_VP]),
            "orc_plan_info": (C.c_int64, [_VP, C.c_int]),
            "orc_plan_pattern": (None, [_VP, _VP, _VP]),
            "orc_plan_join": (None, [_VP, _VP, _VP, _VP]),
            "orc_plan_slots": (None, [_VP, _VP, _VP, _VP, _VP]),
            "orc_ws_create": (_VP, [_VP]),
            "orc_ws_destroy": (None, [_VP]),
            "orc_residual": (None, [_VP, C.c_int, _VP, _VP]),
            "orc_jacobian": (None, [_VP, C.c_int, _VP, _VP]),
            "orc_ws_pool": (_VP, [_VP]),
            "orc_ws_vals": (_VP, [_VP]),
            "orc_line_injections": (None, [_VP, C.c_int, _VP, _VP, _VP, _VP, _VP]),
            "orc_sincos_poly": (None, [_VP, _VP, _VP, C.c_int64]),
            "orc_libm_sincos": (None, [_VP, _VP, _VP, C.c_int64]),
            "orc_eval_threaded": (None, [_VP, _VP, _VP, _VP, C.c_int]),
            "orc_eval_scenarios": (C.c_int, [_VP, C.c_int, C.c_int32, _VP, _VP, _VP, _VP, _VP,
                                             _VP, _VP, _VP, C.c_int]),
        }
        for name, (res, args) in sigs.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = h
    return _LIB


def _p(a):
    return None if a is None else a.ctypes.data


class Oracle:
    """The reference's workspaces + kernels restated in C, for one system."""

    def __init__(self, sys):
        self.sys = sys
        t, keep = topology(sys)
        L = lib()
        self._plan = L.orc_plan_create(C.byref(t))
        del keep
        self._ws = L.orc_ws_create(self._plan)
        self.n_var = L.orc_plan_info(self._plan, ORC_NVAR)
        self.nnz = L.orc_plan_info(self._plan, ORC_NNZ)
        self.n_slots = L.orc_plan_info(self._plan, ORC_NSLOTS)
        self.n_pool = L.orc_plan_info(self._plan, ORC_NPOOL)
        self.n_join = L.orc_plan_info(self._plan, ORC_NJOIN)

    def __del__(self):
        L = _LIB
        if L is not None and getattr(self, "_plan", None):
            L.orc_ws_destroy(self._ws)
            L.orc_plan_destroy(self._plan)
            self._plan = None

    # -- structure ----------------------------------------------------------
    def pattern_csc(self):
        indptr = np.zeros(self.n_var + 1, np.int32)
        indices = np.zeros(self.nnz, np.int32)
        lib().orc_plan_pattern(self._plan, _p(indptr), _p(indices))
        return indptr, indices

    def join(self):
        ptr = np.zeros(self.n_var + 1, np.int32)
        split = np.zeros(self.n_var, np.int32)
        idx = np.zeros(self.n_join, np.int32)
        lib().orc_plan_join(self._plan, _p(ptr), _p(split), _p(idx))
        return ptr, split, idx

    def slots(self):
        rows = np.zeros(self.n_slots, np.int32)
        cols = np.zeros(self.n_slots, np.int32)
        s2c = np.zeros(self.n_slots, np.int32)
        gp = np.zeros(self.nnz + 1, np.int32)
        lib().orc_plan_slots(self._plan, _p(rows), _p(cols), _p(s2c), _p(gp))
        return rows, cols, s2c, gp

    # -- evaluation ---------------------------------------------------------
    def residual(self, y, wf: int = 1):
        y = np.ascontiguousarray(y, dtype=np.float64)
        g = np.zeros(self.n_var)
        lib().orc_residual(self._ws, wf, _p(y), _p(g))
        return g

    def jacobian(self, y, wf: int = 1):
        """CSC data in the reference's order (pflow JacobianWorkspace.csc)."""
        y = np.ascontiguousarray(y, dtype=np.float64)
        d = np.zeros(self.nnz)
        lib().orc_jacobian(self._ws, wf, _p(y), _p(d))
        return d

    def pool(self):
        a = (C.c_double * self.n_pool).from_address(lib().orc_ws_pool(self._ws))
        return np.frombuffer(a, dtype=np.float64).copy()

    def vals(self):
        a = (C.c_double * self.n_slots).from_address(lib().orc_ws_vals(self._ws))
        return np.frombuffer(a, dtype=np.float64).copy()

    def line_injections(self, y, wf: int = 1):
        y = np.ascontiguousarray(y, dtype=np.float64)
        L = len(self.sys.lines)
        out = [np.zeros(L) for _ in range(4)]
        lib().orc_line_injections(self._ws, wf, _p(y), *[_p(o) for o in out])
        return tuple(out)  # ph, pk, qh, qk

    def eval_threaded(self, y, nthreads: int):
        y = np.ascontiguousarray(y, dtype=np.float64)
        g = np.zeros(self.n_var)
        d = np.zeros(self.nnz)
        lib().orc_eval_threaded(self._ws, _p(y), _p(g), _p(d), nthreads)
        return g, d

    def eval_scenarios(self, K, y, pq_p=None, pq_q=None, pv_p=None, outage=None,
                       want_g=True, want_j=True, wf: int = 1, nthreads: int = 1):
        """Blocked-layout scenario batch (see include/pfgpu.h)."""
        nblk = -(-K // 32)
        g = np.zeros(nblk * 32 * self.n_var) if want_g else None
        j = np.zeros(nblk * 32 * self.nnz) if want_j else None
        norms = np.zeros(K)
        f = lambda a: None if a is None else np.ascontiguousarray(a)
        y, pq_p, pq_q, pv_p = f(y), f(pq_p), f(pq_q), f(pv_p)
        outage = None if outage is None else np.ascontiguousarray(outage, dtype=np.int32)
        lib().orc_eval_scenarios(self._plan, wf, K, _p(y), _p(pq_p), _p(pq_q), _p(pv_p),
                                 _p(outage), _p(g), _p(j), _p(norms), nthreads)
        return g, j, norms


def sincos_poly(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    s, c = np.zeros_like(x), np.zeros_like(x)
    lib().orc_sincos_poly(_p(x), _p(s), _p(c), x.size)
    return s, c


def libm_sincos(x):
    """glibc sin/cos (what pflow wf1 calls through @llvm.sin/cos.f64)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    s, c = np.zeros_like(x), np.zeros_like(x)
    lib().orc_libm_sincos(_p(x), _p(s), _p(c), x.size)
    return s, c
