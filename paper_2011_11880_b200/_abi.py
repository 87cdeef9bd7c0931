"""ctypes view of include/pfgpu.h and the loader for libpfgpu.so.

The product path has no fallback: if the CUDA library is missing or fails
to load, :func:`lib` raises ``RuntimeError`` naming the build command.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libpfgpu.so"

PF_OK, PF_EINVAL, PF_ECUDA, PF_ESHAPE, PF_ENOMEM = 0, 1, 2, 3, 4
PF_LANES = 32
(PF_DIM_NBUS, PF_DIM_NLINE, PF_DIM_NVAR, PF_DIM_NNZ, PF_DIM_NPQ, PF_DIM_NPV,
 PF_DIM_NSLACK, PF_DIM_NSHUNT, PF_DIM_NINC, PF_DIM_MAXDEG, PF_DIM_SG_CHUNKS, PF_DIM_SG_BIG,
 PF_DIM_COUNT) = range(13)

_I32P = C.POINTER(C.c_int32)
_F64P = C.POINTER(C.c_double)


class PfTopology(C.Structure):
    """``pf_topology`` (include/pfgpu.h)."""

    _fields_ = [
        ("n_bus", C.c_int32), ("n_line", C.c_int32),
        ("bus_h", _I32P), ("bus_k", _I32P),
        ("gl", _F64P), ("bl", _F64P), ("gl2", _F64P), ("bl2", _F64P),
        ("g_self_h", _F64P), ("b_self_h", _F64P), ("g_self_k", _F64P), ("b_self_k", _F64P),
        ("n_pq", C.c_int32), ("pq_bus", _I32P), ("pq_p0", _F64P), ("pq_q0", _F64P),
        ("n_pv", C.c_int32), ("pv_bus", _I32P), ("pv_p0", _F64P), ("pv_v0", _F64P),
        ("pv_qg", _I32P),
        ("n_slack", C.c_int32), ("sl_bus", _I32P), ("sl_v0", _F64P), ("sl_th0", _F64P),
        ("sl_qg", _I32P), ("sl_ps", _I32P),
        ("n_shunt", C.c_int32), ("sh_bus", _I32P), ("sh_g", _F64P), ("sh_b", _F64P),
    ]


def topology(sys):
    """Build a ``PfTopology`` from a PowerSystem (this package's or pflow's).

    Returns ``(struct, keepalive)``; keep ``keepalive`` referenced while the
    struct is in use (it owns the contiguous copies the pointers refer to).
    """
    keep = []

    def i32(a):
        a = np.ascontiguousarray(a, dtype=np.int32)
        keep.append(a)
        return a.ctypes.data_as(_I32P)

    def f64(a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        keep.append(a)
        return a.ctypes.data_as(_F64P)

    ln, pq, pv, sl, sh = sys.lines, sys.pq, sys.pv, sys.slack, sys.shunts
    t = PfTopology(
        n_bus=sys.n_bus, n_line=len(ln),
        bus_h=i32(ln.bus_h), bus_k=i32(ln.bus_k),
        gl=f64(ln.gl), bl=f64(ln.bl), gl2=f64(ln.gl2), bl2=f64(ln.bl2),
        g_self_h=f64(ln.g_self_h), b_self_h=f64(ln.b_self_h),
        g_self_k=f64(ln.g_self_k), b_self_k=f64(ln.b_self_k),
        n_pq=len(pq), pq_bus=i32(pq.bus), pq_p0=f64(pq.p0), pq_q0=f64(pq.q0),
        n_pv=len(pv), pv_bus=i32(pv.bus), pv_p0=f64(pv.p0), pv_v0=f64(pv.v0),
        pv_qg=i32(pv.qg),
        n_slack=len(sl), sl_bus=i32(sl.bus), sl_v0=f64(sl.v0), sl_th0=f64(sl.theta0),
        sl_qg=i32(sl.qg), sl_ps=i32(sl.ps),
        n_shunt=len(sh), sh_bus=i32(sh.bus), sh_g=f64(sh.g), sh_b=f64(sh.b),
    )
    return t, keep


_LIB = None
_VP = C.c_void_p

# name -> (restype, argtypes)
_SIGS = {
    "pf_last_error": (C.c_char_p, []),
    "pf_version": (C.c_int, []),
    "pf_plan_create": (C.c_int, [C.POINTER(PfTopology), C.POINTER(_VP)]),
    "pf_plan_destroy": (C.c_int, [_VP]),
    "pf_plan_dims": (C.c_int, [_VP, C.POINTER(C.c_int64)]),
    "pf_plan_pattern_csr": (C.c_int, [_VP, _VP, _VP]),
    "pf_plan_pattern_csc": (C.c_int, [_VP, _VP, _VP, _VP]),
    "pf_eval": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP]),
    "pf_eval_batched": (C.c_int, [_VP, C.c_int32, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "pf_jac_to_csc": (C.c_int, [_VP, C.c_int32, _VP, _VP, _VP]),
    "pf_eval_host": (C.c_int, [_VP, _VP, _VP, _VP, _VP]),
    "pf_eval_batched_host": (C.c_int, [_VP, C.c_int32, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                       _VP, C.c_int32, C.c_int32]),
    "pf_line_injections": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "pf_line_jacobian_slots": (C.c_int, [_VP, _VP, _VP, _VP]),
    "pf_device_injections": (C.c_int, [_VP, _VP, _VP, _VP]),
    "pf_device_jacobian_slots": (C.c_int, [_VP, _VP, _VP, _VP]),
    "pf_join_rows": (C.c_int, [C.c_int32, _VP, _VP, _VP, _VP, _VP, _VP]),
    "pf_gather_sum": (C.c_int, [C.c_int32, _VP, _VP, _VP, _VP, _VP]),
    "pf_sincos": (C.c_int, [C.c_int64, _VP, _VP, _VP, _VP]),
    "pf_batch_unblock": (C.c_int, [C.c_int32, C.c_int32, _VP, _VP, C.c_double, _VP]),
    "pf_batch_update": (C.c_int, [C.c_int32, C.c_int32, _VP, _VP, _VP, _VP]),
    "pf_lu_scatter": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _VP, _VP, _VP, _VP]),
    "pf_lu_eliminate": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _VP, _VP, _VP, _VP, _VP]),
    "pf_lu_tail_gather": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _VP, _VP, _VP, _VP]),
    "pf_lu_rhs": (C.c_int, [C.c_int32, C.c_int32, _VP, _VP, _VP, C.c_double, _VP]),
    "pf_lu_forward": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, _VP, _VP, _VP,
                                C.c_int32, _VP, _VP, _VP]),
    "pf_lu_backward": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, _VP, _VP, _VP,
                                 _VP, _VP, _VP, _VP]),
    "pf_lu_tail_vec": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, _VP, _VP, C.c_int32,
                                 _VP]),
    "pf_lu_apply": (C.c_int, [C.c_int32, C.c_int32, _VP, _VP, _VP, _VP, _VP]),
    "pf_lu_residual": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _VP, _VP, _VP, _VP, _VP, _VP,
                                 _VP]),
    "pf_launch_count": (C.c_int64, []),
    "pf_alloc_count": (C.c_int64, []),
    "pf_host_register": (C.c_int, [_VP, C.c_size_t]),
    "pf_host_unregister": (C.c_int, [_VP]),
}

EXPORTED = tuple(_SIGS)


def lib():
    """The loaded libpfgpu.so (raises if it is not built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = Path(os.environ.get("PFGPU_LIB", LIB_PATH))
    if not path.exists():
        raise RuntimeError(
            f"CUDA library {path} is missing: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    try:
        handle = C.CDLL(str(path))
    except OSError as e:
        raise RuntimeError(f"failed to load {path}: {e}") from e
    partial = os.environ.get("PFGPU_LIB_PARTIAL") == "1"   # dev A/B of older builds only
    for name, (res, args) in _SIGS.items():
        if partial and not hasattr(handle, name):
            continue
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = handle
    return _LIB


class PfError(RuntimeError):
    """Non-shape failure reported by libpfgpu (CUDA error, allocation)."""


def check(status: int) -> None:
    """Map a pf status code to a Python exception (pflow raises ValueError
    for argument/shape problems, residual.py:141-144)."""
    if status == PF_OK:
        return
    msg = lib().pf_last_error()
    msg = msg.decode() if msg else f"status {status}"
    if status in (PF_EINVAL, PF_ESHAPE):
        raise ValueError(msg)
    raise PfError(msg)


def ptr(t) -> int | None:
    """data_ptr of a torch tensor / numpy array, or None."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()
