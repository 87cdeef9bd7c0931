"""Device plan: the network uploaded once, symbolic pattern built on the GPU.

``Plan`` wraps ``pf_plan`` from libpfgpu.so (include/pfgpu.h).  PyTorch is
used only for device buffers and streams; every kernel is this package's own
sm_100a CUDA code.  There is no CPU fallback: constructing a Plan without a
GPU or without the built library raises.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import PF_LANES, check, lib


def _torch():
    import torch

    return torch


def _stream_ptr(stream, device=None) -> int:
    """Raw cudaStream_t: ``stream`` (a torch stream or an int), else the
    current stream of ``device``.  A torch stream of another device is
    rejected."""
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream(device)
    if device is not None and hasattr(stream, "device") and stream.device != device:
        raise ValueError(f"stream is on {stream.device}, the plan on {device}")
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _on_device(fn):
    """Run a Plan method with the plan's device current: kernels launch, and
    plan-owned staging is allocated, in the plan's context whatever device
    the caller has current (switched only when it differs)."""
    import functools

    @functools.wraps(fn)
    def wrapped(self, *a, **k):
        torch = _torch()
        if torch.cuda.current_device() == self.device.index:
            return fn(self, *a, **k)
        with torch.cuda.device(self.device):
            return fn(self, *a, **k)

    return wrapped


class HostPin:
    """Page-locks one caller-owned host array at a time (pf_host_register)
    and keeps a reference to it until released, so the pages stay valid
    while registered.  The workspaces pin the state vector they are bound to:
    pflow's Newton loop keeps one y for the whole solve (newton.py:69), so
    every upload after the first runs at full PCIe rate."""

    def __init__(self):
        self._arr = None

    def hold(self, a) -> None:
        if a is self._arr:
            return
        self.release()
        if (isinstance(a, np.ndarray) and a.flags.c_contiguous and a.nbytes
                and _torch().cuda.is_available()):
            check(lib().pf_host_register(a.ctypes.data, a.nbytes))
            self._arr = a

    def release(self) -> None:
        if self._arr is not None:
            a, self._arr = self._arr, None
            check(lib().pf_host_unregister(a.ctypes.data))

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def _host(a, n: int, name: str, dtype=np.float64):
    """Host array argument of the *_host entry points: C-contiguous, of
    ``dtype``, at least ``n`` entries; returns its address (None passes)."""
    if a is None:
        return None
    if not isinstance(a, np.ndarray):
        raise ValueError(f"{name} must be a numpy array")
    if a.dtype != dtype or not a.flags.c_contiguous:
        raise ValueError(f"{name} must be a C-contiguous {np.dtype(dtype).name} array")
    if a.size < n:
        raise ValueError(f"{name} has {a.size} entries, expected >= {n}")
    return a.ctypes.data


def pinned_zeros(n: int):
    """(owner, array): a zeroed float64 numpy array of n entries in
    page-locked host memory when CUDA is available (pageable otherwise);
    keep ``owner`` alive as long as the array is used."""
    torch = _torch()
    if torch.cuda.is_available():
        t = torch.zeros(max(n, 1), dtype=torch.float64, pin_memory=True)
        return t, t.numpy()[:n]
    a = np.zeros(n)
    return a, a


def n_blocks(K: int) -> int:
    return -(-int(K) // PF_LANES)


def to_blocked(a: np.ndarray) -> np.ndarray:
    """[K, n] scenario-major -> flat PF_LANES-blocked layout (include/pfgpu.h)."""
    a = np.asarray(a)
    K, n = a.shape
    nb = n_blocks(K)
    pad = np.zeros((nb * PF_LANES, n), dtype=a.dtype)
    pad[:K] = a
    return np.ascontiguousarray(pad.reshape(nb, PF_LANES, n).transpose(0, 2, 1)).reshape(-1)


def from_blocked(flat, K: int, n: int):
    """Inverse of :func:`to_blocked` (numpy or torch), returns [K, n]."""
    nb = n_blocks(K)
    if isinstance(flat, np.ndarray):
        return flat.reshape(nb, n, PF_LANES).transpose(0, 2, 1).reshape(nb * PF_LANES, n)[:K]
    return flat.reshape(nb, n, PF_LANES).permute(0, 2, 1).reshape(nb * PF_LANES, n)[:K]


class Plan:
    """One network on one GPU: topology, coefficients, Jacobian pattern."""

    def __init__(self, sys, device=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2011_11880_b200 needs a CUDA GPU (no CPU fallback)")
        dev = torch.device("cuda" if device is None else device)
        if dev.type != "cuda":
            raise ValueError(f"Plan needs a CUDA device, got {dev}")
        self.device = torch.device("cuda", torch.cuda.current_device() if dev.index is None
                                   else dev.index)
        self.sys = sys
        L = lib()
        t, keep = _abi.topology(sys)
        handle = C.c_void_p()
        with torch.cuda.device(self.device):
            check(L.pf_plan_create(C.byref(t), C.byref(handle)))
        del keep
        self._h = handle
        dims = (C.c_int64 * _abi.PF_DIM_COUNT)()
        check(L.pf_plan_dims(self._h, dims))
        self.n_bus = dims[_abi.PF_DIM_NBUS]
        self.n_line = dims[_abi.PF_DIM_NLINE]
        self.n_var = dims[_abi.PF_DIM_NVAR]
        self.n_eq = self.n_var
        self.nnz = dims[_abi.PF_DIM_NNZ]
        self.n_pq = dims[_abi.PF_DIM_NPQ]
        self.n_pv = dims[_abi.PF_DIM_NPV]
        self.n_slack = dims[_abi.PF_DIM_NSLACK]
        self.n_shunt = dims[_abi.PF_DIM_NSHUNT]
        self.max_degree = dims[_abi.PF_DIM_MAXDEG]
        self.single_chunks = dims[_abi.PF_DIM_SG_CHUNKS]      # single-grid CTAs
        self.single_serial = dims[_abi.PF_DIM_SG_BIG]         # over-cap buses done serially

    def close(self) -> None:
        if getattr(self, "_h", None):
            with _torch().cuda.device(self.device):
                lib().pf_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- pattern ------------------------------------------------------------
    @_on_device
    def pattern_csr(self):
        indptr = np.zeros(self.n_var + 1, np.int32)
        indices = np.zeros(max(self.nnz, 1), np.int32)
        check(lib().pf_plan_pattern_csr(self._h, indptr.ctypes.data, indices.ctypes.data))
        return indptr, indices[: self.nnz]

    @_on_device
    def pattern_csc(self):
        indptr = np.zeros(self.n_var + 1, np.int32)
        indices = np.zeros(max(self.nnz, 1), np.int32)
        perm = np.zeros(max(self.nnz, 1), np.int32)
        check(lib().pf_plan_pattern_csc(self._h, indptr.ctypes.data, indices.ctypes.data,
                                        perm.ctypes.data))
        return indptr, indices[: self.nnz], perm[: self.nnz]

    # -- buffers ------------------------------------------------------------
    def empty(self, n: int, K: int = 0, dtype=None):
        """Device buffer for ``n`` entries (single grid) or K scenarios."""
        torch = _torch()
        dtype = dtype or torch.float64
        size = n if K == 0 else n_blocks(K) * PF_LANES * n
        return torch.empty(max(size, 1), dtype=dtype, device=self.device)

    def _dev(self, t, n: int, name: str, K: int = 0, dtype=None):
        if t is None:
            return None
        torch = _torch()
        dtype = dtype or torch.float64
        need = n if K == 0 else n_blocks(K) * PF_LANES * n
        if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
            raise ValueError(f"{name} must be a CUDA tensor")
        if t.device != self.device:
            raise ValueError(f"{name} is on {t.device}, the plan on {self.device}")
        if t.dtype != dtype or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous {dtype} tensor")
        if t.numel() < need:
            raise ValueError(f"{name} has {t.numel()} elements, expected >= {need}")
        return t.data_ptr()

    # -- evaluation (device pointers) -----------------------------------------
    @_on_device
    def eval(self, y, g=None, jval=None, norm=None, stream=None) -> None:
        """Fused f+J of one grid: ``pf_eval``.  jval is CSR-ordered."""
        check(lib().pf_eval(self._h, self._dev(y, self.n_var, "y"), self._dev(g, self.n_var, "g"),
                            self._dev(jval, self.nnz, "jval"), self._dev(norm, 1, "norm"),
                            _stream_ptr(stream, self.device)))

    @_on_device
    def eval_batched(self, K: int, y, pq_p=None, pq_q=None, pv_p=None, outage=None, g=None,
                     jval=None, norms=None, stream=None) -> None:
        """K scenarios in the blocked layout: ``pf_eval_batched``."""
        torch = _torch()
        check(lib().pf_eval_batched(
            self._h, int(K), self._dev(y, self.n_var, "y", K),
            self._dev(pq_p, self.n_pq, "pq_p", K), self._dev(pq_q, self.n_pq, "pq_q", K),
            self._dev(pv_p, self.n_pv, "pv_p", K),
            self._dev(outage, K, "outage", 0, torch.int32),
            self._dev(g, self.n_var, "g", K), self._dev(jval, self.nnz, "jval", K),
            self._dev(norms, K, "norms"), _stream_ptr(stream, self.device)))

    @_on_device
    def jac_to_csc(self, jcsr, jcsc, K: int = 0, stream=None) -> None:
        check(lib().pf_jac_to_csc(self._h, int(K), self._dev(jcsr, self.nnz, "jcsr", K),
                                  self._dev(jcsc, self.nnz, "jcsc", K),
                                  _stream_ptr(stream, self.device)))

    # -- host-buffer drop-in ------------------------------------------------
    @_on_device
    def eval_host(self, y: np.ndarray, g: np.ndarray | None = None,
                  jcsc: np.ndarray | None = None, norm: np.ndarray | None = None) -> None:
        """``pf_eval_host``: numpy in, numpy out (J in the reference's CSC order)."""
        def chk(a, n, name):
            if a is None:
                return None
            if a.dtype != np.float64 or not a.flags.c_contiguous or a.size != n:
                raise ValueError(f"{name} must be a contiguous float64 array of size {n}")
            return a.ctypes.data
        y = np.ascontiguousarray(y, dtype=np.float64)
        if y.shape != (self.n_var,):
            raise ValueError(f"state vector has shape {y.shape}, expected ({self.n_var},)")
        check(lib().pf_eval_host(self._h, y.ctypes.data, chk(g, self.n_var, "g"),
                                 chk(jcsc, self.nnz, "jcsc"), chk(norm, 1, "norm")))

    @_on_device
    def eval_batched_host(self, K: int, y, pq_p=None, pq_q=None, pv_p=None, outage=None,
                          g=None, jval=None, norms=None, blocks_per_stage: int = 1,
                          n_streams: int = 3) -> None:
        """``pf_eval_batched_host``: host arrays (ideally pinned) in blocked
        layout.  Every array is checked (dtype, contiguity, size; outage
        indices in [-1, n_line)) before any copy touches it."""
        K = int(K)
        if K < 0:
            raise ValueError(f"K = {K} < 0")
        lanes = n_blocks(K) * PF_LANES
        if y is None:
            raise ValueError("y is required")
        args = [_host(y, lanes * self.n_var, "y"), _host(pq_p, lanes * self.n_pq, "pq_p"),
                _host(pq_q, lanes * self.n_pq, "pq_q"), _host(pv_p, lanes * self.n_pv, "pv_p"),
                _host(outage, K, "outage", np.int32), _host(g, lanes * self.n_var, "g"),
                _host(jval, lanes * self.nnz, "jval"), _host(norms, K, "norms")]
        if outage is not None and K and (outage[:K].min() < -1 or outage[:K].max() >= self.n_line):
            raise ValueError(f"outage indices must lie in [-1, {self.n_line})")
        check(lib().pf_eval_batched_host(self._h, K, *args, int(blocks_per_stage),
                                         int(n_streams)))

    # -- per-model entry points -----------------------------------------------
    @_on_device
    def line_injections(self, y, stream=None):
        """(ph, pk, qh, qk) device tensors (pflow residual.py:287-314)."""
        out = [self.empty(self.n_line) for _ in range(4)]
        check(lib().pf_line_injections(self._h, self._dev(y, self.n_var, "y"),
                                       *[o.data_ptr() for o in out],
                                       _stream_ptr(stream, self.device)))
        return tuple(o[: self.n_line] for o in out)

    @_on_device
    def line_jacobian_slots(self, y, stream=None):
        """[16, n_line] line partials (pflow kernels.py:128-163)."""
        out = self.empty(16 * self.n_line)
        check(lib().pf_line_jacobian_slots(self._h, self._dev(y, self.n_var, "y"),
                                           out.data_ptr(), _stream_ptr(stream, self.device)))
        return out[: 16 * self.n_line].view(16, self.n_line)

    @_on_device
    def device_injections(self, y, stream=None):
        """Pool segments 4..14 of pflow residual.py:57."""
        n = 2 * self.n_pq + 3 * self.n_pv + 4 * self.n_slack + 2 * self.n_shunt
        out = self.empty(n)
        check(lib().pf_device_injections(self._h, self._dev(y, self.n_var, "y"), out.data_ptr(),
                                         _stream_ptr(stream, self.device)))
        return out[:n]

    @_on_device
    def device_jacobian_slots(self, y, stream=None):
        n = 2 * self.n_pv + 4 * self.n_slack + 2 * self.n_shunt
        out = self.empty(n)
        check(lib().pf_device_jacobian_slots(self._h, self._dev(y, self.n_var, "y"),
                                             out.data_ptr(), _stream_ptr(stream, self.device)))
        return out[:n]


def join_rows(ptr_, split, idx, pool, out, stream=None) -> None:
    """Device row join (pflow kernels.py:265-274) on int32/float64 CUDA tensors."""
    n = out.numel()
    with _torch().cuda.device(out.device):
        check(lib().pf_join_rows(n, ptr_.data_ptr(), split.data_ptr(), idx.data_ptr(),
                                 pool.data_ptr(), out.data_ptr(), _stream_ptr(stream, out.device)))


def gather_sum(ptr_, idx, vals, out, stream=None) -> None:
    """Device duplicate-slot assembly (pflow kernels.py:277-282)."""
    n = out.numel()
    with _torch().cuda.device(out.device):
        check(lib().pf_gather_sum(n, ptr_.data_ptr(), idx.data_ptr(), vals.data_ptr(),
                                  out.data_ptr(), _stream_ptr(stream, out.device)))


def sincos(x, stream=None):
    """(sin x, cos x) with the engine's device trig (CUDA float64 tensor in)."""
    torch = _torch()
    x = x.contiguous()
    s, c = torch.empty_like(x), torch.empty_like(x)
    with torch.cuda.device(x.device):
        check(lib().pf_sincos(x.numel(), x.data_ptr(), s.data_ptr(), c.data_ptr(),
                              _stream_ptr(stream, x.device)))
    return s, c


def launch_count() -> int:
    """Kernels libpfgpu has launched in this process."""
    return int(lib().pf_launch_count())


def alloc_count() -> int:
    """Device allocations libpfgpu has made in this process."""
    return int(lib().pf_alloc_count())
