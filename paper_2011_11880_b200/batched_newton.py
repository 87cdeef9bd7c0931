"""Scenario-batched Newton-Raphson on the device.

Each iteration:

* evaluates g, J and the per-scenario norms of all K scenarios with
  ``pf_eval_batched`` (the product path);
* hands J and -g to a batched sparse LU refactorisation on the fixed pattern,
  and solves;
* updates the scenarios that are still iterating with ``y += dy``.

The refactorisation is cuSOLVER's refactorisation on a fixed pattern
(cusolverRf): one symbolic LU with fixed pivoting, shared by every scenario
and every iteration. This mirrors what pflow's ``BuiltinLU`` does for one
system (linear_solver.py:158-226): keep the pattern and the symbolic
factorisation, and refactor numerically each iteration. The base
factorisation of each scenario comes from SuperLU on its Jacobian at the
initial state (see ``base_lu``).

cusolverRf's batched entry points (cusolverRfBatch*) crash inside
cusolverRfBatchAnalyze on this B200 stack (CUDA 12.9, driver 580), even for a
6 x 6 tridiagonal system; scripts/dbg/rf_test.cu reproduces it. So each
scenario gets its own cusolverRf handle and the scenarios are refactored one
after another.

Fill limits the size. Random spanning-tree grids with long-range extra edges
fill badly: L+U has 0.31M entries for config 0 (2k buses) and 6.5M for
config 1 (10k buses), so K scenarios need K times that on the device.

The convergence logic restates pflow/newton.py:49-112 per scenario. A
scenario stops when max|g| <= tol. It diverges when the norm is non-finite or
above 1e6, or when its pivots break down (for example an outage that islands
buses). After ``max_iter`` updates it is reported as not converged.

The linear solve is outside the product (BASELINE.json north star): this
module is the hand-off, measured by ``scripts/batched_newton_bench.py``.
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import _abi
from .plan import PF_LANES, Plan

_DIVERGENCE_LIMIT = 1e6   # pflow/newton.py:23
_LIN_RTOL = 1e-10         # accepted residual of a device solve, relative to max|g|

# cusolverRf enums (cusolverRf.h)
_RF_FORMAT_CSR = 0
_RF_UNIT_DIAGONAL_STORED_L = 0
_RF_FACTORIZATION_ALG0 = 0
_RF_TRIANGULAR_SOLVE_ALG1 = 1
_STATUS_ZERO_PIVOT = 10       # CUSOLVER_STATUS_ZERO_PIVOT (cusolver_common.h)


def _load_cusolver():
    """libcusolver matching torch's CUDA runtime (the pip wheel torch ships),
    else the toolkit's."""
    cands = []
    try:
        import nvidia.cusolver as m

        for d in m.__path__:
            cands.append(os.path.join(d, "lib", "libcusolver.so.11"))
    except ImportError:
        pass
    cands += ["/usr/local/cuda/lib64/libcusolver.so.11", "libcusolver.so.11"]
    err = None
    for c in cands:
        try:
            return C.CDLL(c)
        except OSError as e:
            err = e
    raise RuntimeError(f"libcusolver not found: {err}")


_LIB = None


def _rf():
    global _LIB
    if _LIB is None:
        lib = _load_cusolver()
        vp, i32, f64 = C.c_void_p, C.c_int, C.c_double
        sigs = {
            "cusolverRfCreate": [C.POINTER(vp)],
            "cusolverRfDestroy": [vp],
            "cusolverRfSetMatrixFormat": [vp, i32, i32],
            "cusolverRfSetAlgs": [vp, i32, i32],
            "cusolverRfSetNumericProperties": [vp, f64, f64],
            "cusolverRfSetupHost": [i32, i32, vp, vp, vp, i32, vp, vp, vp, i32, vp, vp, vp, vp, vp,
                                    vp],
            "cusolverRfAnalyze": [vp],
            "cusolverRfResetValues": [i32, i32, vp, vp, vp, vp, vp, vp],
            "cusolverRfRefactor": [vp],
            "cusolverRfSolve": [vp, vp, vp, i32, vp, i32, vp, i32],
        }
        for name, args in sigs.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
        _LIB = lib
    return _LIB


def _ck(status: int, what: str) -> None:
    if status != 0:
        raise RuntimeError(f"{what} failed (cusolverStatus {status})")


def robust_row_match(csr: sp.csr_matrix, n_bus: int):
    """Row order that puts outage-proof entries on the diagonal.

    Every generator row (g_V, g_theta: rows >= 2N, a single entry of value 1)
    goes to its only column (V_i or theta_i). Every generator column (Q_g,
    P_s: columns >= 2N, a single entry of value 1 in row g_q[i] or g_p[i])
    takes that row. The remaining bus rows keep their own diagonal, which is
    a sum over the bus's branches. No single outage can zero such a pivot, so
    one pivot order serves every contingency scenario. Returns the row order,
    or None when the structure does not allow it (for example two generators
    regulating one bus, which makes the Jacobian singular anyway)."""
    n = csr.shape[0]
    row_of = np.full(n, -1, np.int64)       # column -> matched row
    used = np.zeros(n, bool)
    csc = csr.tocsc()
    for r in range(2 * n_bus, n):
        cols = csr.indices[csr.indptr[r]:csr.indptr[r + 1]]
        if cols.size != 1 or row_of[cols[0]] >= 0:
            return None
        row_of[cols[0]] = r
        used[r] = True
    for c in range(2 * n_bus, n):
        rows = csc.indices[csc.indptr[c]:csc.indptr[c + 1]]
        rows = rows[rows < 2 * n_bus]
        if rows.size != 1 or used[rows[0]] or row_of[c] >= 0:
            return None
        row_of[c] = rows[0]
        used[rows[0]] = True
    for i in range(2 * n_bus):
        if row_of[i] < 0:
            if used[i]:
                return None
            row_of[i] = i
            used[i] = True
    if not used.all():
        return None
    return row_of


def base_lu(csc: sp.csc_matrix, seed: int = 0, n_bus: int | None = None):
    """Fixed pivoting and a closed symbolic pattern for cusolverRf.

    1. SuperLU on the actual base matrix, minimum degree on A^T + A with
       diagonal-preferring pivoting, gives the row / column orders: P, Q with
       M = A[P][:, Q] factorisable without further pivoting. With ``n_bus``
       the rows are first matched to outage-proof diagonals
       (``robust_row_match``) and SuperLU keeps the diagonal (symmetric mode,
       no threshold pivoting).
    2. The factor pattern must contain every entry that the numeric
       refactorisation can fill. SuperLU stores no exact zeros, so cancellation
       in step 1 would lose positions. The pattern is therefore recomputed on M
       with random values and a dominant diagonal (natural order, no pivoting,
       no cancellation).
    Returns CSR L (unit diagonal stored) and U with that pattern (their values
    are placeholders: every use refactors first), and P, Q."""
    A = csc.tocsc()
    match = robust_row_match(A.tocsr(), n_bus) if n_bus is not None else None
    if match is not None:
        A0 = sp.csr_matrix(A)[match].tocsc()
        lu = spla.splu(A0, permc_spec="MMD_AT_PLUS_A",
                       options=dict(DiagPivotThresh=0.0, SymmetricMode=True))
        P = match[np.argsort(lu.perm_r)].astype(np.int32)
        Q = np.argsort(lu.perm_c).astype(np.int32)
    else:
        lu = spla.splu(A, permc_spec="MMD_AT_PLUS_A", options=dict(DiagPivotThresh=0.001))
        P = np.argsort(lu.perm_r).astype(np.int32)
        Q = np.argsort(lu.perm_c).astype(np.int32)
    M = sp.csr_matrix(A)[P][:, Q].tocsr()
    rng = np.random.default_rng(seed)
    M.data = rng.uniform(0.5, 1.0, M.nnz)
    M = M.tolil()
    rows = np.asarray(abs(M).sum(axis=1)).ravel()
    M.setdiag(rows + 1.0)
    sym = spla.splu(M.tocsc(), permc_spec="NATURAL",
                    options=dict(DiagPivotThresh=0.0, SymmetricMode=True))
    if not (np.array_equal(sym.perm_r, np.arange(M.shape[0]))
            and np.array_equal(sym.perm_c, np.arange(M.shape[0]))):
        raise RuntimeError("symbolic factorisation pivoted")
    L = sp.csr_matrix(sym.L)
    U = sp.csr_matrix(sym.U)
    L.sort_indices()
    U.sort_indices()
    return L, U, P, Q


class BatchedLU:
    """K systems A_s x = b_s on one CSR pattern (the Jacobian's), refactored on
    the device each time the values change.  Scenario s keeps the pivoting and
    factor pattern of its own base matrix ``base_vals[s]`` (an outage changes
    which pivots are safe); a base that is singular marks the scenario
    singular from the start."""

    def __init__(self, K: int, indptr: np.ndarray, indices: np.ndarray, base_vals: np.ndarray,
                 device="cuda"):
        import torch

        self.K, self.n = int(K), int(indptr.shape[0] - 1)
        self.nnz = int(indices.shape[0])
        lib = _rf()
        rp = np.ascontiguousarray(indptr, dtype=np.int32)
        ci = np.ascontiguousarray(indices, dtype=np.int32)
        c32 = lambda a: np.ascontiguousarray(a, np.int32)
        f64 = lambda a: np.ascontiguousarray(a, np.float64)
        p = lambda a: a.ctypes.data
        t = lambda a: torch.as_tensor(a, device=device)
        self._h = [None] * self.K
        self._pq = [None] * self.K
        self.singular0 = np.zeros(self.K, dtype=bool)
        self.nnz_lu = np.zeros(self.K, dtype=np.int64)
        try:
            for s in range(self.K):
                vals = f64(base_vals[s])
                try:
                    L, U, P, Q = base_lu(sp.csr_matrix((vals, ci, rp), shape=(self.n, self.n)))
                except RuntimeError:           # SuperLU: exactly singular
                    self.singular0[s] = True
                    continue
                self.nnz_lu[s] = L.nnz + U.nnz
                h = C.c_void_p()
                _ck(lib.cusolverRfCreate(C.byref(h)), "cusolverRfCreate")
                self._h[s] = h
                _ck(lib.cusolverRfSetMatrixFormat(h, _RF_FORMAT_CSR, _RF_UNIT_DIAGONAL_STORED_L),
                    "cusolverRfSetMatrixFormat")
                _ck(lib.cusolverRfSetAlgs(h, _RF_FACTORIZATION_ALG0, _RF_TRIANGULAR_SOLVE_ALG1),
                    "cusolverRfSetAlgs")
                Lp, Li, Lx = c32(L.indptr), c32(L.indices), f64(L.data)
                Up, Ui, Ux = c32(U.indptr), c32(U.indices), f64(U.data)
                _ck(lib.cusolverRfSetupHost(self.n, self.nnz, p(rp), p(ci), p(vals), int(L.nnz),
                                            p(Lp), p(Li), p(Lx), int(U.nnz), p(Up), p(Ui), p(Ux),
                                            p(P), p(Q), h), "cusolverRfSetupHost")
                _ck(lib.cusolverRfAnalyze(h), "cusolverRfAnalyze")
                self._pq[s] = (t(P), t(Q))
        except Exception:
            self.close()
            raise
        self.d_rp, self.d_ci = t(rp), t(ci)
        self.vals = torch.empty((self.K, self.nnz), dtype=torch.float64, device=device)
        self.rhs = torch.empty((self.K, self.n), dtype=torch.float64, device=device)
        self.temp = torch.empty(self.n, dtype=torch.float64, device=device)

    def refactor_solve(self, which=None) -> np.ndarray:
        """self.rhs[s] <- A_s^{-1} self.rhs[s], A_s = self.vals[s] (CSR), for
        every s in ``which`` (default: all).  Returns the scenarios that are
        singular (a singular base, or a zero pivot in this refactorisation,
        e.g. an islanding outage); their rhs is left unsolved."""
        import torch

        torch.cuda.synchronize(self.vals.device)   # cusolverRf runs on the legacy stream
        lib = _rf()
        rp, ci = self.d_rp.data_ptr(), self.d_ci.data_ptr()
        singular = []
        for s in (range(self.K) if which is None else which):
            h = self._h[s]
            if h is None:
                singular.append(s)
                continue
            P, Q = (x.data_ptr() for x in self._pq[s])
            _ck(lib.cusolverRfResetValues(self.n, self.nnz, rp, ci, self.vals[s].data_ptr(), P, Q,
                                          h), "cusolverRfResetValues")
            st = lib.cusolverRfRefactor(h)
            if st == _STATUS_ZERO_PIVOT:
                singular.append(s)
                continue
            _ck(st, "cusolverRfRefactor")
            _ck(lib.cusolverRfSolve(h, P, Q, 1, self.temp.data_ptr(), self.n,
                                    self.rhs[s].data_ptr(), self.n), "cusolverRfSolve")
        torch.cuda.synchronize(self.vals.device)
        return np.asarray(singular, dtype=np.int64)

    def close(self) -> None:
        for h in getattr(self, "_h", []):
            if h:
                _rf().cusolverRfDestroy(h)
        self._h = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _host_solve(plan, K, j, g, sc, indptr, indices):
    """Scenario ``sc``'s Newton step on the host with SuperLU (own pivoting);
    None when its Jacobian is singular."""
    return _host_solves(plan, j, g, [sc], indptr, indices)[0]


_POOL = None


def _pool():
    """Worker processes for host SuperLU solves (spawned once, on first use)."""
    global _POOL
    if _POOL is None:
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor

        _POOL = ProcessPoolExecutor(max_workers=min(16, os.cpu_count() or 1),
                                    mp_context=mp.get_context("spawn"))
    return _POOL


def _host_solves(plan, j, g, scs, indptr, indices):
    """SuperLU steps of several scenarios, in parallel worker processes
    (``_superlu``); None where the Jacobian is singular."""
    import torch

    from . import _superlu

    n, nnz = plan.n_var, plan.nnz
    sc_t = torch.as_tensor(np.asarray(scs, dtype=np.int64), device=j.device)
    jv = j.view(-1, nnz, PF_LANES)[sc_t // PF_LANES, :, sc_t % PF_LANES].cpu().numpy()
    gv = g.view(-1, n, PF_LANES)[sc_t // PF_LANES, :, sc_t % PF_LANES].cpu().numpy()
    jobs = [(jv[i], -gv[i], indptr, indices, n) for i in range(len(scs))]
    if len(jobs) == 1 or (os.cpu_count() or 1) == 1:
        return [_superlu.solve(a) for a in jobs]
    return list(_pool().map(_superlu.solve, jobs))


# dense device fallback: largest system and the memory one chunk of dense
# matrices may take
_DENSE_MAX_N = 16384
_DENSE_CHUNK_BYTES = 8 << 30
_DENSE_PIVOT_RATIO = 1e-13   # below: near-singular, the host's SuperLU decides


def _device_fallback(plan, j, g, scs, csr_rows, csr_cols):
    """Newton steps of the scenarios ``scs`` whose shared-pivot solve failed.

    A Jacobian with an exactly zero row or column is singular for any
    pivoting, so SuperLU raises on it as pflow's solve does: those are
    reported singular without a host factorisation.  The others are
    factorised densely on the device with partial pivoting (cuSOLVER getrf
    through ``torch.linalg.lu_factor_ex``), in chunks that fit
    ``_DENSE_CHUNK_BYTES``.  Returns (steps, singular, host): a dict
    scenario -> dy (device tensor), the scenarios found singular, and those
    left to the host (a zero pivot inside the dense factorisation, or a
    system too large to densify)."""
    import torch

    n, nnz = plan.n_var, plan.nnz
    sc_t = torch.as_tensor(np.asarray(scs, dtype=np.int64), device=j.device)
    vals = j.view(-1, nnz, PF_LANES)[sc_t // PF_LANES, :, sc_t % PF_LANES]   # [m, nnz]
    rhs = g.view(-1, n, PF_LANES)[sc_t // PF_LANES, :, sc_t % PF_LANES]      # [m, n]
    nzv = (vals != 0).to(torch.int8)
    m = len(scs)
    col_any = torch.zeros((m, n), dtype=torch.int8, device=j.device)
    row_any = torch.zeros((m, n), dtype=torch.int8, device=j.device)
    col_any.scatter_reduce_(1, csr_cols[None, :].expand(m, -1), nzv, reduce="amax")
    row_any.scatter_reduce_(1, csr_rows[None, :].expand(m, -1), nzv, reduce="amax")
    zero_line = ((col_any == 0).any(1) | (row_any == 0).any(1)).cpu().numpy()
    singular = [int(scs[i]) for i in range(m) if zero_line[i]]
    rest = [i for i in range(m) if not zero_line[i]]
    steps, host = {}, []
    if n > _DENSE_MAX_N:
        return steps, singular, [int(scs[i]) for i in rest]
    chunk = max(1, _DENSE_CHUNK_BYTES // (8 * n * n))
    prev = torch.backends.cuda.preferred_linalg_library()
    torch.backends.cuda.preferred_linalg_library("cusolver")   # getrf per matrix, not MAGMA batched
    try:
        for c0 in range(0, len(rest), chunk):
            idx = torch.as_tensor(rest[c0:c0 + chunk], device=j.device)
            mc = idx.numel()
            dense = torch.zeros((mc, n, n), dtype=torch.float64, device=j.device)
            bi = torch.arange(mc, device=j.device)[:, None]
            dense[bi, csr_rows[None, :], csr_cols[None, :]] = vals[idx]
            lu, piv, info = torch.linalg.lu_factor_ex(dense)
            dx = torch.linalg.lu_solve(lu, piv, -rhs[idx][:, :, None])[:, :, 0]
            # a pivot many orders below the largest: SuperLU (other pivots)
            # may hit an exact zero there, so the host decides
            du = lu.diagonal(dim1=1, dim2=2).abs()
            ratio = (du.amin(1) / du.amax(1)).cpu().numpy()
            info = info.cpu().numpy()
            for k in range(mc):
                sc = int(scs[rest[c0 + k]])
                if info[k] == 0 and ratio[k] > _DENSE_PIVOT_RATIO:
                    steps[sc] = dx[k]
                else:
                    host.append(sc)
            del dense, lu
    finally:
        torch.backends.cuda.preferred_linalg_library(prev)
    return steps, singular, host


@dataclass
class BatchedResult:
    converged: np.ndarray          # [K] bool
    diverged: np.ndarray           # [K] bool
    iterations: np.ndarray         # [K] updates applied
    final_mismatch: np.ndarray     # [K] max|g| at the last evaluation
    singular: np.ndarray           # [K] bool: zero pivot in the refactorisation
    timings: dict = field(default_factory=dict)


def batched_newton_solve(plan: Plan, K: int, y, pq_p=None, pq_q=None, pv_p=None, outage=None,
                         tol: float = 1e-8, max_iter: int = 20, lu: BatchedLU | None = None,
                         linear: str = "device", fallback: str = "device") -> BatchedResult:
    """Newton on K scenarios in place on the blocked state ``y`` (CUDA
    float64, plan layout).  Returns per-scenario outcomes; ``y`` holds each
    scenario's last iterate.

    ``linear="device"`` (default): one elimination schedule shared by all
    scenarios (batched_lu.py), with outage-proof pivots
    (``robust_row_match``); a singular scenario shows up as a non-finite
    mismatch and is reported diverged.  ``linear="cusolverrf"``: one
    cusolverRf handle per scenario, each with its own pivoting.

    A scenario whose shared-pivot solve fails its accuracy check is solved
    with its own pivoting: ``fallback="device"`` (default) factorises it
    densely on the device (``_device_fallback``; an exactly zero row or
    column is reported singular, as pflow's SuperLU solve raises on it), and
    only a zero pivot inside that factorisation goes to SuperLU on the host;
    ``fallback="host"`` sends every such scenario to SuperLU."""
    import torch

    if tol <= 0 or max_iter < 1:
        raise ValueError("tol must be positive and max_iter >= 1")
    lib = _abi.lib()
    dev = y.device
    n, nnz = plan.n_var, plan.nnz
    g = plan.empty(n, K)
    j = plan.empty(nnz, K)
    norms = plan.empty(K)
    active = torch.ones(K, dtype=torch.int32, device=dev)
    timings = {"eval": 0.0, "handoff": 0.0, "lu": 0.0, "update": 0.0, "setup": 0.0}
    if linear not in ("device", "cusolverrf"):
        raise ValueError("linear must be 'device' or 'cusolverrf'")
    if fallback not in ("device", "host"):
        raise ValueError("fallback must be 'device' or 'host'")
    dlu = None
    if linear == "device" and lu is None:
        # one schedule for every scenario: pivoting from scenario 0 at the
        # initial state without its outage (an outage can island buses)
        from .batched_lu import DeviceSparseLU, analyze

        t0 = time.perf_counter()
        indptr, indices = plan.pattern_csr()
        plan.eval_batched(K, y, pq_p, pq_q, pv_p, None, None, j, None)
        j0 = torch.empty(nnz, dtype=torch.float64, device=dev)
        _abi.check(lib.pf_batch_unblock(1, nnz, j.data_ptr(), j0.data_ptr(), 1.0, None))
        base = sp.csr_matrix((j0.cpu().numpy(), indices, indptr), shape=(n, n))
        L, U, P, Q = base_lu(base.tocsc(), n_bus=plan.n_bus)
        dlu = DeviceSparseLU(analyze(indptr, indices, L, U, P, Q), K, device=dev)
        indptr_h, indices_h = indptr, indices
        csr_ptr = torch.as_tensor(indptr, dtype=torch.int32, device=dev)
        csr_idx = torch.as_tensor(indices, dtype=torch.int32, device=dev)
        csr_idx_l = csr_idx.to(torch.int64)
        csr_row = torch.repeat_interleave(torch.arange(n, device=dev),
                                          torch.as_tensor(np.diff(indptr), device=dev))
        res = plan.empty(K)
        torch.cuda.synchronize(dev)
        timings["setup"] = time.perf_counter() - t0
    elif lu is None:   # pivoting and factor pattern of each scenario at its initial state
        t0 = time.perf_counter()
        indptr, indices = plan.pattern_csr()
        plan.eval_batched(K, y, pq_p, pq_q, pv_p, outage, None, j, None)
        base = torch.empty((K, nnz), dtype=torch.float64, device=dev)
        _abi.check(lib.pf_batch_unblock(K, nnz, j.data_ptr(), base.data_ptr(), 1.0, None))
        lu = BatchedLU(K, indptr, indices, base.cpu().numpy(), device=dev)
        del base
        torch.cuda.synchronize(dev)
        timings["setup"] = time.perf_counter() - t0
    conv = np.zeros(K, dtype=bool)
    div = np.zeros(K, dtype=bool)
    singular = np.zeros(K, dtype=bool)
    host_solves = device_fallback = zero_line_singular = 0
    host_only = np.zeros(K, dtype=bool)
    iters = np.zeros(K, dtype=np.int64)
    mism = np.full(K, np.inf)
    stream = torch.cuda.current_stream(dev).cuda_stream
    for it in range(max_iter + 1):
        t0 = time.perf_counter()
        plan.eval_batched(K, y, pq_p, pq_q, pv_p, outage, g, j, norms)
        nh = norms[:K].cpu().numpy()           # the one host read per iteration
        timings["eval"] += time.perf_counter() - t0
        live = ~(conv | div | singular)
        mism[live] = nh[live]
        newly_div = live & (~np.isfinite(nh) | (nh > _DIVERGENCE_LIMIT))
        div |= newly_div
        conv |= live & ~newly_div & (nh <= tol)
        live = ~(conv | div | singular)
        if not live.any() or it == max_iter:
            break
        if dlu is not None:   # refactor all scenarios together, update the live ones
            t0 = time.perf_counter()
            dlu.factor(j)
            dx = dlu.solve(g)
            # accuracy check of every solve: the shared pivot order can fail for
            # a scenario whose outage makes a pivot vanish after elimination;
            # those few are solved on the host with their own pivoting
            _abi.check(lib.pf_lu_residual(K, n, nnz, csr_ptr.data_ptr(), csr_idx.data_ptr(),
                                          j.data_ptr(), dx.data_ptr(), g.data_ptr(),
                                          res.data_ptr(), stream))
            rh = res[:K].cpu().numpy()
            timings["lu"] += time.perf_counter() - t0
            t0 = time.perf_counter()
            ok = live & np.isfinite(rh) & (rh <= _LIN_RTOL * np.maximum(nh, 1e-300))
            active.copy_(torch.as_tensor(ok.astype(np.int32)))
            dlu.add(dx, y, active)
            failed = np.nonzero(live & ~ok)[0]
            yv = y.view(-1, n, PF_LANES)
            # a scenario that was near-singular once goes straight to the host
            host_list = [int(sc) for sc in failed if host_only[sc]]
            dev_try = np.array([sc for sc in failed if not host_only[sc]], dtype=np.int64)
            if dev_try.size and fallback == "device":
                steps, sing, more = _device_fallback(plan, j, g, dev_try, csr_row, csr_idx_l)
                for sc in sing:             # exactly singular: pflow's solve raises here
                    singular[sc] = True
                    live[sc] = False
                for sc, dy in steps.items():
                    yv[sc // PF_LANES, :, sc % PF_LANES] += dy
                host_only[more] = True
                host_list += more
                device_fallback += len(steps)
                zero_line_singular += len(sing)
            else:
                host_list += [int(sc) for sc in dev_try]
            if host_list:
                for sc, dy in zip(host_list, _host_solves(plan, j, g, host_list, indptr_h,
                                                          indices_h)):
                    if dy is None:          # singular: pflow's solve raises here
                        singular[sc] = True
                        live[sc] = False
                        continue
                    yv[sc // PF_LANES, :, sc % PF_LANES] += torch.as_tensor(dy, device=dev)
                    host_solves += 1
            iters[live] += 1
            torch.cuda.synchronize(dev)
            timings["update"] += time.perf_counter() - t0
            continue
        t0 = time.perf_counter()
        _abi.check(lib.pf_batch_unblock(K, nnz, j.data_ptr(), lu.vals.data_ptr(), 1.0, stream))
        _abi.check(lib.pf_batch_unblock(K, n, g.data_ptr(), lu.rhs.data_ptr(), -1.0, stream))
        active.copy_(torch.as_tensor(live.astype(np.int32)), non_blocking=False)
        torch.cuda.synchronize(dev)
        timings["handoff"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        sing = lu.refactor_solve(np.nonzero(live)[0])
        timings["lu"] += time.perf_counter() - t0
        if sing.size:   # singular Jacobian: pflow's solve raises; the scenario stops here
            singular[sing] = True
            live[sing] = False
            active.copy_(torch.as_tensor(live.astype(np.int32)))
        t0 = time.perf_counter()
        _abi.check(lib.pf_batch_update(K, n, y.data_ptr(), lu.rhs.data_ptr(),
                                       active.data_ptr(), stream))
        iters[live] += 1
        timings["update"] += time.perf_counter() - t0
    torch.cuda.synchronize(dev)
    timings["host_fallback_solves"] = host_solves
    timings["device_fallback_solves"] = device_fallback
    timings["zero_line_singular"] = zero_line_singular
    return BatchedResult(converged=conv, diverged=div, iterations=iters, final_mismatch=mism,
                         singular=singular, timings=timings)
