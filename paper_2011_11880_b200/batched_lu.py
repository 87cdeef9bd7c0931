"""Batched sparse LU refactorisation on a fixed pattern, scenarios in lanes
(the hand-off after the product path).

All K scenarios share one sparsity pattern, one pivot order and one
elimination schedule, and differ only in values. That is the blocked layout
of the evaluation kernels (lanes = 32 scenarios of one block). One warp can
therefore eliminate a row for 32 scenarios at once with coalesced 256-byte
accesses, and the schedule is warp-uniform. This replaces cusolverRf, whose
batched entry points crash on this stack (batched_newton.py).

Structure of A = J (CSR pattern of the plan), P A Q^T = L U:
  * pivot order and closed fill pattern from ``batched_newton.base_lu``
    (SuperLU on a base matrix, then a symbolic pass without cancellation);
  * rows [0, n - D): sparse rows, eliminated row by row in dependency levels
    (row i needs every row k with L[i, k] != 0). Each update is a
    multiply-add m_ij -= l_ik u_kj on precomputed positions;
  * rows [n - D, n): first the same updates from the sparse rows k < n - D
    (the border). That leaves the D x D trailing Schur complement, which is
    nearly dense for these grids. It is then factorised as a dense batch
    with partial pivoting inside the block (``torch.linalg.lu_factor``,
    cuSOLVER).

The solve runs forward over the sparse levels and the border, through the
dense tail (two triangular solves), and backward over the sparse levels in
reverse.

This module holds the symbolic analysis (host, numpy) and a numpy reference of
the numeric phases (``reference_factor_solve``), which the tests use to pin
the device kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


@dataclass
class LUSchedule:
    n: int
    D: int                    # dense tail size
    P: np.ndarray             # row order: M[i, :] = A[P[i], Q[:]]
    Q: np.ndarray
    # M = L + U - I pattern (CSR, sorted), diagonal position of every row
    m_ptr: np.ndarray
    m_idx: np.ndarray
    m_diag: np.ndarray
    a2m: np.ndarray           # A entry (CSR order) -> M position
    # elimination records of sparse + border rows, grouped by row:
    # rec[r] = (pos_ik, pos_kk, upd_begin, upd_end), upd pairs = (pos_kj, pos_ij)
    row_list: np.ndarray      # rows in processing order (sparse rows by level, then tail rows)
    row_rec_ptr: np.ndarray   # [len(row_list)+1] into rec
    rec: np.ndarray           # [n_rec, 4] int32
    upd: np.ndarray           # [n_upd, 2] int32
    level_ptr: np.ndarray     # sparse levels: row_list[level_ptr[l]:level_ptr[l+1]]
    n_sparse_rows: int        # rows in row_list before the tail rows
    bwd_rows: np.ndarray      # sparse rows grouped by backward level (U dependencies)
    bwd_ptr: np.ndarray
    # dense tail: M positions of the D x D block (-1 = structurally zero)
    tail_pos: np.ndarray      # [D, D] int32


def choose_tail(m_ptr, m_idx, n, min_density=0.3, max_d=1536):
    """Largest trailing block (<= max_d) with density >= min_density: the
    block of size d holds the entries with min(row, col) >= n - d."""
    rows = np.repeat(np.arange(n), np.diff(m_ptr))
    lo = np.minimum(rows, m_idx)
    # nnz(d) = #{entries with lo >= n - d}, d = 1..n
    cnt = np.bincount(n - 1 - lo, minlength=n).cumsum()
    d = np.arange(1, n + 1)
    ok = (cnt >= min_density * d.astype(np.float64) ** 2) & (d <= max_d)
    return int(d[ok].max()) if ok.any() else 0


def analyze(indptr, indices, L: sp.csr_matrix, U: sp.csr_matrix, P, Q, D: int | None = None,
            min_density: float = 0.3) -> LUSchedule:
    n = int(indptr.shape[0] - 1)
    M = (sp.csr_matrix(L) + sp.csr_matrix(U)).tocsr()
    M.sort_indices()
    m_ptr = M.indptr.astype(np.int64)
    m_idx = M.indices.astype(np.int32)
    m_diag = np.searchsorted(np.repeat(np.arange(n, dtype=np.int64), np.diff(m_ptr)) * n
                             + m_idx, np.arange(n, dtype=np.int64) * (n + 1))
    if not np.array_equal(m_idx[np.minimum(m_diag, m_idx.size - 1)], np.arange(n)):
        raise AssertionError("missing diagonal")
    Pinv = np.empty(n, np.int64)
    Pinv[P] = np.arange(n)
    Qinv = np.empty(n, np.int64)
    Qinv[Q] = np.arange(n)
    # A entry (r, c) -> M entry (Pinv[r], Qinv[c])
    a_rows = np.repeat(np.arange(n), np.diff(indptr))
    mi, mj = Pinv[a_rows], Qinv[indices]
    m_rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(m_ptr))
    m_keys = m_rows * n + m_idx                  # sorted: CSR with sorted columns
    a_keys = mi * n + mj
    a2m = np.searchsorted(m_keys, a_keys)
    if not (a2m < m_keys.size).all() or not np.array_equal(m_keys[np.minimum(a2m, m_keys.size - 1)],
                                                           a_keys):
        raise AssertionError("A entry outside the factor pattern")
    if D is None:
        D = choose_tail(m_ptr, m_idx, n, min_density)
    t0 = n - D
    # elimination records
    level = np.zeros(n, np.int64)
    recs, upds, rec_ptr_rows = [], [], {}
    for i in range(n):
        row = m_idx[m_ptr[i]:m_ptr[i + 1]]
        pos_of = {int(c): int(m_ptr[i] + q) for q, c in enumerate(row)}
        ks = row[row < min(i, t0)]            # sparse / border multipliers only
        lv = 0
        start = len(recs)
        for k in ks:
            k = int(k)
            lv = max(lv, int(level[k]) + 1)
            urow = m_idx[m_diag[k] + 1:m_ptr[k + 1]]
            b = len(upds)
            for q, j in enumerate(urow):
                upds.append((int(m_diag[k] + 1 + q), pos_of[int(j)]))
            recs.append((pos_of[k], int(m_diag[k]), b, len(upds)))
        rec_ptr_rows[i] = (start, len(recs))
        level[i] = lv if i < t0 else 0
    sparse_rows = np.arange(t0)
    order = sparse_rows[np.argsort(level[:t0], kind="stable")]
    lv_sorted = level[order]
    n_lv = int(lv_sorted.max()) + 1 if t0 else 0
    level_ptr = np.searchsorted(lv_sorted, np.arange(n_lv + 1))
    row_list = np.concatenate([order, np.arange(t0, n)]).astype(np.int32)
    rec_arr = np.zeros((max(len(recs), 1), 4), np.int32)
    if recs:
        rec_arr[: len(recs)] = np.asarray(recs, np.int64)
    # records reordered to follow row_list
    new_rec, new_ptr = [], [0]
    for i in row_list:
        a, b = rec_ptr_rows[int(i)]
        new_rec.extend(recs[a:b])
        new_ptr.append(len(new_rec))
    rec_arr = np.asarray(new_rec, np.int64).reshape(-1, 4).astype(np.int32) if new_rec else \
        np.zeros((0, 4), np.int32)
    upd_arr = np.asarray(upds, np.int64).reshape(-1, 2).astype(np.int32) if upds else \
        np.zeros((0, 2), np.int32)
    # backward levels over the sparse rows: row i needs x_j for j in U(i)
    blev = np.zeros(t0, np.int64)
    for i in range(t0 - 1, -1, -1):
        cols = m_idx[m_diag[i] + 1:m_ptr[i + 1]]
        cols = cols[cols < t0]
        blev[i] = 1 + int(blev[cols].max()) if cols.size else 0
    border = np.argsort(blev, kind="stable")
    bl_sorted = blev[border]
    n_bl = int(bl_sorted.max()) + 1 if t0 else 0
    bwd_ptr = np.searchsorted(bl_sorted, np.arange(n_bl + 1))
    tail_pos = np.full((D, D), -1, np.int32)
    for i in range(t0, n):
        row = m_idx[m_ptr[i]:m_ptr[i + 1]]
        sel = row >= t0
        tail_pos[i - t0, row[sel] - t0] = (m_ptr[i] + np.nonzero(sel)[0]).astype(np.int32)
    return LUSchedule(n=n, D=D, P=np.asarray(P, np.int32), Q=np.asarray(Q, np.int32),
                      m_ptr=m_ptr.astype(np.int32), m_idx=m_idx, m_diag=m_diag.astype(np.int32),
                      a2m=a2m.astype(np.int32), row_list=row_list,
                      row_rec_ptr=np.asarray(new_ptr, np.int32), rec=rec_arr, upd=upd_arr,
                      level_ptr=level_ptr.astype(np.int32), n_sparse_rows=int(t0),
                      bwd_rows=border.astype(np.int32), bwd_ptr=bwd_ptr.astype(np.int32),
                      tail_pos=tail_pos)


def reference_factor_solve(s: LUSchedule, a_vals: np.ndarray, b: np.ndarray) -> np.ndarray:
    """numpy restatement of the device phases for one scenario: returns x
    with A x = b (A in the plan's CSR order)."""
    n, D, t0 = s.n, s.D, s.n - s.D
    m = np.zeros(s.m_idx.shape[0])
    m[s.a2m] = a_vals
    # sparse rows (levels) and border updates of the tail rows
    for r, i in enumerate(s.row_list):
        for pos_ik, pos_kk, u0, u1 in s.rec[s.row_rec_ptr[r]:s.row_rec_ptr[r + 1]]:
            l = m[pos_ik] / m[pos_kk]
            m[pos_ik] = l
            for pkj, pij in s.upd[u0:u1]:
                m[pij] -= l * m[pkj]
    # dense tail: LU of the Schur complement (unpivoted here; the device path
    # pivots within the block, which gives the same solution)
    T = np.where(s.tail_pos >= 0, m[np.maximum(s.tail_pos, 0)], 0.0)
    for k in range(D):
        T[k + 1:, k] /= T[k, k]
        T[k + 1:, k + 1:] -= np.outer(T[k + 1:, k], T[k, k + 1:])
    # solve: M = P A Q^T, so A x = b <=> M (Q x) = P b
    y = b[s.P].astype(np.float64).copy()
    m_rows = [(s.m_idx[s.m_ptr[i]:s.m_ptr[i + 1]], np.arange(s.m_ptr[i], s.m_ptr[i + 1]))
              for i in range(n)]
    for i in s.row_list:                        # forward: sparse rows and border
        cols, pos = m_rows[i]
        sel = cols < min(i, t0)
        y[i] -= np.dot(m[pos[sel]], y[cols[sel]])
    for k in range(D):                          # dense unit-lower forward
        y[t0 + k + 1:] -= T[k + 1:, k] * y[t0 + k]
    for k in range(D - 1, -1, -1):              # dense upper backward
        y[t0 + k] /= T[k, k]
        y[t0:t0 + k] -= T[:k, k] * y[t0 + k]
    for i in s.bwd_rows:                        # backward over sparse rows, by level
        cols, pos = m_rows[i]
        sel = cols > i
        y[i] = (y[i] - np.dot(m[pos[sel]], y[cols[sel]])) / m[s.m_diag[i]]
    x = np.empty(n)
    x[s.Q] = y
    return x


class DeviceSparseLU:
    """K systems sharing one ``LUSchedule``: refactor on the device from the
    blocked CSR values of J, then solve J dx = -g and add dx to the state for
    the scenarios still active (libpfgpu pf_lu_* kernels + cuSOLVER for the
    dense tail through torch)."""

    def __init__(self, sched: LUSchedule, K: int, device="cuda"):
        import torch

        from . import _abi

        self.s, self.K = sched, int(K)
        self._lib, self._check = _abi.lib(), _abi.check
        t = lambda a, dt=torch.int32: torch.as_tensor(np.ascontiguousarray(a), dtype=dt,
                                                     device=device)
        self.a2m, self.rec, self.upd = t(sched.a2m), t(sched.rec), t(sched.upd)
        self.rec_ptr, self.rows = t(sched.row_rec_ptr), t(sched.row_list)
        self.bwd = t(sched.bwd_rows)
        self.m_ptr, self.m_idx, self.m_diag = t(sched.m_ptr), t(sched.m_idx), t(sched.m_diag)
        self.tail_pos, self.P, self.Q = t(sched.tail_pos), t(sched.P), t(sched.Q)
        self.nnz_m = int(sched.m_idx.shape[0])
        nb = -(-self.K // 32)
        f64 = dict(dtype=torch.float64, device=device)
        self.M = torch.empty(nb * self.nnz_m * 32, **f64)
        self.Y = torch.empty(nb * sched.n * 32, **f64)
        self.T = torch.empty((self.K, sched.D, sched.D), **f64)
        self.DX = torch.empty(nb * sched.n * 32, **f64)
        self.iota = torch.arange(sched.n, dtype=torch.int32, device=device)
        self.V = torch.empty((self.K, sched.D), **f64)
        self.LU = self.piv = None

    def _p(self, x, off=0):
        return x.data_ptr() + off * x.element_size()

    def factor(self, j_blocked, stream=None) -> None:
        import torch

        s, lib, ck, K = self.s, self._lib, self._check, self.K
        stream = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        ck(lib.pf_lu_scatter(K, int(s.a2m.shape[0]), self.nnz_m, self._p(self.a2m),
                             j_blocked.data_ptr(), self._p(self.M), stream))
        lp = s.level_ptr
        for lv in range(len(lp) - 1):
            ck(lib.pf_lu_eliminate(K, self.nnz_m, int(lp[lv + 1] - lp[lv]),
                                   self._p(self.rec_ptr, int(lp[lv])), self._p(self.rec),
                                   self._p(self.upd), self._p(self.M), stream))
        ck(lib.pf_lu_eliminate(K, self.nnz_m, s.D, self._p(self.rec_ptr, s.n_sparse_rows),
                               self._p(self.rec), self._p(self.upd), self._p(self.M), stream))
        if s.D:
            ck(lib.pf_lu_tail_gather(K, self.nnz_m, s.D, self._p(self.tail_pos), self._p(self.M),
                                     self._p(self.T), stream))
            # partial pivoting inside the dense tail (rows of the Schur
            # complement only: the sparse rows and the columns are unaffected)
            # (_ex: no host-side singularity check; a singular scenario turns
            # into a non-finite update and is reported by the Newton driver)
            self.LU, self.piv, _ = torch.linalg.lu_factor_ex(self.T)

    def solve(self, g_blocked, stream=None):
        """dx = -J^{-1} g for every scenario; returns the blocked dx (plan
        variable order)."""
        import torch

        s, lib, ck, K = self.s, self._lib, self._check, self.K
        stream = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        t0 = s.n - s.D
        ck(lib.pf_lu_rhs(K, s.n, self._p(self.P), g_blocked.data_ptr(), self._p(self.Y), -1.0,
                         stream))
        lp = s.level_ptr
        for lv in range(len(lp) - 1):
            ck(lib.pf_lu_forward(K, s.n, self.nnz_m, int(lp[lv + 1] - lp[lv]),
                                 self._p(self.rows, int(lp[lv])), self._p(self.m_ptr),
                                 self._p(self.m_idx), t0, self._p(self.M), self._p(self.Y), stream))
        ck(lib.pf_lu_forward(K, s.n, self.nnz_m, s.D, self._p(self.rows, s.n_sparse_rows),
                             self._p(self.m_ptr), self._p(self.m_idx), t0, self._p(self.M),
                             self._p(self.Y), stream))
        if s.D:
            ck(lib.pf_lu_tail_vec(K, s.n, t0, s.D, self._p(self.Y), self._p(self.V), 1, stream))
            self.V.copy_(torch.linalg.lu_solve(self.LU, self.piv, self.V.unsqueeze(-1)).squeeze(-1))
            ck(lib.pf_lu_tail_vec(K, s.n, t0, s.D, self._p(self.Y), self._p(self.V), 0, stream))
        bp = s.bwd_ptr
        for lv in range(len(bp) - 1):
            ck(lib.pf_lu_backward(K, s.n, self.nnz_m, int(bp[lv + 1] - bp[lv]),
                                  self._p(self.bwd, int(bp[lv])), self._p(self.m_ptr),
                                  self._p(self.m_diag), self._p(self.m_idx), self._p(self.M),
                                  self._p(self.Y), stream))
        self.DX.zero_()
        ck(lib.pf_lu_apply(K, s.n, self._p(self.Q), self._p(self.Y), self._p(self.DX), None,
                           stream))
        return self.DX

    def add(self, dx_blocked, state_blocked, active=None, stream=None) -> None:
        """state += dx for the active scenarios (both blocked, plan order)."""
        import torch

        stream = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        self._check(self._lib.pf_lu_apply(self.K, self.s.n, self._p(self.iota),
                                          dx_blocked.data_ptr(), state_blocked.data_ptr(),
                                          active.data_ptr() if active is not None else None,
                                          stream))

    def solve_update(self, g_blocked, state_blocked, active=None, stream=None) -> None:
        """state += J^{-1} (-g) for the active scenarios (blocked vectors)."""
        self.add(self.solve(g_blocked, stream), state_blocked, active, stream)
