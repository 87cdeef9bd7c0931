// pf_lu.cu - batched sparse LU refactorisation and solve on a fixed schedule
// (the hand-off after the product path).
//
// All K scenarios share one pattern, one pivot order and one elimination
// schedule (paper_2011_11880_b200/batched_lu.py builds it on the host), so the
// factor values live in the blocked scenario layout of the evaluation kernels:
// value q of scenario s at ((s / 32) * nnz + q) * 32 + s % 32.  One warp works
// on one matrix row for the 32 scenarios of a block: every schedule read is
// warp-uniform and every value access one coalesced 256-byte transaction.
// The sparse rows run level by level (one launch per level); the dense
// trailing Schur complement is handed to cuSOLVER through torch.
#include <cuda_runtime.h>

#include "pf_internal.cuh"

namespace pf {
namespace {

constexpr int LU_WARPS = 8;

inline unsigned cdiv(int64_t n, int64_t d) { return (unsigned)((n + d - 1) / d); }

// A (plan CSR order) -> M positions; fill positions start at zero.
__global__ void k_lu_scatter(int32_t nnz_a, int32_t nnz_m, const int32_t* __restrict__ a2m,
                             const double* __restrict__ a, double* __restrict__ m) {
    const int lane = threadIdx.x & 31;
    const int64_t blk = blockIdx.y;
    const int32_t e = blockIdx.x * LU_WARPS + (threadIdx.x >> 5);
    if (e >= nnz_a) return;
    m[(blk * nnz_m + __ldg(a2m + e)) * PF_LANES + lane] = a[(blk * nnz_a + e) * PF_LANES + lane];
}

// Row-oriented elimination of the rows listed (one warp each): for every
// multiplier record {pos_ik, pos_kk, u0, u1} in order, l = m_ik / u_kk and
// m_ij -= l u_kj over the update pairs {pos_kj, pos_ij}.
__global__ void k_lu_eliminate(int32_t n_rows, int32_t nnz_m, const int32_t* __restrict__ rec_ptr,
                               const int4* __restrict__ rec, const int2* __restrict__ upd,
                               double* __restrict__ m) {
    const int lane = threadIdx.x & 31;
    const int32_t r = blockIdx.x * LU_WARPS + (threadIdx.x >> 5);
    if (r >= n_rows) return;
    double* mb = m + (int64_t)blockIdx.y * nnz_m * PF_LANES + lane;
    const int32_t q1 = __ldg(rec_ptr + r + 1);
    for (int32_t q = __ldg(rec_ptr + r); q < q1; ++q) {
        const int4 rc = __ldg(rec + q);
        const double l = mb[(int64_t)rc.x * PF_LANES] / mb[(int64_t)rc.y * PF_LANES];
        mb[(int64_t)rc.x * PF_LANES] = l;
        for (int32_t p = rc.z; p < rc.w; ++p) {
            const int2 u = __ldg(upd + p);
            mb[(int64_t)u.y * PF_LANES] -= l * mb[(int64_t)u.x * PF_LANES];
        }
    }
}

// Dense trailing block, blocked -> scenario-major [K][D][D] through a 32 x 33
// tile (columns c0..c0+31 of row r for the 32 scenarios of block blockIdx.z).
__global__ void k_lu_tail_gather(int32_t K, int32_t nnz_m, int32_t D,
                                 const int32_t* __restrict__ tail_pos,
                                 const double* __restrict__ m, double* __restrict__ t) {
    __shared__ double tile[32][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int32_t r = blockIdx.y, c0 = blockIdx.x * 32;
    const int64_t blk = blockIdx.z;
    for (int c = w; c < 32; c += LU_WARPS) {
        const int32_t cc = c0 + c;
        const int32_t pos = cc < D ? __ldg(tail_pos + (int64_t)r * D + cc) : -1;
        tile[c][lane] = pos >= 0 ? m[(blk * nnz_m + pos) * PF_LANES + lane] : 0.0;
    }
    __syncthreads();
    for (int sl = w; sl < 32; sl += LU_WARPS) {
        const int64_t s = blk * PF_LANES + sl;
        const int32_t cc = c0 + lane;
        if (s < K && cc < D) t[(s * D + r) * D + cc] = tile[lane][sl];
    }
}

// y(i) = alpha * g(P[i]) (blocked vectors)
__global__ void k_lu_rhs(int32_t n, const int32_t* __restrict__ P, const double* __restrict__ g,
                         double* __restrict__ y, double alpha) {
    const int lane = threadIdx.x & 31;
    const int32_t i = blockIdx.x * LU_WARPS + (threadIdx.x >> 5);
    if (i >= n) return;
    const int64_t b = (int64_t)blockIdx.y * n;
    y[(b + i) * PF_LANES + lane] = alpha * g[(b + __ldg(P + i)) * PF_LANES + lane];
}

// forward substitution of the rows listed: y_i -= sum m_ik y_k over the
// L entries with k < min(i, col_end), in column order
__global__ void k_lu_forward(int32_t n_rows, const int32_t* __restrict__ rows, int32_t n,
                             int32_t nnz_m, const int32_t* __restrict__ m_ptr,
                             const int32_t* __restrict__ m_idx, int32_t col_end,
                             const double* __restrict__ m, double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int32_t r = blockIdx.x * LU_WARPS + (threadIdx.x >> 5);
    if (r >= n_rows) return;
    const int32_t i = __ldg(rows + r), lim = min(i, col_end);
    const double* mb = m + (int64_t)blockIdx.y * nnz_m * PF_LANES + lane;
    double* yb = y + (int64_t)blockIdx.y * n * PF_LANES + lane;
    double acc = yb[(int64_t)i * PF_LANES];
    const int32_t q1 = __ldg(m_ptr + i + 1);
    for (int32_t q = __ldg(m_ptr + i); q < q1; ++q) {
        const int32_t k = __ldg(m_idx + q);
        if (k >= lim) break;
        acc -= mb[(int64_t)q * PF_LANES] * yb[(int64_t)k * PF_LANES];
    }
    yb[(int64_t)i * PF_LANES] = acc;
}

// backward substitution of the rows listed: y_i = (y_i - sum_{j > i} m_ij y_j) / m_ii
__global__ void k_lu_backward(int32_t n_rows, const int32_t* __restrict__ rows, int32_t n,
                              int32_t nnz_m, const int32_t* __restrict__ m_ptr,
                              const int32_t* __restrict__ m_diag, const int32_t* __restrict__ m_idx,
                              const double* __restrict__ m, double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int32_t r = blockIdx.x * LU_WARPS + (threadIdx.x >> 5);
    if (r >= n_rows) return;
    const int32_t i = __ldg(rows + r);
    const double* mb = m + (int64_t)blockIdx.y * nnz_m * PF_LANES + lane;
    double* yb = y + (int64_t)blockIdx.y * n * PF_LANES + lane;
    double acc = yb[(int64_t)i * PF_LANES];
    const int32_t dq = __ldg(m_diag + i), q1 = __ldg(m_ptr + i + 1);
    for (int32_t q = dq + 1; q < q1; ++q)
        acc -= mb[(int64_t)q * PF_LANES] * yb[(int64_t)__ldg(m_idx + q) * PF_LANES];
    yb[(int64_t)i * PF_LANES] = acc / mb[(int64_t)dq * PF_LANES];
}

// entries [t0, t0 + D) of blocked y <-> scenario-major v[K][D]
__global__ void k_lu_tail_vec(int32_t K, int32_t n, int32_t t0, int32_t D, double* __restrict__ y,
                              double* __restrict__ v, int to_dense) {
    __shared__ double tile[32][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int32_t d0 = blockIdx.x * 32;
    const int64_t blk = blockIdx.y;
    double* yb = y + (blk * n + t0) * PF_LANES;
    if (to_dense) {
        for (int d = w; d < 32; d += LU_WARPS)
            tile[d][lane] = d0 + d < D ? yb[(int64_t)(d0 + d) * PF_LANES + lane] : 0.0;
        __syncthreads();
        for (int sl = w; sl < 32; sl += LU_WARPS) {
            const int64_t s = blk * PF_LANES + sl;
            if (s < K && d0 + lane < D) v[s * D + d0 + lane] = tile[lane][sl];
        }
    } else {
        for (int sl = w; sl < 32; sl += LU_WARPS) {
            const int64_t s = blk * PF_LANES + sl;
            tile[sl][lane] = (s < K && d0 + lane < D) ? v[s * D + d0 + lane] : 0.0;
        }
        __syncthreads();
        for (int d = w; d < 32; d += LU_WARPS)
            if (d0 + d < D) yb[(int64_t)(d0 + d) * PF_LANES + lane] = tile[lane][d];
    }
}

// state(Q[j]) += x(j) for the active scenarios (blocked vectors)
__global__ void k_lu_apply(int32_t K, int32_t n, const int32_t* __restrict__ Q,
                           const double* __restrict__ x, double* __restrict__ state,
                           const int32_t* __restrict__ active) {
    const int lane = threadIdx.x & 31;
    const int32_t j = blockIdx.x * LU_WARPS + (threadIdx.x >> 5);
    if (j >= n) return;
    const int64_t s = (int64_t)blockIdx.y * PF_LANES + lane;
    if (s >= K || (active && !__ldg(active + s))) return;
    const int64_t b = (int64_t)blockIdx.y * n;
    state[(b + __ldg(Q + j)) * PF_LANES + lane] += x[(b + j) * PF_LANES + lane];
}

// max_i |g_i + sum_j J_ij x_j| per scenario (residual of the linear solve),
// as the integer max of |r| bit patterns (NaN-propagating) into out[K]
__global__ void k_lu_residual(int32_t K, int32_t n, int32_t nnz, const int32_t* __restrict__ ptr,
                              const int32_t* __restrict__ idx, const double* __restrict__ jv,
                              const double* __restrict__ x, const double* __restrict__ g,
                              unsigned long long* __restrict__ out) {
    __shared__ unsigned long long red[LU_WARPS][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int32_t i = blockIdx.x * LU_WARPS + w;
    const int64_t b = blockIdx.y;
    unsigned long long v = 0;
    if (i < n) {
        const double* jb = jv + b * nnz * PF_LANES + lane;
        const double* xb = x + b * n * PF_LANES + lane;
        double r = g[(b * n + i) * PF_LANES + lane];
        const int32_t q1 = __ldg(ptr + i + 1);
        for (int32_t q = __ldg(ptr + i); q < q1; ++q)
            r += jb[(int64_t)q * PF_LANES] * xb[(int64_t)__ldg(idx + q) * PF_LANES];
        v = static_cast<unsigned long long>(__double_as_longlong(fabs(r)));
    }
    red[w][lane] = v;
    __syncthreads();
    if (w == 0) {
        for (int k = 1; k < LU_WARPS; ++k) v = max(v, red[k][lane]);
        const int64_t s = b * PF_LANES + lane;
        if (s < K && v) atomicMax(out + s, v);
    }
}

}  // namespace
}  // namespace pf

// ================================ C ABI =====================================

#define LU_CHECK()                                               \
    do {                                                         \
        pf::count_launch();                                      \
        cudaError_t e_ = cudaGetLastError();                     \
        if (e_ != cudaSuccess) return pf::cuda_fail(e_, "launch"); \
    } while (0)

static int lu_invalid(const char* msg) {
    pf::set_error(msg);
    return PF_EINVAL;
}

extern "C" {

int pf_lu_scatter(int32_t K, int32_t nnz_a, int32_t nnz_m, const int32_t* a2m, const double* a,
                  double* m, void* stream) {
    if (K <= 0 || nnz_a < 0 || nnz_m < nnz_a) return lu_invalid("bad sizes");
    if (!a2m || !a || !m) return lu_invalid("NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned nb = pf::cdiv(K, PF_LANES);
    PF_CUDA(cudaMemsetAsync(m, 0, sizeof(double) * (size_t)nnz_m * PF_LANES * nb, st));
    if (nnz_a == 0) return PF_OK;
    pf::k_lu_scatter<<<dim3(pf::cdiv(nnz_a, pf::LU_WARPS), nb), 32 * pf::LU_WARPS, 0, st>>>(
        nnz_a, nnz_m, a2m, a, m);
    LU_CHECK();
    return PF_OK;
}

int pf_lu_eliminate(int32_t K, int32_t nnz_m, int32_t n_rows, const int32_t* rec_ptr,
                    const int32_t* rec, const int32_t* upd, double* m, void* stream) {
    if (K <= 0 || n_rows < 0 || nnz_m < 0) return lu_invalid("bad sizes");
    if (n_rows == 0) return PF_OK;
    if (!rec_ptr || !m) return lu_invalid("NULL argument");
    pf::k_lu_eliminate<<<dim3(pf::cdiv(n_rows, pf::LU_WARPS), pf::cdiv(K, PF_LANES)),
                         32 * pf::LU_WARPS, 0, (cudaStream_t)stream>>>(
        n_rows, nnz_m, rec_ptr, reinterpret_cast<const int4*>(rec),
        reinterpret_cast<const int2*>(upd), m);
    LU_CHECK();
    return PF_OK;
}

int pf_lu_tail_gather(int32_t K, int32_t nnz_m, int32_t D, const int32_t* tail_pos,
                      const double* m, double* t, void* stream) {
    if (K <= 0 || D < 0) return lu_invalid("bad sizes");
    if (D == 0) return PF_OK;
    if (!tail_pos || !m || !t) return lu_invalid("NULL argument");
    pf::k_lu_tail_gather<<<dim3(pf::cdiv(D, 32), D, pf::cdiv(K, PF_LANES)), 32 * pf::LU_WARPS, 0,
                           (cudaStream_t)stream>>>(K, nnz_m, D, tail_pos, m, t);
    LU_CHECK();
    return PF_OK;
}

int pf_lu_rhs(int32_t K, int32_t n, const int32_t* P, const double* g, double* y, double alpha,
              void* stream) {
    if (K <= 0 || n < 0) return lu_invalid("bad sizes");
    if (n == 0) return PF_OK;
    if (!P || !g || !y) return lu_invalid("NULL argument");
    pf::k_lu_rhs<<<dim3(pf::cdiv(n, pf::LU_WARPS), pf::cdiv(K, PF_LANES)), 32 * pf::LU_WARPS, 0,
                   (cudaStream_t)stream>>>(n, P, g, y, alpha);
    LU_CHECK();
    return PF_OK;
}

int pf_lu_forward(int32_t K, int32_t n, int32_t nnz_m, int32_t n_rows, const int32_t* rows,
                  const int32_t* m_ptr, const int32_t* m_idx, int32_t col_end, const double* m,
                  double* y, void* stream) {
    if (K <= 0 || n_rows < 0) return lu_invalid("bad sizes");
    if (n_rows == 0) return PF_OK;
    if (!rows || !m_ptr || !m_idx || !m || !y) return lu_invalid("NULL argument");
    pf::k_lu_forward<<<dim3(pf::cdiv(n_rows, pf::LU_WARPS), pf::cdiv(K, PF_LANES)),
                       32 * pf::LU_WARPS, 0, (cudaStream_t)stream>>>(
        n_rows, rows, n, nnz_m, m_ptr, m_idx, col_end, m, y);
    LU_CHECK();
    return PF_OK;
}

int pf_lu_backward(int32_t K, int32_t n, int32_t nnz_m, int32_t n_rows, const int32_t* rows,
                   const int32_t* m_ptr, const int32_t* m_diag, const int32_t* m_idx,
                   const double* m, double* y, void* stream) {
    if (K <= 0 || n_rows < 0) return lu_invalid("bad sizes");
    if (n_rows == 0) return PF_OK;
    if (!rows || !m_ptr || !m_diag || !m_idx || !m || !y) return lu_invalid("NULL argument");
    pf::k_lu_backward<<<dim3(pf::cdiv(n_rows, pf::LU_WARPS), pf::cdiv(K, PF_LANES)),
                        32 * pf::LU_WARPS, 0, (cudaStream_t)stream>>>(
        n_rows, rows, n, nnz_m, m_ptr, m_diag, m_idx, m, y);
    LU_CHECK();
    return PF_OK;
}

int pf_lu_tail_vec(int32_t K, int32_t n, int32_t t0, int32_t D, double* y, double* v,
                   int32_t to_dense, void* stream) {
    if (K <= 0 || D < 0 || t0 < 0 || t0 + D > n) return lu_invalid("bad sizes");
    if (D == 0) return PF_OK;
    if (!y || !v) return lu_invalid("NULL argument");
    pf::k_lu_tail_vec<<<dim3(pf::cdiv(D, 32), pf::cdiv(K, PF_LANES)), 32 * pf::LU_WARPS, 0,
                        (cudaStream_t)stream>>>(K, n, t0, D, y, v, to_dense);
    LU_CHECK();
    return PF_OK;
}

int pf_lu_residual(int32_t K, int32_t n, int32_t nnz, const int32_t* csr_ptr,
                   const int32_t* csr_idx, const double* jv, const double* x, const double* g,
                   double* res, void* stream) {
    if (K <= 0 || n < 0 || nnz < 0) return lu_invalid("bad sizes");
    if (!csr_ptr || !csr_idx || !jv || !x || !g || !res) return lu_invalid("NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    PF_CUDA(cudaMemsetAsync(res, 0, sizeof(double) * (size_t)K, st));
    if (n == 0) return PF_OK;
    pf::k_lu_residual<<<dim3(pf::cdiv(n, pf::LU_WARPS), pf::cdiv(K, PF_LANES)), 32 * pf::LU_WARPS,
                        0, st>>>(K, n, nnz, csr_ptr, csr_idx, jv, x, g,
                                 reinterpret_cast<unsigned long long*>(res));
    LU_CHECK();
    return PF_OK;
}

int pf_lu_apply(int32_t K, int32_t n, const int32_t* Q, const double* x, double* state,
                const int32_t* active, void* stream) {
    if (K <= 0 || n < 0) return lu_invalid("bad sizes");
    if (n == 0) return PF_OK;
    if (!Q || !x || !state) return lu_invalid("NULL argument");
    pf::k_lu_apply<<<dim3(pf::cdiv(n, pf::LU_WARPS), pf::cdiv(K, PF_LANES)), 32 * pf::LU_WARPS, 0,
                     (cudaStream_t)stream>>>(K, n, Q, x, state, active);
    LU_CHECK();
    return PF_OK;
}

}  // extern "C"
