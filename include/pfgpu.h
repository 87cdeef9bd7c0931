/*
 * pfgpu.h - C ABI of the B200 power-flow evaluation engine (libpfgpu.so).
 *
 * The engine evaluates the power-flow residual g(y) and the Jacobian values
 * dg/dy on a fixed sparsity pattern for the extended Newton formulation of
 * arXiv 2011.11880: Line pi-branches (tap + phase shift), bus P/Q balance,
 * PQ loads, PV voltage control, Slack V/theta control, bus shunts.
 *
 * It replaces the reference package pflow's per-model evaluation path
 * (/root/reference/pkg/src/pflow).  Each entry point below names the
 * reference function it stands in for.  Conventions:
 *   - plain pointers and sizes only; no framework types;
 *   - every function returns an int status (PF_OK = 0); on failure the
 *     message is available from pf_last_error() (thread-local);
 *   - "device" pointers are CUDA global-memory pointers (e.g. from
 *     torch.Tensor.data_ptr()); "host" pointers are ordinary CPU memory
 *     (pinned memory makes the copies asynchronous DMA);
 *   - stream arguments are cudaStream_t passed as void* (NULL = legacy
 *     default stream); device entry points only enqueue work;
 *   - the plan owns only immutable topology, coefficients and the symbolic
 *     pattern; evaluation allocates nothing (pflow SPEC.md:197).
 *
 * Addressing (pflow/system_model.py:3-11): y = [theta(N) | V(N) | Q_g(G+S) |
 * P_s(S)], g = [g_p(N) | g_q(N) | g_V(G+S) | g_theta(S)], n = 2N+G+2S.
 *
 * Batched layout ("scenario blocks"): K scenarios are stored in blocks of
 * PF_LANES = 32 scenarios; element (entry e, scenario s) of an array with
 * n_e entries per scenario lives at ((s / 32) * n_e + e) * 32 + (s % 32).
 * Buffers hold ceil(K/32) full blocks.
 */
#ifndef PFGPU_H
#define PFGPU_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PF_API __attribute__((visibility("default")))
#else
#define PF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define PF_OK 0
#define PF_EINVAL 1   /* bad argument / unsupported topology     */
#define PF_ECUDA 2    /* CUDA runtime error                       */
#define PF_ESHAPE 3   /* size mismatch                            */
#define PF_ENOMEM 4   /* allocation failure                       */

#define PF_LANES 32   /* scenarios per block in batched layout    */

/* Network in per-unit structure-of-arrays form: the fields of
 * pflow.PowerSystem (pflow/system_model.py:45-180).  All pointers are host
 * pointers, read during pf_plan_create only.  Arrays of length 0 may be
 * NULL.  Requirements (guaranteed by pflow.build_system): bus indices in
 * [0, n_bus); pv_qg = 0..n_pv-1; sl_qg = n_pv..n_pv+n_slack-1;
 * sl_ps = 0..n_slack-1; no self-loop branches (bus_h != bus_k). */
typedef struct pf_topology {
    int32_t n_bus;
    int32_t n_line;
    const int32_t* bus_h;   const int32_t* bus_k;
    const double* gl;       const double* bl;
    const double* gl2;      const double* bl2;
    const double* g_self_h; const double* b_self_h;
    const double* g_self_k; const double* b_self_k;
    int32_t n_pq;
    const int32_t* pq_bus;  const double* pq_p0;  const double* pq_q0;
    int32_t n_pv;
    const int32_t* pv_bus;  const double* pv_p0;  const double* pv_v0;
    const int32_t* pv_qg;
    int32_t n_slack;
    const int32_t* sl_bus;  const double* sl_v0;  const double* sl_th0;
    const int32_t* sl_qg;   const int32_t* sl_ps;
    int32_t n_shunt;
    const int32_t* sh_bus;  const double* sh_g;   const double* sh_b;
} pf_topology;

typedef struct pf_plan pf_plan;

/* indices into the dims array of pf_plan_dims */
enum {
    PF_DIM_NBUS = 0, PF_DIM_NLINE, PF_DIM_NVAR, PF_DIM_NNZ, PF_DIM_NPQ,
    PF_DIM_NPV, PF_DIM_NSLACK, PF_DIM_NSHUNT, PF_DIM_NINC, PF_DIM_MAXDEG,
    PF_DIM_SG_CHUNKS,   /* single-grid CTAs (bus chunks) */
    PF_DIM_SG_BIG,      /* of which single over-cap buses evaluated serially */
    PF_DIM_COUNT
};

PF_API const char* pf_last_error(void);
PF_API int pf_version(void);

/* Upload the network and build the symbolic Jacobian pattern on the device.
 * Replaces ResidualWorkspace.__init__/_build_join (pflow/residual.py:49-125)
 * and symbolic_pattern/_enumerate_slots (pflow/jacobian.py:42-80, 179-213).
 * Uses the current CUDA device. */
PF_API int pf_plan_create(const pf_topology* topo, pf_plan** out);
PF_API int pf_plan_destroy(pf_plan* plan);
PF_API int pf_plan_dims(const pf_plan* plan, int64_t* dims /* [PF_DIM_COUNT] */);

/* Symbolic pattern as CSR (host outputs, indptr[n_var+1], indices[nnz]);
 * equals pflow JacobianWorkspace.csc.tocsr() (pflow/jacobian.py:50-72). */
PF_API int pf_plan_pattern_csr(const pf_plan* plan, int32_t* indptr, int32_t* indices);
/* CSC view (host outputs): csc_indptr[n_var+1], csc_indices[nnz] equal
 * JacobianWorkspace.csc.indptr/.indices; csc_data[q] = csr_data[perm[q]]. */
PF_API int pf_plan_pattern_csc(const pf_plan* plan, int32_t* csc_indptr, int32_t* csc_indices,
                        int32_t* perm);

/* Fused residual + Jacobian evaluation for one grid (device pointers).
 * y[n_var] -> g[n_eq] (pflow evaluate_residual, residual.py:262-274),
 * jval[nnz] CSR-ordered values (pflow evaluate_jacobian, jacobian.py:216-221),
 * norm[1] = max|g| (pflow/newton.py:84-85).  Any output may be NULL to skip it.
 * One launch.  The norm reduction uses a plan-owned accumulator: evaluations
 * of one plan that request `norm` must not run concurrently (different plans
 * may; batched evaluations are unaffected). */
PF_API int pf_eval(const pf_plan* plan, const double* y, double* g, double* jval, double* norm,
            void* stream);

/* K scenarios over the shared topology (device pointers, batched layout).
 * y: n_var entries; pq_p/pq_q: n_pq entries; pv_p: n_pv entries (NULL = the
 * plan's base values); outage[K]: branch index zeroed in that scenario, -1 =
 * none (NULL = no outages; an index outside [-1, n_line) is treated as none
 * here and rejected with PF_EINVAL by pf_eval_batched_host).  Outputs g (n_var entries), jval (nnz entries,
 * CSR order), norms[K] = max_r |g_s[r]|; any may be NULL.  Equivalent to
 * mutating pflow.PowerSystem arrays per scenario and running wf1. */
PF_API int pf_eval_batched(const pf_plan* plan, int32_t K, const double* y, const double* pq_p,
                    const double* pq_q, const double* pv_p, const int32_t* outage,
                    double* g, double* jval, double* norms, void* stream);

/* Permute CSR-ordered Jacobian values into the reference's CSC order
 * (device pointers). K = 0: single grid (nnz values); K > 0: batched layout. */
PF_API int pf_jac_to_csc(const pf_plan* plan, int32_t K, const double* jcsr, double* jcsc,
                  void* stream);

/* Host-buffer drop-in: copies y in, evaluates, copies g / CSC-ordered J /
 * norm out, synchronously, through plan-owned device staging.
 * Same contract as pflow evaluate_residual + evaluate_jacobian (host arrays).
 * Any output may be NULL. */
PF_API int pf_eval_host(pf_plan* plan, const double* y, double* g, double* jcsc, double* norm);

/* Host-buffer batched evaluation, pipelined over scenario blocks on
 * n_streams streams (H2D / kernel / D2H overlap).  Host arrays in batched
 * layout; jval is CSR-ordered.  Synchronous. */
PF_API int pf_eval_batched_host(pf_plan* plan, int32_t K, const double* y, const double* pq_p,
                         const double* pq_q, const double* pv_p, const int32_t* outage,
                         double* g, double* jval, double* norms, int32_t blocks_per_stage,
                         int32_t n_streams);

/* ---- per-model entry points (unit parity with the reference kernels) ---- */

/* Line terminal injections ph, pk, qh, qk [n_line] (pflow kernels.py:79-97,
 * residual.py:287-314 line_injections). */
PF_API int pf_line_injections(const pf_plan* plan, const double* y, double* ph, double* pk,
                       double* qh, double* qk, void* stream);
/* The 16 line partial sections [16][n_line] in pflow/jacobian.py:31-36 order
 * (kernels.py:128-163). */
PF_API int pf_line_jacobian_slots(const pf_plan* plan, const double* y, double* slots, void* stream);
/* Device contributions laid out as pool segments 4..14 of
 * pflow/residual.py:57: [pq_p|pq_q|pv_p|pv_q|pv_v|sl_p|sl_q|sl_v|sl_th|sh_p|sh_q]
 * (kernels.py:215-241). */
PF_API int pf_device_injections(const pf_plan* plan, const double* y, double* pool, void* stream);
/* Device Jacobian slots [pv_gq_qg|pv_gv_v|sl_gp_ps|sl_gq_qg|sl_gv_v|sl_gth_th|
 * sh_gp_v|sh_gq_v] (kernels.py:244-262, jacobian.py:200-207). */
PF_API int pf_device_jacobian_slots(const pf_plan* plan, const double* y, double* slots,
                             void* stream);
/* Generic row gather-sums over a pool (device pointers):
 * join: out[r] = 0 - pool[idx[ptr[r]..split[r])] + pool[idx[split[r]..ptr[r+1])]
 * (kernels.py:265-274);  gather: out[r] = sum pool[idx[ptr[r]..ptr[r+1])]
 * (kernels.py:277-282); both in index order. */
PF_API int pf_join_rows(int32_t n_rows, const int32_t* ptr, const int32_t* split, const int32_t* idx,
                 const double* pool, double* out, void* stream);
PF_API int pf_gather_sum(int32_t n_rows, const int32_t* ptr, const int32_t* idx, const double* vals,
                  double* out, void* stream);

/* sin/cos over an array with the engine's trig routine (device pointers);
 * test surface like pflow kernels.py:66-72 `sincos`. */
PF_API int pf_sincos(int64_t n, const double* x, double* s, double* c, void* stream);

/* ---- hand-off to a batched linear solver ----------------
 * Scenario-major <-> blocked layout.  pf_batch_unblock: dst[s * n_e + e] =
 * alpha * src(e, s) for s < K (alpha = 1 or -1 is exact), e.g. the CSR
 * Jacobian values of each scenario as one contiguous array, or -g as the
 * right-hand sides.  pf_batch_update: y(e, s) += dx[s * n_e + e] for every
 * scenario with active[s] != 0 (active may be NULL: all).  Device pointers. */
PF_API int pf_batch_unblock(int32_t K, int32_t n_e, const double* src, double* dst, double alpha,
                            void* stream);
PF_API int pf_batch_update(int32_t K, int32_t n_e, double* y, const double* dx,
                           const int32_t* active, void* stream);

/* ---- batched sparse LU on a fixed schedule -------------
 * The K scenarios share one pattern, pivot order and elimination schedule
 * (built on the host by paper_2011_11880_b200/batched_lu.py); factor values
 * M (nnz_m per scenario) and vectors (n per scenario) use the blocked layout.
 *   pf_lu_scatter     M = 0, then M[a2m[e]] = A[e]                     (A: CSR values)
 *   pf_lu_eliminate   rows by records {pos_ik, pos_kk, u0, u1} (int32[4]) and
 *                     update pairs {pos_kj, pos_ij} (int32[2]): l = m_ik / u_kk,
 *                     m_ik = l, m_ij -= l u_kj; rec_ptr[n_rows + 1]
 *   pf_lu_tail_gather dense trailing block t[K][D][D] (tail_pos[D*D], -1 = zero)
 *   pf_lu_rhs         y(i) = alpha g(P[i])
 *   pf_lu_forward     rows[]: y_i -= sum m_ik y_k, k < min(i, col_end)
 *   pf_lu_backward    rows[]: y_i = (y_i - sum_{j > i} m_ij y_j) / m_ii
 *   pf_lu_tail_vec    entries [t0, t0 + D) of y <-> v[K][D] (to_dense = 1: y -> v)
 *   pf_lu_apply       state(Q[j]) += x(j) where active[s] (NULL: all)
 *   pf_lu_residual    max_i |g_i + (J x)_i| per scenario
 * Device pointers; asynchronous on `stream`. */
PF_API int pf_lu_scatter(int32_t K, int32_t nnz_a, int32_t nnz_m, const int32_t* a2m,
                         const double* a, double* m, void* stream);
PF_API int pf_lu_eliminate(int32_t K, int32_t nnz_m, int32_t n_rows, const int32_t* rec_ptr,
                           const int32_t* rec, const int32_t* upd, double* m, void* stream);
PF_API int pf_lu_tail_gather(int32_t K, int32_t nnz_m, int32_t D, const int32_t* tail_pos,
                             const double* m, double* t, void* stream);
PF_API int pf_lu_rhs(int32_t K, int32_t n, const int32_t* P, const double* g, double* y,
                     double alpha, void* stream);
PF_API int pf_lu_forward(int32_t K, int32_t n, int32_t nnz_m, int32_t n_rows, const int32_t* rows,
                         const int32_t* m_ptr, const int32_t* m_idx, int32_t col_end,
                         const double* m, double* y, void* stream);
PF_API int pf_lu_backward(int32_t K, int32_t n, int32_t nnz_m, int32_t n_rows,
                          const int32_t* rows, const int32_t* m_ptr, const int32_t* m_diag,
                          const int32_t* m_idx, const double* m, double* y, void* stream);
PF_API int pf_lu_tail_vec(int32_t K, int32_t n, int32_t t0, int32_t D, double* y, double* v,
                          int32_t to_dense, void* stream);
PF_API int pf_lu_apply(int32_t K, int32_t n, const int32_t* Q, const double* x, double* state,
                       const int32_t* active, void* stream);
/* res[s] = max_i |g_i + sum_j J_ij x_j| for scenario s (J: CSR values of the
 * plan pattern, all blocked): the accuracy check of a batched solve. */
PF_API int pf_lu_residual(int32_t K, int32_t n, int32_t nnz, const int32_t* csr_ptr,
                          const int32_t* csr_idx, const double* jv, const double* x,
                          const double* g, double* res, void* stream);

/* Number of kernels this library has launched (process-wide counter). */
PF_API int64_t pf_launch_count(void);

/* Page-lock (and release) a caller-owned host range, so host-buffer calls
 * on it move data by DMA at full PCIe rate (the workspaces register the
 * state vector they are bound to).  Registering an already registered range
 * and unregistering an unregistered one are no-ops. */
PF_API int pf_host_register(void* ptr, size_t bytes);
PF_API int pf_host_unregister(void* ptr);

/* Number of device allocations this library has made (process-wide counter):
 * plan creation and the first host-buffer call per plan allocate; evaluations
 * never do (SPEC.md:197, 457 allocation contract). */
PF_API int64_t pf_alloc_count(void);

#ifdef __cplusplus
}
#endif
#endif /* PFGPU_H */
