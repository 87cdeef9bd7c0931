// pf_internal.cuh - device plan layout shared by the libpfgpu translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/pfgpu.h"

namespace pf {

// Per-incidence metadata flag bits (inc_meta.z).
constexpr int32_t KSIDE = 1 << 30;   // this bus is the branch's k (to) terminal
constexpr int32_t FIRST = 1 << 29;   // first incidence of this neighbour in the bus's list
constexpr int32_t SOLO = 1 << 28;    // the only incidence of this neighbour (no parallel branch)
constexpr int32_t POS_MASK = (1 << 28) - 1;

// Per-bus row descriptor (bus_row.w flag bits).
constexpr int32_t VDIAG = 1 << 30;   // row holds a (g, V_i) diagonal entry
constexpr int32_t DUPS = 1 << 29;    // some neighbour is reached by parallel branches

// buses with at least this many incidences are scheduled first (batched)
constexpr int HUB_DEG = 16;

// Single grid (k_eval_single): one CTA of SG_THREADS per chunk of at most
// SG_THREADS consecutive buses whose incidences, Jacobian rows g_p / g_q and
// parallel-branch slots fit the shared-memory caps below (plan-built).
constexpr int SG_THREADS = 128;
// 5 CTAs per SM (<= 102 registers): config 2's ~700 chunks run in one wave.
// Measured on B200 (config 2, f+J+norm): 4 CTAs 15.0 us, 5 CTAs 10.2 us,
// 6 CTAs (80 registers, spills) 13.2 us; 256-thread CTAs 14.2-15.2 us.
constexpr int SG_MINB = 5;
constexpr int SG_CAP_BUS = SG_THREADS;
constexpr int SG_CAP_INC = 2 * SG_THREADS;   // incidences per chunk (two per thread)
constexpr int SG_CAP_J = 16 * SG_THREADS;    // Jacobian values in the chunk's rows g_p, g_q
constexpr int SG_CAP_DUP = SG_THREADS / 4;   // incidences sharing a neighbour with a parallel branch
constexpr int32_t SG_BIG = 1 << 30;  // chunk flag: one bus over the caps, evaluated serially
// sg_inc.y: owner bus (chunk-local, bits 0-9) | dup slot << SG_DUP_SHIFT | SOLO | KSIDE
constexpr int32_t SG_FIELD_MASK = 0x3ff;
constexpr int SG_DUP_SHIFT = 10;
static_assert(SG_CAP_BUS <= SG_FIELD_MASK + 1 && SG_CAP_DUP <= SG_FIELD_MASK + 1, "sg_inc");

// Batched kernel, warp-specialised (k_eval_staged): a producer warp copies
// each bus's operands into a consumer warp's shared-memory slot with cp.async.
// Per bus (processing order) the plan holds a packet of 16-byte units
//   [0] bus_row[2i]  [1] bus_row[2i+1]  [2] {ni, nv, bus, 0}
//   [3, 3+ni) inc_meta   [3+ni, 3+3ni) inc_coef   [3+3ni, +nv) dev_list
//   [3+3ni+nv, +nv) device constants {c, d} (double2)
// and a stage record of WS_REC_WORDS int32: {packet offset (units),
// packet units | rows << 16, row code x WS_ROWS} naming the 256-byte scenario
// rows to stage: 0 theta_i, 1 V_i, 2+2t / 3+2t theta_j / V_j of staged
// incidence t < ni, 2+2ni+2u / 3+2ni+2u operands a / b of staged device u < nv.
// Row code = (array << 29) | entry (array 0 y, 1 pq_p, 2 pq_q, 3 pv_p), -1 none.
// Incidences and devices past the staged ones are read from global memory.
#ifndef PF_WS_ROWS
#define PF_WS_ROWS 14
#endif
constexpr int WS_ROWS = PF_WS_ROWS;
constexpr int WS_MAXINC = 6;
// CTA shape: WS_W warps, WS_MINB CTAs per SM (24 warps/SM at 80 registers).
// A CTA's item is a group of WS_W consecutive slots of the processing order.
// Measured on B200 (ms per launch, config 3 / config 4): 24 x 1 0.597 /
// 0.645 with hubs first in the order (0.61 with hubs spread, see
// pf_plan.cu), 12 x 2 0.625 / 0.615, 20 x 1 (91 registers) 0.613 / 0.627,
// 16 x 1 (104 registers) 0.662 / 0.636, 6 x 4 0.640 / 0.608.
#ifndef PF_WS_W
#define PF_WS_W 24
#define PF_WS_MINB 1
#endif
constexpr int WS_W = PF_WS_W;
constexpr int WS_MINB = PF_WS_MINB;
constexpr int WS_MAXDEV = 2;
constexpr int WS_PKT_UNITS = 3 + 3 * WS_MAXINC + 2 * WS_MAXDEV;   // 25
constexpr int WS_REC_WORDS = 2 + WS_ROWS;                        // 16 (64 bytes)
static_assert(WS_PKT_UNITS <= 32, "one cp.async per lane covers the packet");

// Device-list entry types, in the reference's pool-segment order (residual.py:57).
enum DevType : int32_t { DEV_PQ = 0, DEV_PV = 1, DEV_SLACK = 2, DEV_SHUNT = 3 };

// Everything the evaluation kernels read.  All pointers are device memory.
struct DevicePlan {
    int32_t N, L, P, G, S, H, n_gen, n_var, nnz, n_inc;
    // single grid: chunk records [2 sg_chunks]: {b0, b1 | SG_BIG, e0, e1},
    // {p0, p1, q0, q1} (CSR ranges of rows g_p[b0..b1), g_q[b0..b1)), and per
    // incidence {neighbour, sg_inc.y fields, staged position of the
    // (g_p[i], theta_j) entry, staged position of the (g_q[i], theta_j) entry}
    int32_t sg_chunks;
    const int4* sg_chunk;
    const int4* sg_inc;
    unsigned long long* sg_acc;   // norm accumulator, 0 between launches
    unsigned int* sg_count;       // CTAs done, 0 between launches
    // incidence lists: bus i owns [inc_ptr[i], inc_ptr[i+1]) in the order
    // (branches with h=i ascending) ++ (branches with k=i ascending)
    const int32_t* inc_ptr;   // [N+1]
    const int4* inc_meta;     // [n_inc] {neighbour j, branch l, pos|flags, owning bus}
    const double4* inc_coef;  // [n_inc] {g1, b1, gs, bs}: h side {gl, bl, gsh, bsh},
                              //          k side {gl2, bl2, gsk, bsk}
    const int4* bus_row;      // [2N] bus header: [2i] = {rp, rq, nb, pos_i|VDIAG}: CSR
                              // offsets of rows g_p[i], g_q[i], theta-block size,
                              // diagonal rank; [2i+1] = {e0, e1, t0, t1}: incidence
                              // and device-list ranges (one 32-byte load)
    const int32_t* bus_order; // [N] batched processing order (hubs spread, then bus order)
    int32_t n_hubs;           // buses with degree >= HUB_DEG
    const int4* ws_pkt;       // staged-kernel packets (see WS_ROWS above)
    const int4* ws_rec;       // [N * WS_REC_WORDS / 4] stage records in processing order
    int32_t ws_keep;          // 1: packets and records are read with an L2 evict-last
                              // policy (they fit in L2 beside one block's states)
    const int32_t* dev_ptr;   // [N+1]
    const int4* dev_list;     // [n_dev] {type, index, jpos_a, jpos_b}
    // device parameters (base values; scenarios may override P/Q)
    const double *pq_p0, *pq_q0, *pv_p0, *pv_v0, *sl_v0, *sl_th0, *sh_g, *sh_b;
    const int32_t *pv_qg, *sl_qg, *sl_ps;
    const int32_t* gen_row_pos;  // [n_gen + S]: CSR position of the single entry of
                                 // rows g_V (n_gen) then g_theta (S)
    // original branch-indexed SoA (per-model entry points)
    const int32_t *bus_h, *bus_k;
    const double *gl, *bl, *gl2, *bl2, *gsh, *bsh, *gsk, *bsk;
    const int32_t *pq_bus, *pv_bus, *sl_bus, *sh_bus;
    // pattern
    const int32_t* csr_indptr;   // [n_var+1]
    const int32_t* csr_indices;  // [nnz]
    const int32_t* csc_indptr;   // [n_var+1]
    const int32_t* csc_indices;  // [nnz]
    const int32_t* csc_perm;     // [nnz] csc value q = csr value csc_perm[q]
};

struct Staging {
    int32_t n_streams = 0;
    int32_t blocks = 0;           // scenario blocks per stage
    cudaStream_t streams[8] = {};
    double* y[8] = {};
    double* g[8] = {};
    double* j[8] = {};
    double* pq_p[8] = {};
    double* pq_q[8] = {};
    double* pv_p[8] = {};
    int32_t* outage[8] = {};
    double* norms[8] = {};
};

}  // namespace pf

struct pf_plan {
    pf::DevicePlan d;
    int32_t max_deg = 0;
    int32_t sg_big = 0;     // single-grid chunks evaluated serially (one over-cap bus)
    void* owned[96] = {};   // device allocations to free
    int n_owned = 0;
    // single-grid host drop-in staging
    double *s_y = nullptr, *s_g = nullptr, *s_j = nullptr, *s_jc = nullptr, *s_norm = nullptr;
    cudaStream_t s_stream = nullptr;
    pf::Staging batch;
};

namespace pf {

void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
void count_launch(int n = 1);

#define PF_CUDA(call)                                         \
    do {                                                      \
        cudaError_t _e = (call);                              \
        if (_e != cudaSuccess) return pf::cuda_fail(_e, #call); \
    } while (0)

// kernel launchers (pf_eval.cu)
cudaError_t launch_eval_single(const DevicePlan& d, const double* y, double* g, double* j,
                               double* norm, cudaStream_t st);
cudaError_t launch_eval_batched(const DevicePlan& d, int32_t K, const double* y,
                                const double* pq_p, const double* pq_q, const double* pv_p,
                                const int32_t* outage, double* g, double* j, double* norms,
                                cudaStream_t st);
cudaError_t launch_jac_to_csc(const DevicePlan& d, int32_t K, const double* jcsr, double* jcsc,
                              cudaStream_t st);
cudaError_t launch_line_injections(const DevicePlan& d, const double* y, double* ph, double* pk,
                                   double* qh, double* qk, cudaStream_t st);
cudaError_t launch_line_jac_slots(const DevicePlan& d, const double* y, double* slots,
                                  cudaStream_t st);
cudaError_t launch_device_injections(const DevicePlan& d, const double* y, double* pool,
                                     cudaStream_t st);
cudaError_t launch_device_jac_slots(const DevicePlan& d, const double* y, double* slots,
                                    cudaStream_t st);
cudaError_t launch_join_rows(int32_t n, const int32_t* ptr, const int32_t* split,
                             const int32_t* idx, const double* pool, double* out,
                             cudaStream_t st);
cudaError_t launch_sincos(int64_t n, const double* x, double* s, double* c, cudaStream_t st);
cudaError_t launch_batch_unblock(int32_t K, int32_t n_e, const double* src, double* dst,
                                 double alpha, cudaStream_t st);
cudaError_t launch_batch_update(int32_t K, int32_t n_e, double* y, const double* dx,
                                const int32_t* active, cudaStream_t st);
cudaError_t launch_gather_sum(int32_t n, const int32_t* ptr, const int32_t* idx,
                              const double* vals, double* out, cudaStream_t st);

}  // namespace pf
