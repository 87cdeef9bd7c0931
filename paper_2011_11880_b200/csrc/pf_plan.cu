// pf_plan.cu - device-side symbolic build and the C ABI of libpfgpu.
//
// pf_plan_create uploads the network once and builds, on the device, every
// index structure the evaluation kernels read: the bus -> incident-branch
// CSR (incidence order = the reference's join order, residual.py:79-125),
// per-incidence coefficient records, the per-bus device lists, the Jacobian
// CSR pattern and its CSC permutation (the pattern the reference builds with
// np.lexsort in jacobian.py:50-72).  Sorting uses CUB's stable LSD radix
// sort, so the build is deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <cub/cub.cuh>
#include <string>
#include <vector>

#include "pf_internal.cuh"

namespace pf {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};
static std::atomic<int64_t> g_allocs{0};

// Every device allocation of the library goes through here (counted: the
// zero-allocation steady state of SPEC.md:197 / 457 is asserted in tests).
template <class T>
static cudaError_t dmalloc(T** p, size_t bytes) {
    g_allocs.fetch_add(1, std::memory_order_relaxed);
    return cudaMalloc((void**)p, bytes);
}

void set_error(const std::string& msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
    return PF_ECUDA;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {

constexpr unsigned long long SENTINEL = ~0ull;

inline unsigned grid_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

int nbits(uint64_t v) {
    int b = 0;
    while (v) { ++b; v >>= 1; }
    return b > 0 ? b : 1;
}

// ---- build kernels ----------------------------------------------------------

__global__ void k_iota_keys(int64_t n, const int32_t* key_src0, int64_t n0, const int32_t* key_src1,
                            int64_t n1, const int32_t* key_src2, int64_t n2,
                            const int32_t* key_src3, uint32_t* keys, int32_t* vals) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n) return;
    int32_t k;
    if (e < n0) k = key_src0[e];
    else if (e < n0 + n1) k = key_src1[e - n0];
    else if (e < n0 + n1 + n2) k = key_src2[e - n0 - n1];
    else k = key_src3[e - n0 - n1 - n2];
    keys[e] = (uint32_t)k;
    vals[e] = (int32_t)e;
}

// ptr[i] = first position with key >= i (keys sorted ascending), i in [0, n]
__global__ void k_lower_bound_u32(const uint32_t* keys, int64_t m, int32_t n, int32_t* ptr) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < (uint32_t)i) lo = mid + 1; else hi = mid;
    }
    ptr[i] = (int32_t)lo;
}

__global__ void k_lower_bound_hi(const unsigned long long* keys, int64_t m, int32_t n,
                                 int32_t* ptr) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if ((keys[mid] >> 32) < (unsigned long long)i) lo = mid + 1; else hi = mid;
    }
    ptr[i] = (int32_t)lo;
}

// incidence records in sorted (bus, side, branch) order
__global__ void k_inc_records(int32_t L, const int32_t* sorted_e, const int32_t* bh,
                              const int32_t* bk, const double* gl, const double* bl,
                              const double* gl2, const double* bl2, const double* gsh,
                              const double* bsh, const double* gsk, const double* bsk,
                              int4* meta, double4* coef) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= 2 * (int64_t)L) return;
    int32_t e = sorted_e[t];
    bool ks = e >= L;
    int32_t l = ks ? e - L : e;
    meta[t] = make_int4(ks ? bh[l] : bk[l], l, ks ? KSIDE : 0, ks ? bk[l] : bh[l]);
    coef[t] = ks ? make_double4(gl2[l], bl2[l], gsk[l], bsk[l])
                 : make_double4(gl[l], bl[l], gsh[l], bsh[l]);
}

// closed-neighbourhood pairs: incidences, then one self pair per bus with
// at least one incidence (other buses get the sentinel key, sorted last)
__global__ void k_nbr_pairs(int32_t N, int32_t n_inc, const int4* meta, const int32_t* inc_ptr,
                            const uint32_t* sorted_bus, unsigned long long* keys,
                            int32_t* vals) {
    int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (u < n_inc) {
        keys[u] = ((unsigned long long)sorted_bus[u] << 32) | (uint32_t)meta[u].x;
        vals[u] = (int32_t)u;
    } else if (u < (int64_t)n_inc + N) {
        int32_t i = (int32_t)(u - n_inc);
        bool has = inc_ptr[i + 1] > inc_ptr[i];
        keys[u] = has ? (((unsigned long long)i << 32) | (uint32_t)i) : SENTINEL;
        vals[u] = n_inc + i;
    }
}

__global__ void k_heads(int64_t m, const unsigned long long* keys, int32_t* head) {
    int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (u >= m) return;
    head[u] = (keys[u] != SENTINEL) && (u == 0 || keys[u] != keys[u - 1]) ? 1 : 0;
}

// q = inclusive scan of heads (1-based unique index).  ubase[bus] = unique
// index of the bus's first column, uend[bus] = one past its last.
__global__ void k_seg_bounds(int64_t m, const unsigned long long* keys, const int32_t* q,
                             int32_t* ubase, int32_t* uend) {
    int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (u >= m || keys[u] == SENTINEL) return;
    uint32_t bus = (uint32_t)(keys[u] >> 32);
    if (u == 0 || (uint32_t)(keys[u - 1] >> 32) != bus) ubase[bus] = q[u] - 1;
    if (u == m - 1 || keys[u + 1] == SENTINEL || (uint32_t)(keys[u + 1] >> 32) != bus)
        uend[bus] = q[u];
}

// per pair: unique column list, incidence rank/flags, diagonal rank
__global__ void k_nbr_ranks(int64_t m, int32_t n_inc, const unsigned long long* keys,
                            const int32_t* vals, const int32_t* head, const int32_t* q,
                            const int32_t* ubase, int32_t* ucol, int4* meta, int32_t* pos_i) {
    int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (u >= m || keys[u] == SENTINEL) return;
    uint32_t bus = (uint32_t)(keys[u] >> 32);
    int32_t col = (int32_t)(uint32_t)(keys[u] & 0xffffffffull);
    int32_t uq = q[u] - 1;
    if (head[u]) ucol[uq] = col;
    int32_t pos = uq - ubase[bus];
    int32_t v = vals[u];
    // SOLO: the only incidence of this (bus, neighbour) pair
    const bool solo = head[u] && (u + 1 == m || keys[u + 1] != keys[u]);
    if (v < n_inc) meta[v].z |= pos | (head[u] ? FIRST : 0) | (solo ? SOLO : 0);
    else pos_i[bus] = pos;
}

struct DevGroups {
    int32_t P, G, S, H;
    const int32_t *pv_qg, *sl_qg, *sl_ps;
};

__device__ __forceinline__ void dev_of(const DevGroups& dg, int32_t id, int32_t& type,
                                       int32_t& idx) {
    if (id < dg.P) { type = DEV_PQ; idx = id; return; }
    id -= dg.P;
    if (id < dg.G) { type = DEV_PV; idx = id; return; }
    id -= dg.G;
    if (id < dg.S) { type = DEV_SLACK; idx = id; return; }
    type = DEV_SHUNT; idx = id - dg.S;
}

// row lengths of g_p[i], g_q[i]; gen rows have one entry each
__global__ void k_row_len(int32_t N, int32_t n_gen, int32_t S, const int32_t* ubase,
                          const int32_t* uend, const int32_t* inc_ptr, const int32_t* dev_ptr,
                          const int32_t* dev_sorted, DevGroups dg, int64_t* rowlen) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < N) {
        int32_t i = (int32_t)t;
        int32_t nb = inc_ptr[i + 1] > inc_ptr[i] ? uend[i] - ubase[i] : 0;
        int32_t n_pv = 0, n_sl = 0;
        bool sh = false;
        for (int32_t u = dev_ptr[i]; u < dev_ptr[i + 1]; ++u) {
            int32_t type, idx;
            dev_of(dg, dev_sorted[u], type, idx);
            n_pv += type == DEV_PV;
            n_sl += type == DEV_SLACK;
            sh |= type == DEV_SHUNT;
        }
        int32_t nv = nb > 0 ? nb : (sh ? 1 : 0);
        rowlen[i] = nb + nv + n_sl;
        rowlen[N + i] = nb + nv + n_pv + n_sl;
    } else if (t >= 2 * (int64_t)N && t < 2 * (int64_t)N + n_gen + S) {
        rowlen[t] = 1;
    }
}

__global__ void k_fill(int32_t N, int32_t n_gen, const int32_t* ubase, const int32_t* uend,
                       const int32_t* inc_ptr, const int32_t* ucol, const int32_t* pos_i,
                       const int32_t* dev_ptr, const int32_t* dev_sorted, DevGroups dg,
                       const int64_t* indptr, int32_t* indices, int4* bus_row, int4* dev_list,
                       int32_t* gen_row_pos) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N) return;
    int32_t i = (int32_t)t;
    int32_t nb = inc_ptr[i + 1] > inc_ptr[i] ? uend[i] - ubase[i] : 0;
    bool sh = false;
    for (int32_t u = dev_ptr[i]; u < dev_ptr[i + 1]; ++u) {
        int32_t type, idx;
        dev_of(dg, dev_sorted[u], type, idx);
        sh |= type == DEV_SHUNT;
    }
    int32_t nv = nb > 0 ? nb : (sh ? 1 : 0);
    int64_t rp = indptr[i], rq = indptr[N + i];
    for (int32_t u = 0; u < nb; ++u) {
        int32_t c = ucol[ubase[i] + u];
        indices[rp + u] = c;
        indices[rp + nb + u] = N + c;
        indices[rq + u] = c;
        indices[rq + nb + u] = N + c;
    }
    if (nb == 0 && sh) {
        indices[rp] = N + i;
        indices[rq] = N + i;
    }
    int32_t cp = 0, cq = 0;  // device columns placed in rows g_p[i], g_q[i]
    for (int32_t u = dev_ptr[i]; u < dev_ptr[i + 1]; ++u) {
        int32_t type, idx;
        dev_of(dg, dev_sorted[u], type, idx);
        int4 ent = make_int4(type, idx, 0, 0);
        if (type == DEV_PV) {
            int32_t qg = dg.pv_qg[idx];
            int64_t at = rq + nb + nv + cq++;
            indices[at] = 2 * N + qg;                   // (g_q[i], Q_g)
            int64_t gr = indptr[2 * (int64_t)N + qg];   // row g_V of this gen
            indices[gr] = N + i;                        // (g_V, V_i)
            gen_row_pos[qg] = (int32_t)gr;
            ent.z = (int32_t)at;
            ent.w = (int32_t)gr;
        } else if (type == DEV_SLACK) {
            int32_t qg = dg.sl_qg[idx], ps = dg.sl_ps[idx];
            int64_t ap = rp + nb + nv + cp++;
            indices[ap] = 2 * N + n_gen + ps;           // (g_p[i], P_s)
            int64_t aq = rq + nb + nv + cq++;
            indices[aq] = 2 * N + qg;                   // (g_q[i], Q_g)
            int64_t gv = indptr[2 * (int64_t)N + qg];
            int64_t gt = indptr[2 * (int64_t)N + n_gen + ps];
            indices[gv] = N + i;                        // (g_V, V_i)
            indices[gt] = i;                            // (g_theta, theta_i)
            gen_row_pos[qg] = (int32_t)gv;
            gen_row_pos[n_gen + ps] = (int32_t)gt;
            ent.z = (int32_t)ap;
            ent.w = (int32_t)aq;
        }
        dev_list[u] = ent;
    }
    // parallel branches: more incidences than distinct neighbours (the theta
    // block also holds the bus itself)
    const bool dups = nb > 0 && inc_ptr[i + 1] - inc_ptr[i] > nb - 1;
    bus_row[2 * i] = make_int4((int32_t)rp, (int32_t)rq, nb,
                               pos_i[i] | (nv > 0 ? VDIAG : 0) | (dups ? DUPS : 0));
    bus_row[2 * i + 1] = make_int4(inc_ptr[i], inc_ptr[i + 1], dev_ptr[i], dev_ptr[i + 1]);
}

__global__ void k_csr_keys(int32_t n, const int64_t* indptr, const int32_t* indices,
                           unsigned long long* keys, int32_t* vals) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    for (int64_t p = indptr[r]; p < indptr[r + 1]; ++p) {
        keys[p] = ((unsigned long long)(uint32_t)indices[p] << 32) | (uint32_t)r;
        vals[p] = (int32_t)p;
    }
}

__global__ void k_csc_rows(int64_t nnz, const unsigned long long* keys, int32_t* rows) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < nnz) rows[q] = (int32_t)(uint32_t)(keys[q] & 0xffffffffull);
}

__global__ void k_i64_to_i32(int64_t n, const int64_t* a, int32_t* b) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n) b[t] = (int32_t)a[t];
}

// ---- host helpers ---------------------------------------------------------------

struct Scratch {
    std::vector<void*> ptrs;
    ~Scratch() {
        for (void* p : ptrs) cudaFree(p);
    }
    template <class T>
    cudaError_t alloc(T** p, int64_t n) {
        *p = nullptr;
        cudaError_t e = dmalloc(p, sizeof(T) * (size_t)(n > 0 ? n : 1));
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
};

template <class T>
cudaError_t owned_alloc(pf_plan* P, T** p, int64_t n) {
    *p = nullptr;
    if (P->n_owned >= (int)(sizeof(P->owned) / sizeof(P->owned[0]))) return cudaErrorMemoryAllocation;
    cudaError_t e = dmalloc(p, sizeof(T) * (size_t)(n > 0 ? n : 1));
    if (e == cudaSuccess) P->owned[P->n_owned++] = *p;
    return e;
}

template <class T>
cudaError_t upload(pf_plan* P, const T** dst, const T* src, int64_t n, cudaStream_t st) {
    T* d = nullptr;
    cudaError_t e = owned_alloc(P, &d, n);
    if (e != cudaSuccess) return e;
    if (n > 0 && src) e = cudaMemcpyAsync(d, src, sizeof(T) * (size_t)n, cudaMemcpyHostToDevice, st);
    *dst = d;
    return e;
}

void free_plan(pf_plan* P) {
    if (!P) return;
    for (int i = 0; i < P->n_owned; ++i) cudaFree(P->owned[i]);
    cudaFree(P->s_y); cudaFree(P->s_g); cudaFree(P->s_j); cudaFree(P->s_jc); cudaFree(P->s_norm);
    if (P->s_stream) cudaStreamDestroy(P->s_stream);
    Staging& b = P->batch;
    for (int s = 0; s < b.n_streams; ++s) {
        cudaFree(b.y[s]); cudaFree(b.g[s]); cudaFree(b.j[s]); cudaFree(b.pq_p[s]);
        cudaFree(b.pq_q[s]); cudaFree(b.pv_p[s]); cudaFree(b.outage[s]); cudaFree(b.norms[s]);
        if (b.streams[s]) cudaStreamDestroy(b.streams[s]);
    }
    delete P;
}

int invalid(const std::string& m) {
    set_error(m);
    return PF_EINVAL;
}

int validate(const pf_topology* t) {
    if (!t) return invalid("topology is NULL");
    if (t->n_bus < 0 || t->n_line < 0 || t->n_pq < 0 || t->n_pv < 0 || t->n_slack < 0 ||
        t->n_shunt < 0)
        return invalid("negative group size");
    const int32_t N = t->n_bus;
    auto in_range = [&](const int32_t* a, int32_t n, const char* what) -> int {
        if (n > 0 && !a) return invalid(std::string(what) + " is NULL");
        for (int32_t i = 0; i < n; ++i)
            if (a[i] < 0 || a[i] >= N)
                return invalid(std::string(what) + "[" + std::to_string(i) + "] = " +
                               std::to_string(a[i]) + " is not a bus index in [0, " +
                               std::to_string(N) + ")");
        return PF_OK;
    };
    int rc;
    if ((rc = in_range(t->bus_h, t->n_line, "bus_h"))) return rc;
    if ((rc = in_range(t->bus_k, t->n_line, "bus_k"))) return rc;
    if ((rc = in_range(t->pq_bus, t->n_pq, "pq_bus"))) return rc;
    if ((rc = in_range(t->pv_bus, t->n_pv, "pv_bus"))) return rc;
    if ((rc = in_range(t->sl_bus, t->n_slack, "sl_bus"))) return rc;
    if ((rc = in_range(t->sh_bus, t->n_shunt, "sh_bus"))) return rc;
    for (int32_t i = 0; i < t->n_line; ++i)
        if (t->bus_h[i] == t->bus_k[i])
            return invalid("branch " + std::to_string(i) + " is a self-loop (bus_h == bus_k), "
                           "which the engine does not support");
    const double* f[] = {t->gl, t->bl, t->gl2, t->bl2, t->g_self_h, t->b_self_h, t->g_self_k,
                         t->b_self_k};
    for (const double* a : f)
        if (t->n_line > 0 && !a) return invalid("branch coefficient array is NULL");
    if (t->n_pq > 0 && (!t->pq_p0 || !t->pq_q0)) return invalid("pq arrays are NULL");
    if (t->n_pv > 0 && (!t->pv_p0 || !t->pv_v0 || !t->pv_qg)) return invalid("pv arrays are NULL");
    if (t->n_slack > 0 && (!t->sl_v0 || !t->sl_th0 || !t->sl_qg || !t->sl_ps))
        return invalid("slack arrays are NULL");
    if (t->n_shunt > 0 && (!t->sh_g || !t->sh_b)) return invalid("shunt arrays are NULL");
    for (int32_t i = 0; i < t->n_pv; ++i)
        if (t->pv_qg[i] != i) return invalid("pv_qg must be 0..n_pv-1 (pflow build_system layout)");
    for (int32_t s = 0; s < t->n_slack; ++s) {
        if (t->sl_qg[s] != t->n_pv + s) return invalid("sl_qg must be n_pv..n_pv+n_slack-1");
        if (t->sl_ps[s] != s) return invalid("sl_ps must be 0..n_slack-1");
    }
    const int64_t n_var = 2 * (int64_t)N + t->n_pv + 2 * (int64_t)t->n_slack;
    if (n_var >= (1ll << 31) || 2 * (int64_t)t->n_line >= (1ll << 31))
        return invalid("network too large for 32-bit indices");
    return PF_OK;
}

// Processing order of the batched kernels' ordinary buses: the preorder of a
// spanning forest or the bus order.  The preorder removes most re-reads of
// neighbour state rows (ncu, DRAM reads per launch: config 3 804 -> 683 MB,
// config 4 879 -> 633 MB) but turns the sequential first reads of a bus's own
// rows into random 256-byte reads, so it pays where one 32-scenario block's
// state rows crowd L2 (B200: config 4, 110 MB of rows, 0.535-0.538 ->
// 0.512-0.513 ms) and not where they fit well (config 3, 37 MB: 0.570-0.574
// -> 0.575-0.576 ms).  PF_ORDER=tree|bus forces one (read once per process).
static bool tree_order(int64_t n_var) {
    static const int v = [] {
        const char* e = getenv("PF_ORDER");
        return !e ? 0 : std::strcmp(e, "bus") == 0 ? 1 : std::strcmp(e, "tree") == 0 ? 2 : 0;
    }();
    return v ? v == 2 : n_var * PF_LANES * 8 > (64ll << 20);
}

#define PF_TRY(call)                                               \
    do {                                                           \
        cudaError_t _e = (call);                                   \
        if (_e != cudaSuccess) {                                   \
            free_plan(P);                                          \
            return cuda_fail(_e, #call);                           \
        }                                                          \
    } while (0)

int build(const pf_topology* t, pf_plan** out) {
    pf_plan* P = new pf_plan();
    DevicePlan& d = P->d;
    d.N = t->n_bus; d.L = t->n_line; d.P = t->n_pq; d.G = t->n_pv; d.S = t->n_slack;
    d.H = t->n_shunt;
    d.n_gen = d.G + d.S;
    d.n_var = 2 * d.N + d.G + 2 * d.S;
    d.n_inc = 2 * d.L;
    const int32_t N = d.N, L = d.L, n_inc = d.n_inc, n_var = d.n_var;
    cudaStream_t st;
    PF_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard { cudaStream_t s; ~StreamGuard() { cudaStreamDestroy(s); } } sg{st};
    Scratch S;

    // uploads (branch-indexed SoA + device groups)
    PF_TRY(upload(P, &d.bus_h, t->bus_h, L, st));
    PF_TRY(upload(P, &d.bus_k, t->bus_k, L, st));
    PF_TRY(upload(P, &d.gl, t->gl, L, st));
    PF_TRY(upload(P, &d.bl, t->bl, L, st));
    PF_TRY(upload(P, &d.gl2, t->gl2, L, st));
    PF_TRY(upload(P, &d.bl2, t->bl2, L, st));
    PF_TRY(upload(P, &d.gsh, t->g_self_h, L, st));
    PF_TRY(upload(P, &d.bsh, t->b_self_h, L, st));
    PF_TRY(upload(P, &d.gsk, t->g_self_k, L, st));
    PF_TRY(upload(P, &d.bsk, t->b_self_k, L, st));
    PF_TRY(upload(P, &d.pq_bus, t->pq_bus, d.P, st));
    PF_TRY(upload(P, &d.pq_p0, t->pq_p0, d.P, st));
    PF_TRY(upload(P, &d.pq_q0, t->pq_q0, d.P, st));
    PF_TRY(upload(P, &d.pv_bus, t->pv_bus, d.G, st));
    PF_TRY(upload(P, &d.pv_p0, t->pv_p0, d.G, st));
    PF_TRY(upload(P, &d.pv_v0, t->pv_v0, d.G, st));
    PF_TRY(upload(P, &d.pv_qg, t->pv_qg, d.G, st));
    PF_TRY(upload(P, &d.sl_bus, t->sl_bus, d.S, st));
    PF_TRY(upload(P, &d.sl_v0, t->sl_v0, d.S, st));
    PF_TRY(upload(P, &d.sl_th0, t->sl_th0, d.S, st));
    PF_TRY(upload(P, &d.sl_qg, t->sl_qg, d.S, st));
    PF_TRY(upload(P, &d.sl_ps, t->sl_ps, d.S, st));
    PF_TRY(upload(P, &d.sh_bus, t->sh_bus, d.H, st));
    PF_TRY(upload(P, &d.sh_g, t->sh_g, d.H, st));
    PF_TRY(upload(P, &d.sh_b, t->sh_b, d.H, st));

    const int bus_bits = nbits((uint64_t)N + 1);
    size_t tmp_bytes = 0;
    void* tmp = nullptr;
    auto ensure_tmp = [&](size_t need) -> cudaError_t {
        if (need <= tmp_bytes) return cudaSuccess;
        cudaError_t e = S.alloc((char**)&tmp, (int64_t)need);
        if (e == cudaSuccess) tmp_bytes = need;
        return e;
    };

    // 1. incidence lists: stable sort of [h-side | k-side] by bus
    uint32_t *ikeys, *ikeys_s;
    int32_t *ivals, *ivals_s;
    PF_TRY(S.alloc(&ikeys, n_inc)); PF_TRY(S.alloc(&ikeys_s, n_inc));
    PF_TRY(S.alloc(&ivals, n_inc)); PF_TRY(S.alloc(&ivals_s, n_inc));
    if (n_inc) {
        k_iota_keys<<<grid_for(n_inc, 256), 256, 0, st>>>(n_inc, d.bus_h, L, d.bus_k, L, nullptr, 0,
                                                          nullptr, ikeys, ivals);
        size_t need = 0;
        PF_TRY(cub::DeviceRadixSort::SortPairs(nullptr, need, ikeys, ikeys_s, ivals, ivals_s,
                                               n_inc, 0, bus_bits, st));
        PF_TRY(ensure_tmp(need));
        PF_TRY(cub::DeviceRadixSort::SortPairs(tmp, need, ikeys, ikeys_s, ivals, ivals_s, n_inc,
                                               0, bus_bits, st));
    }
    int32_t* inc_ptr;
    PF_TRY(owned_alloc(P, &inc_ptr, N + 1));
    k_lower_bound_u32<<<grid_for(N + 1, 256), 256, 0, st>>>(ikeys_s, n_inc, N, inc_ptr);
    d.inc_ptr = inc_ptr;
    int4* meta;
    double4* coef;
    PF_TRY(owned_alloc(P, &meta, n_inc));
    PF_TRY(owned_alloc(P, &coef, n_inc));
    if (n_inc)
        k_inc_records<<<grid_for(n_inc, 256), 256, 0, st>>>(L, ivals_s, d.bus_h, d.bus_k, d.gl, d.bl,
                                                            d.gl2, d.bl2, d.gsh, d.bsh, d.gsk,
                                                            d.bsk, meta, coef);
    d.inc_meta = meta;
    d.inc_coef = coef;

    // 2. closed neighbourhoods: sort (bus, neighbour) pairs, dedupe, rank
    const int64_t m = (int64_t)n_inc + N;
    unsigned long long *nkeys, *nkeys_s;
    int32_t *nvals, *nvals_s, *head, *q;
    PF_TRY(S.alloc(&nkeys, m)); PF_TRY(S.alloc(&nkeys_s, m));
    PF_TRY(S.alloc(&nvals, m)); PF_TRY(S.alloc(&nvals_s, m));
    PF_TRY(S.alloc(&head, m)); PF_TRY(S.alloc(&q, m));
    int32_t *ubase, *uend, *ucol, *pos_i;
    PF_TRY(S.alloc(&ubase, N)); PF_TRY(S.alloc(&uend, N));
    PF_TRY(S.alloc(&ucol, m)); PF_TRY(S.alloc(&pos_i, N));
    PF_TRY(cudaMemsetAsync(ubase, 0, sizeof(int32_t) * (size_t)(N > 0 ? N : 1), st));
    PF_TRY(cudaMemsetAsync(uend, 0, sizeof(int32_t) * (size_t)(N > 0 ? N : 1), st));
    PF_TRY(cudaMemsetAsync(pos_i, 0, sizeof(int32_t) * (size_t)(N > 0 ? N : 1), st));
    if (m) {
        k_nbr_pairs<<<grid_for(m, 256), 256, 0, st>>>(N, n_inc, meta, inc_ptr, ikeys_s, nkeys,
                                                      nvals);
        size_t need = 0;
        PF_TRY(cub::DeviceRadixSort::SortPairs(nullptr, need, nkeys, nkeys_s, nvals, nvals_s,
                                               (int)m, 0, 64, st));
        PF_TRY(ensure_tmp(need));
        PF_TRY(cub::DeviceRadixSort::SortPairs(tmp, need, nkeys, nkeys_s, nvals, nvals_s, (int)m,
                                               0, 64, st));
        k_heads<<<grid_for(m, 256), 256, 0, st>>>(m, nkeys_s, head);
        need = 0;
        PF_TRY(cub::DeviceScan::InclusiveSum(nullptr, need, head, q, (int)m, st));
        PF_TRY(ensure_tmp(need));
        PF_TRY(cub::DeviceScan::InclusiveSum(tmp, need, head, q, (int)m, st));
        k_seg_bounds<<<grid_for(m, 256), 256, 0, st>>>(m, nkeys_s, q, ubase, uend);
        k_nbr_ranks<<<grid_for(m, 256), 256, 0, st>>>(m, n_inc, nkeys_s, nvals_s, head, q, ubase,
                                                      ucol, meta, pos_i);
    }

    // 3. per-bus device lists in (bus, PQ < PV < Slack < Shunt, index) order
    const int64_t n_dev = (int64_t)d.P + d.G + d.S + d.H;
    uint32_t *dkeys, *dkeys_s;
    int32_t *dvals, *dvals_s;
    PF_TRY(S.alloc(&dkeys, n_dev)); PF_TRY(S.alloc(&dkeys_s, n_dev));
    PF_TRY(S.alloc(&dvals, n_dev)); PF_TRY(S.alloc(&dvals_s, n_dev));
    if (n_dev) {
        k_iota_keys<<<grid_for(n_dev, 256), 256, 0, st>>>(n_dev, d.pq_bus, d.P, d.pv_bus, d.G,
                                                          d.sl_bus, d.S, d.sh_bus, dkeys, dvals);
        size_t need = 0;
        PF_TRY(cub::DeviceRadixSort::SortPairs(nullptr, need, dkeys, dkeys_s, dvals, dvals_s,
                                               (int)n_dev, 0, bus_bits, st));
        PF_TRY(ensure_tmp(need));
        PF_TRY(cub::DeviceRadixSort::SortPairs(tmp, need, dkeys, dkeys_s, dvals, dvals_s,
                                               (int)n_dev, 0, bus_bits, st));
    }
    int32_t* dev_ptr;
    PF_TRY(owned_alloc(P, &dev_ptr, N + 1));
    k_lower_bound_u32<<<grid_for(N + 1, 256), 256, 0, st>>>(dkeys_s, n_dev, N, dev_ptr);
    d.dev_ptr = dev_ptr;
    DevGroups dg{d.P, d.G, d.S, d.H, d.pv_qg, d.sl_qg, d.sl_ps};

    // 4. row lengths -> indptr (int64 scan, checked against 2^31)
    int64_t *rowlen, *indptr64;
    PF_TRY(S.alloc(&rowlen, n_var + 1)); PF_TRY(S.alloc(&indptr64, n_var + 1));
    PF_TRY(cudaMemsetAsync(rowlen, 0, sizeof(int64_t) * (size_t)(n_var + 1), st));
    if (n_var)
        k_row_len<<<grid_for(n_var, 256), 256, 0, st>>>(N, d.n_gen, d.S, ubase, uend, inc_ptr,
                                                        dev_ptr, dvals_s, dg, rowlen);
    {
        size_t need = 0;
        PF_TRY(cub::DeviceScan::ExclusiveSum(nullptr, need, rowlen, indptr64, n_var + 1, st));
        PF_TRY(ensure_tmp(need));
        PF_TRY(cub::DeviceScan::ExclusiveSum(tmp, need, rowlen, indptr64, n_var + 1, st));
    }
    int64_t nnz64 = 0;
    PF_TRY(cudaMemcpyAsync(&nnz64, indptr64 + n_var, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    PF_TRY(cudaStreamSynchronize(st));
    if (nnz64 >= (1ll << 31) / PF_LANES) {
        free_plan(P);
        return invalid("Jacobian pattern too large (nnz = " + std::to_string(nnz64) + ")");
    }
    d.nnz = (int32_t)nnz64;

    // 5. fill indices, bus rows, device entries
    int32_t *indices, *indptr;
    int4 *bus_row, *dev_list;
    int32_t* gen_row_pos;
    PF_TRY(owned_alloc(P, &indices, d.nnz));
    PF_TRY(owned_alloc(P, &indptr, n_var + 1));
    PF_TRY(owned_alloc(P, &bus_row, 2 * (int64_t)N));
    PF_TRY(owned_alloc(P, &dev_list, n_dev));
    PF_TRY(owned_alloc(P, &gen_row_pos, d.n_gen + d.S));
    if (N)
        k_fill<<<grid_for(N, 128), 128, 0, st>>>(N, d.n_gen, ubase, uend, inc_ptr, ucol, pos_i,
                                                 dev_ptr, dvals_s, dg, indptr64, indices,
                                                 bus_row, dev_list, gen_row_pos);
    k_i64_to_i32<<<grid_for(n_var + 1, 256), 256, 0, st>>>(n_var + 1, indptr64, indptr);
    d.csr_indices = indices;
    d.csr_indptr = indptr;
    d.bus_row = bus_row;
    d.dev_list = dev_list;
    d.gen_row_pos = gen_row_pos;

    // 6. CSC permutation: sort entries by (col, row)
    const int64_t nnz = d.nnz;
    unsigned long long *ckeys, *ckeys_s;
    int32_t *cvals, *perm, *csc_indices, *csc_indptr;
    PF_TRY(S.alloc(&ckeys, nnz)); PF_TRY(S.alloc(&ckeys_s, nnz));
    PF_TRY(S.alloc(&cvals, nnz));
    PF_TRY(owned_alloc(P, &perm, nnz));
    PF_TRY(owned_alloc(P, &csc_indices, nnz));
    PF_TRY(owned_alloc(P, &csc_indptr, n_var + 1));
    if (nnz) {
        k_csr_keys<<<grid_for(n_var, 256), 256, 0, st>>>(n_var, indptr64, indices, ckeys, cvals);
        const int key_bits = 32 + nbits((uint64_t)n_var + 1);
        size_t need = 0;
        PF_TRY(cub::DeviceRadixSort::SortPairs(nullptr, need, ckeys, ckeys_s, cvals, perm,
                                               (int)nnz, 0, key_bits, st));
        PF_TRY(ensure_tmp(need));
        PF_TRY(cub::DeviceRadixSort::SortPairs(tmp, need, ckeys, ckeys_s, cvals, perm, (int)nnz,
                                               0, key_bits, st));
        k_csc_rows<<<grid_for(nnz, 256), 256, 0, st>>>(nnz, ckeys_s, csc_indices);
    }
    k_lower_bound_hi<<<grid_for(n_var + 1, 256), 256, 0, st>>>(ckeys_s, nnz, n_var, csc_indptr);
    d.csc_perm = perm;
    d.csc_indices = csc_indices;
    d.csc_indptr = csc_indptr;

    // max degree (informational)
    std::vector<int32_t> hptr(N + 1);
    PF_TRY(cudaMemcpyAsync(hptr.data(), inc_ptr, sizeof(int32_t) * (size_t)(N + 1),
                           cudaMemcpyDeviceToHost, st));
    PF_TRY(cudaStreamSynchronize(st));
    PF_TRY(cudaGetLastError());
    int32_t md = 0;
    for (int32_t i = 0; i < N; ++i) md = std::max(md, hptr[i + 1] - hptr[i]);
    P->max_deg = md;
    // batched processing order (the identity when there are no hubs)
    std::vector<int32_t> order;
    {
        // Hubs go into the first rounds of the staged kernel's schedule,
        // spread so that every CTA (hence every SM) and every warp gets at
        // most one more than the others: CTA c processes groups c, c + G,
        // ... of WS_W slots (G = resident CTAs), so hub h takes CTA h mod G,
        // warp (h / G) mod WS_W, round h / (G WS_W).  Heaviest hubs first.
        // Buses of ordinary degree fill the remaining slots in bus order.
        std::vector<int32_t> hubs;
        for (int32_t i = 0; i < N; ++i)
            if (hptr[i + 1] - hptr[i] >= HUB_DEG) hubs.push_back(i);
        std::stable_sort(hubs.begin(), hubs.end(), [&](int32_t a, int32_t b) {
            return hptr[a + 1] - hptr[a] > hptr[b + 1] - hptr[b];
        });
        d.n_hubs = (int32_t)hubs.size();
        int dev = 0, sms = 0;
        PF_TRY(cudaGetDevice(&dev));
        PF_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const int64_t n_groups = (N + WS_W - 1) / WS_W;
        const int64_t G = std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * WS_MINB, n_groups));
        order.assign(N, -1);
        std::vector<char> taken((size_t)n_groups * WS_W, 0);
        for (int64_t h = 0; h < (int64_t)hubs.size(); ++h) {
            const int64_t c = h % G, w = (h / G) % WS_W, r = h / (G * WS_W);
            int64_t slot = (r * G + c) * WS_W + w;
            while (slot < N && taken[slot]) ++slot;   // (not reached for in-range rounds)
            if (slot >= N) {                            // degenerate tiny grids
                slot = 0;
                while (taken[slot]) ++slot;
            }
            taken[slot] = 1;
            order[slot] = hubs[h];
        }
        // Buses of ordinary degree fill the remaining slots in bus order or
        // (tree_order) in the preorder of a breadth-first spanning forest whose
        // children are visited smallest subtree first.  At any time
        // the kernel works on a window of G WS_W consecutive slots, so a
        // bus's state rows are in L2 for a neighbour's item when the two
        // slots are close; in this order a tree branch (N - 1 of the
        // branches of a connected grid) is 1 + the smaller siblings'
        // subtrees apart.
        std::vector<int32_t> seq;
        seq.reserve(N);
        if (tree_order(d.n_var)) {
            std::vector<int4> hm(n_inc);
            if (n_inc)
                PF_TRY(cudaMemcpy(hm.data(), d.inc_meta, sizeof(int4) * (size_t)n_inc,
                                  cudaMemcpyDeviceToHost));
            std::vector<int32_t> par(N, -2), bfs, sz(N, 1), cptr(N + 2, 0), kids(N);
            bfs.reserve(N);
            // (the forest does not pass through hubs: they are placed in the
            // first rounds whatever their rank, so a bus adopted by a hub would
            // lose the one neighbour that can be near it)
            auto is_hub = [&](int32_t i) { return hptr[i + 1] - hptr[i] >= HUB_DEG; };
            for (int32_t r = 0; r < N; ++r) {
                if (par[r] != -2) continue;
                par[r] = -1;
                bfs.push_back(r);
                if (is_hub(r)) continue;
                for (size_t q = bfs.size() - 1; q < bfs.size(); ++q) {
                    const int32_t u = bfs[q];
                    for (int32_t e = hptr[u]; e < hptr[u + 1]; ++e) {
                        const int32_t v = hm[e].x;
                        if (v < 0 || v >= N || par[v] != -2 || is_hub(v)) continue;
                        par[v] = u;
                        bfs.push_back(v);
                    }
                }
            }
            for (int64_t q = N - 1; q >= 0; --q)
                if (par[bfs[q]] >= 0) sz[par[bfs[q]]] += sz[bfs[q]];
            for (int32_t v = 0; v < N; ++v) cptr[(par[v] >= 0 ? par[v] : N) + 1]++;
            for (int32_t u = 0; u <= N; ++u) cptr[u + 1] += cptr[u];
            {
                std::vector<int32_t> cur(cptr.begin(), cptr.end() - 1);
                for (int32_t v = 0; v < N; ++v) kids[cur[par[v] >= 0 ? par[v] : N]++] = v;
            }
            // cptr[u] .. cptr[u + 1]: children of u (u = N: the roots), by bus
            for (int32_t u = 0; u < N; ++u)
                if (cptr[u + 1] - cptr[u] > 1)   // (ties by bus: deterministic)
                    std::sort(kids.begin() + cptr[u], kids.begin() + cptr[u + 1],
                              [&](int32_t a, int32_t b) {
                                  return sz[a] != sz[b] ? sz[a] < sz[b] : a < b;
                              });
            std::vector<int32_t> stack(kids.rbegin(), kids.rbegin() + (cptr[N + 1] - cptr[N]));   // roots
            while (!stack.empty()) {
                const int32_t u = stack.back();
                stack.pop_back();
                seq.push_back(u);
                for (int32_t c = cptr[u + 1]; c-- > cptr[u];) stack.push_back(kids[c]);
            }
        } else {
            for (int32_t i = 0; i < N; ++i) seq.push_back(i);
        }
        int32_t next = 0;
        for (const int32_t i : seq) {
            if (hptr[i + 1] - hptr[i] >= HUB_DEG) continue;
            while (taken[next]) ++next;
            taken[next] = 1;
            order[next] = i;
        }
        // (kept as a load even when it is the identity: measured faster on
        // B200 than a conditional bypass, 0.738 vs 0.776 ms at config 3)
        int32_t* bus_order;
        PF_TRY(owned_alloc(P, &bus_order, N));
        PF_TRY(cudaMemcpy(bus_order, order.data(), sizeof(int32_t) * (size_t)N,
                          cudaMemcpyHostToDevice));
        d.bus_order = bus_order;
    }
    // single-grid chunks (k_eval_single): consecutive buses while the
    // incidences, the Jacobian values of rows g_p / g_q and the parallel-branch
    // slots fit the shared-memory caps; a lone bus over a cap is flagged SG_BIG
    {
        std::vector<int4> hmeta(n_inc), hrow(2 * (size_t)N);
        std::vector<int64_t> hip(n_var + 1);
        PF_TRY(cudaMemcpy(hmeta.data(), meta, sizeof(int4) * (size_t)n_inc, cudaMemcpyDeviceToHost));
        PF_TRY(cudaMemcpy(hrow.data(), bus_row, sizeof(int4) * 2 * (size_t)N,
                          cudaMemcpyDeviceToHost));
        PF_TRY(cudaMemcpy(hip.data(), indptr64, sizeof(int64_t) * (size_t)(n_var + 1),
                          cudaMemcpyDeviceToHost));
        std::vector<int4> chunks, sginc(n_inc, make_int4(0, 0, 0, 0));
        auto jrows = [&](int32_t i) {
            return (hip[i + 1] - hip[i]) + (hip[N + i + 1] - hip[N + i]);
        };
        auto ndups = [&](int32_t i) {
            int32_t c = 0;
            for (int32_t e = hptr[i]; e < hptr[i + 1]; ++e) c += !(hmeta[e].z & SOLO);
            return c;
        };
        for (int32_t b0 = 0; b0 < N;) {
            int32_t b1 = b0;
            int64_t ninc = 0, nj = 0, ndup = 0;
            while (b1 < N && b1 - b0 < SG_CAP_BUS) {
                const int64_t di = hptr[b1 + 1] - hptr[b1], ji = jrows(b1), ui = ndups(b1);
                if (b1 > b0 && (ninc + di > SG_CAP_INC || nj + ji > SG_CAP_J ||
                                ndup + ui > SG_CAP_DUP))
                    break;
                ninc += di;
                nj += ji;
                ndup += ui;
                ++b1;
            }
            const bool big = ninc > SG_CAP_INC || nj > SG_CAP_J || ndup > SG_CAP_DUP;
            const int32_t p0 = (int32_t)hip[b0], p1 = (int32_t)hip[b1];
            const int32_t q0 = (int32_t)hip[N + b0], q1 = (int32_t)hip[N + b1];
            chunks.push_back(make_int4(b0, b1 | (big ? SG_BIG : 0), hptr[b0], hptr[b1]));
            chunks.push_back(make_int4(p0, p1, q0, q1));
            int32_t slot = 0;
            for (int32_t e = hptr[b0]; !big && e < hptr[b1]; ++e) {
                const int4 m = hmeta[e];
                const int32_t own = m.w, pos = m.z & POS_MASK;
                const int4 r = hrow[2 * (size_t)own];
                int32_t f = (own - b0) | (m.z & (SOLO | KSIDE));
                if (!(m.z & SOLO)) f |= slot++ << SG_DUP_SHIFT;
                sginc[e] = make_int4(m.x, f, r.x + pos - p0, r.y + pos - q0);
            }
            b0 = b1;
        }
        int4 *dchunk, *dinc;
        unsigned long long* acc;
        unsigned int* cnt;
        PF_TRY(owned_alloc(P, &dchunk, (int64_t)chunks.size()));
        PF_TRY(owned_alloc(P, &dinc, n_inc));
        PF_TRY(owned_alloc(P, &acc, 1));
        PF_TRY(owned_alloc(P, &cnt, 1));
        if (!chunks.empty())
            PF_TRY(cudaMemcpy(dchunk, chunks.data(), sizeof(int4) * chunks.size(),
                              cudaMemcpyHostToDevice));
        if (n_inc)
            PF_TRY(cudaMemcpy(dinc, sginc.data(), sizeof(int4) * (size_t)n_inc,
                              cudaMemcpyHostToDevice));
        PF_TRY(cudaMemset(acc, 0, sizeof(unsigned long long)));
        PF_TRY(cudaMemset(cnt, 0, sizeof(unsigned int)));
        d.sg_chunks = (int32_t)(chunks.size() / 2);
        P->sg_big = 0;
        for (size_t c = 0; c < chunks.size(); c += 2) P->sg_big += (chunks[c].y & SG_BIG) != 0;
        d.sg_chunk = dchunk;
        d.sg_inc = dinc;
        d.sg_acc = acc;
        d.sg_count = cnt;
    }
    // warp-specialised batched kernel: per bus (processing order) a packet of
    // its header / staged incidence and device records and a stage record
    // naming the scenario rows to copy (pf_internal.cuh, WS_ROWS)
    {
        std::vector<int4> hmeta(n_inc), hrow(2 * (size_t)N), hdev;
        std::vector<double4> hcoef(n_inc);
        const int32_t n_dev = d.P + d.G + d.S + d.H;
        hdev.resize(n_dev);
        if (n_inc) {
            PF_TRY(cudaMemcpy(hmeta.data(), d.inc_meta, sizeof(int4) * (size_t)n_inc,
                              cudaMemcpyDeviceToHost));
            PF_TRY(cudaMemcpy(hcoef.data(), d.inc_coef, sizeof(double4) * (size_t)n_inc,
                              cudaMemcpyDeviceToHost));
        }
        if (n_dev)
            PF_TRY(cudaMemcpy(hdev.data(), d.dev_list, sizeof(int4) * (size_t)n_dev,
                              cudaMemcpyDeviceToHost));
        PF_TRY(cudaMemcpy(hrow.data(), d.bus_row, sizeof(int4) * 2 * (size_t)N,
                          cudaMemcpyDeviceToHost));
        std::vector<int4> pkt;
        std::vector<int32_t> rec((size_t)N * WS_REC_WORDS, -1);
        pkt.reserve((size_t)N * 12);
        auto code = [](int32_t arr, int64_t e) { return (int32_t)((arr << 29) | (int32_t)e); };
        auto d2 = [](double a, double b) {
            int4 u;
            long long x, y;
            std::memcpy(&x, &a, 8);
            std::memcpy(&y, &b, 8);
            u.x = (int32_t)(x & 0xffffffff); u.y = (int32_t)(x >> 32);
            u.z = (int32_t)(y & 0xffffffff); u.w = (int32_t)(y >> 32);
            return u;
        };
        for (int32_t s = 0; s < N; ++s) {
            const int32_t i = order[s];
            const int4 h0 = hrow[2 * (size_t)i], h1 = hrow[2 * (size_t)i + 1];
            const int32_t deg = h1.y - h1.x, ndev = h1.w - h1.z;
            const int32_t nv = std::min(ndev, WS_MAXDEV);
            const int32_t ni = std::min({deg, WS_MAXINC, (WS_ROWS - 2 - 2 * nv) / 2});
            int32_t* r = &rec[(size_t)s * WS_REC_WORDS];
            const int64_t off = (int64_t)pkt.size();
            if (off >= (1ll << 31)) {
                free_plan(P);
                return invalid("staged packets exceed 2^31 units");
            }
            pkt.push_back(h0);
            pkt.push_back(h1);
            pkt.push_back(make_int4(ni, nv, i, 0));
            for (int32_t q = 0; q < ni; ++q) pkt.push_back(hmeta[h1.x + q]);
            for (int32_t q = 0; q < ni; ++q) {
                const double4 c = hcoef[h1.x + q];
                pkt.push_back(d2(c.x, c.y));
                pkt.push_back(d2(c.z, c.w));
            }
            int32_t* rows = r + 2;
            rows[0] = code(0, i);
            rows[1] = code(0, (int64_t)N + i);
            for (int32_t q = 0; q < ni; ++q) {
                const int32_t j = hmeta[h1.x + q].x;
                rows[2 + 2 * q] = code(0, j);
                rows[3 + 2 * q] = code(0, (int64_t)N + j);
            }
            for (int32_t u = 0; u < nv; ++u) pkt.push_back(hdev[h1.z + u]);
            for (int32_t u = 0; u < nv; ++u) {
                const int4 dv = hdev[h1.z + u];
                const int32_t k = dv.y;
                int32_t* ra = rows + 2 + 2 * ni + 2 * u;
                double c = 0.0, dd = 0.0;
                if (dv.x == DEV_PQ) {          // a = pq_p, b = pq_q; base p0, q0
                    ra[0] = code(1, k);
                    ra[1] = code(2, k);
                    c = t->pq_p0[k];
                    dd = t->pq_q0[k];
                } else if (dv.x == DEV_PV) {   // a = pv_p, b = Q_g; v0, base p0
                    ra[0] = code(3, k);
                    ra[1] = code(0, 2 * (int64_t)N + k);
                    c = t->pv_v0[k];
                    dd = t->pv_p0[k];
                } else if (dv.x == DEV_SLACK) {  // a = P_s, b = Q_g; v0, theta0
                    ra[0] = code(0, 2 * (int64_t)N + d.n_gen + k);
                    ra[1] = code(0, 2 * (int64_t)N + d.G + k);
                    c = t->sl_v0[k];
                    dd = t->sl_th0[k];
                } else {                       // shunt: g, b
                    c = t->sh_g[k];
                    dd = t->sh_b[k];
                }
                pkt.push_back(d2(c, dd));
            }
            r[0] = (int32_t)off;
            r[1] = (int32_t)(pkt.size() - off) | ((2 + 2 * ni + 2 * nv) << 16);
        }
        int4 *dpkt, *drec;
        PF_TRY(owned_alloc(P, &dpkt, std::max<int64_t>((int64_t)pkt.size(), 1)));
        PF_TRY(owned_alloc(P, &drec, std::max<int64_t>((int64_t)N * WS_REC_WORDS / 4, 1)));
        if (!pkt.empty())
            PF_TRY(cudaMemcpy(dpkt, pkt.data(), sizeof(int4) * pkt.size(), cudaMemcpyHostToDevice));
        if (N)
            PF_TRY(cudaMemcpy(drec, rec.data(), sizeof(int32_t) * rec.size(),
                              cudaMemcpyHostToDevice));
        d.ws_pkt = dpkt;
        d.ws_rec = drec;
        // Packets and records are re-read by every 32-scenario block; they stay
        // in L2 across blocks (evict-last) when they and one block's state rows
        // take at most half of it.  B200, ms per launch: config 3 (19 MB +
        // 37 MB) 0.595 -> 0.572; config 4 (51 MB + 110 MB, not kept) would
        // lose 0.533 -> 0.537.
        const int64_t keep = (int64_t)pkt.size() * 16 + (int64_t)N * WS_REC_WORDS * 4 +
                             (int64_t)d.n_var * PF_LANES * 8;
        d.ws_keep = keep <= (64ll << 20) ? 1 : 0;
    }
    count_launch(12);
    *out = P;
    return PF_OK;
}

#undef PF_TRY

}  // namespace
}  // namespace pf

// =============================== C ABI ========================================

using pf::DevicePlan;

extern "C" {

const char* pf_last_error(void) { return pf::g_err.c_str(); }

int pf_version(void) { return 1; }

int64_t pf_launch_count(void) { return pf::g_launches.load(); }

int64_t pf_alloc_count(void) { return pf::g_allocs.load(); }

int pf_host_register(void* ptr, size_t bytes) {
    if (!ptr || !bytes) return pf::invalid("NULL or empty host range");
    const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterDefault);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
        cudaGetLastError();   // clear the sticky-free error state
        return PF_OK;
    }
    PF_CUDA(e);
    return PF_OK;
}

int pf_host_unregister(void* ptr) {
    if (!ptr) return pf::invalid("NULL host pointer");
    const cudaError_t e = cudaHostUnregister(ptr);
    if (e == cudaErrorHostMemoryNotRegistered) {
        cudaGetLastError();
        return PF_OK;
    }
    PF_CUDA(e);
    return PF_OK;
}

int pf_plan_create(const pf_topology* topo, pf_plan** out) {
    if (!out) return pf::invalid("out is NULL");
    *out = nullptr;
    int rc = pf::validate(topo);
    if (rc) return rc;
    return pf::build(topo, out);
}

int pf_plan_destroy(pf_plan* plan) {
    pf::free_plan(plan);
    return PF_OK;
}

int pf_plan_dims(const pf_plan* p, int64_t* dims) {
    if (!p || !dims) return pf::invalid("NULL argument");
    const DevicePlan& d = p->d;
    dims[PF_DIM_NBUS] = d.N;
    dims[PF_DIM_NLINE] = d.L;
    dims[PF_DIM_NVAR] = d.n_var;
    dims[PF_DIM_NNZ] = d.nnz;
    dims[PF_DIM_NPQ] = d.P;
    dims[PF_DIM_NPV] = d.G;
    dims[PF_DIM_NSLACK] = d.S;
    dims[PF_DIM_NSHUNT] = d.H;
    dims[PF_DIM_NINC] = d.n_inc;
    dims[PF_DIM_MAXDEG] = p->max_deg;
    dims[PF_DIM_SG_CHUNKS] = d.sg_chunks;
    dims[PF_DIM_SG_BIG] = p->sg_big;
    return PF_OK;
}

int pf_plan_pattern_csr(const pf_plan* p, int32_t* indptr, int32_t* indices) {
    if (!p || !indptr || !indices) return pf::invalid("NULL argument");
    PF_CUDA(cudaMemcpy(indptr, p->d.csr_indptr, sizeof(int32_t) * (size_t)(p->d.n_var + 1),
                       cudaMemcpyDeviceToHost));
    if (p->d.nnz)
        PF_CUDA(cudaMemcpy(indices, p->d.csr_indices, sizeof(int32_t) * (size_t)p->d.nnz,
                           cudaMemcpyDeviceToHost));
    return PF_OK;
}

int pf_plan_pattern_csc(const pf_plan* p, int32_t* csc_indptr, int32_t* csc_indices,
                        int32_t* perm) {
    if (!p) return pf::invalid("NULL plan");
    if (csc_indptr)
        PF_CUDA(cudaMemcpy(csc_indptr, p->d.csc_indptr, sizeof(int32_t) * (size_t)(p->d.n_var + 1),
                           cudaMemcpyDeviceToHost));
    if (csc_indices && p->d.nnz)
        PF_CUDA(cudaMemcpy(csc_indices, p->d.csc_indices, sizeof(int32_t) * (size_t)p->d.nnz,
                           cudaMemcpyDeviceToHost));
    if (perm && p->d.nnz)
        PF_CUDA(cudaMemcpy(perm, p->d.csc_perm, sizeof(int32_t) * (size_t)p->d.nnz,
                           cudaMemcpyDeviceToHost));
    return PF_OK;
}

int pf_eval(const pf_plan* p, const double* y, double* g, double* jval, double* norm,
            void* stream) {
    if (!p) return pf::invalid("NULL plan");
    if (!y && (g || jval || norm)) return pf::invalid("y is NULL");
    PF_CUDA(pf::launch_eval_single(p->d, y, g, jval, norm, (cudaStream_t)stream));
    return PF_OK;
}

int pf_eval_batched(const pf_plan* p, int32_t K, const double* y, const double* pq_p,
                    const double* pq_q, const double* pv_p, const int32_t* outage, double* g,
                    double* jval, double* norms, void* stream) {
    if (!p) return pf::invalid("NULL plan");
    if (K < 0) return pf::invalid("K must be >= 0");
    if (K > 0 && !y && (g || jval || norms)) return pf::invalid("y is NULL");
    if ((int64_t)(K + PF_LANES - 1) / PF_LANES > 65535) return pf::invalid("K too large");
    PF_CUDA(pf::launch_eval_batched(p->d, K, y, pq_p, pq_q, pv_p, outage, g, jval, norms,
                                    (cudaStream_t)stream));
    return PF_OK;
}

int pf_batch_unblock(int32_t K, int32_t n_e, const double* src, double* dst, double alpha,
                     void* stream) {
    if (K < 0 || n_e < 0) return pf::invalid("negative size");
    if ((K > 0 && n_e > 0) && (!src || !dst)) return pf::invalid("NULL argument");
    PF_CUDA(pf::launch_batch_unblock(K, n_e, src, dst, alpha, (cudaStream_t)stream));
    return PF_OK;
}

int pf_batch_update(int32_t K, int32_t n_e, double* y, const double* dx, const int32_t* active,
                    void* stream) {
    if (K < 0 || n_e < 0) return pf::invalid("negative size");
    if ((K > 0 && n_e > 0) && (!y || !dx)) return pf::invalid("NULL argument");
    PF_CUDA(pf::launch_batch_update(K, n_e, y, dx, active, (cudaStream_t)stream));
    return PF_OK;
}

int pf_jac_to_csc(const pf_plan* p, int32_t K, const double* jcsr, double* jcsc, void* stream) {
    if (!p || !jcsr || !jcsc) return pf::invalid("NULL argument");
    PF_CUDA(pf::launch_jac_to_csc(p->d, K, jcsr, jcsc, (cudaStream_t)stream));
    return PF_OK;
}

int pf_eval_host(pf_plan* p, const double* y, double* g, double* jcsc, double* norm) {
    if (!p || !y) return pf::invalid("NULL argument");
    const DevicePlan& d = p->d;
    if (!p->s_stream) {
        PF_CUDA(cudaStreamCreateWithFlags(&p->s_stream, cudaStreamNonBlocking));
        PF_CUDA(pf::dmalloc(&p->s_y, sizeof(double) * (size_t)(d.n_var + 1)));
        PF_CUDA(pf::dmalloc(&p->s_g, sizeof(double) * (size_t)(d.n_var + 1)));
        PF_CUDA(pf::dmalloc(&p->s_j, sizeof(double) * (size_t)(d.nnz + 1)));
        PF_CUDA(pf::dmalloc(&p->s_jc, sizeof(double) * (size_t)(d.nnz + 1)));
        PF_CUDA(pf::dmalloc(&p->s_norm, sizeof(double)));
    }
    cudaStream_t st = p->s_stream;
    PF_CUDA(cudaMemcpyAsync(p->s_y, y, sizeof(double) * (size_t)d.n_var, cudaMemcpyHostToDevice, st));
    PF_CUDA(pf::launch_eval_single(d, p->s_y, g ? p->s_g : nullptr, jcsc ? p->s_j : nullptr,
                                   norm ? p->s_norm : nullptr, st));
    if (g)
        PF_CUDA(cudaMemcpyAsync(g, p->s_g, sizeof(double) * (size_t)d.n_var,
                                cudaMemcpyDeviceToHost, st));
    if (jcsc) {
        PF_CUDA(pf::launch_jac_to_csc(d, 0, p->s_j, p->s_jc, st));
        PF_CUDA(cudaMemcpyAsync(jcsc, p->s_jc, sizeof(double) * (size_t)d.nnz,
                                cudaMemcpyDeviceToHost, st));
    }
    if (norm)
        PF_CUDA(cudaMemcpyAsync(norm, p->s_norm, sizeof(double), cudaMemcpyDeviceToHost, st));
    PF_CUDA(cudaStreamSynchronize(st));
    return PF_OK;
}

int pf_eval_batched_host(pf_plan* p, int32_t K, const double* y, const double* pq_p,
                         const double* pq_q, const double* pv_p, const int32_t* outage,
                         double* g, double* jval, double* norms, int32_t blocks_per_stage,
                         int32_t n_streams) {
    if (!p || !y) return pf::invalid("NULL argument");
    if (K <= 0) return PF_OK;
    if (outage)   // host array: validate (the device paths read no memory for these)
        for (int32_t k = 0; k < K; ++k)
            if (outage[k] < -1 || outage[k] >= p->d.L)
                return pf::invalid("outage index outside [-1, n_line)");
    if (blocks_per_stage < 1) blocks_per_stage = 1;
    if (n_streams < 1) n_streams = 1;
    if (n_streams > 8) n_streams = 8;
    const DevicePlan& d = p->d;
    pf::Staging& b = p->batch;
    if (b.n_streams != n_streams || b.blocks != blocks_per_stage) {
        for (int s = 0; s < b.n_streams; ++s) {
            cudaFree(b.y[s]); cudaFree(b.g[s]); cudaFree(b.j[s]); cudaFree(b.pq_p[s]);
            cudaFree(b.pq_q[s]); cudaFree(b.pv_p[s]); cudaFree(b.outage[s]); cudaFree(b.norms[s]);
            if (b.streams[s]) cudaStreamDestroy(b.streams[s]);
        }
        b = pf::Staging();
        const size_t lanes = (size_t)blocks_per_stage * PF_LANES;
        for (int s = 0; s < n_streams; ++s) {
            PF_CUDA(cudaStreamCreateWithFlags(&b.streams[s], cudaStreamNonBlocking));
            PF_CUDA(pf::dmalloc(&b.y[s], sizeof(double) * lanes * (size_t)d.n_var));
            PF_CUDA(pf::dmalloc(&b.g[s], sizeof(double) * lanes * (size_t)d.n_var));
            PF_CUDA(pf::dmalloc(&b.j[s], sizeof(double) * lanes * (size_t)(d.nnz + 1)));
            PF_CUDA(pf::dmalloc(&b.pq_p[s], sizeof(double) * lanes * (size_t)(d.P + 1)));
            PF_CUDA(pf::dmalloc(&b.pq_q[s], sizeof(double) * lanes * (size_t)(d.P + 1)));
            PF_CUDA(pf::dmalloc(&b.pv_p[s], sizeof(double) * lanes * (size_t)(d.G + 1)));
            PF_CUDA(pf::dmalloc(&b.outage[s], sizeof(int32_t) * lanes));
            PF_CUDA(pf::dmalloc(&b.norms[s], sizeof(double) * lanes));
            b.n_streams = s + 1;
        }
        b.blocks = blocks_per_stage;
    }
    const int64_t nblk = (K + PF_LANES - 1) / PF_LANES;
    const int64_t n_stage = (nblk + blocks_per_stage - 1) / blocks_per_stage;
    for (int64_t st_i = 0; st_i < n_stage; ++st_i) {
        const int s = (int)(st_i % n_streams);
        cudaStream_t st = b.streams[s];
        const int64_t blk0 = st_i * blocks_per_stage;
        const int64_t nb = std::min<int64_t>(blocks_per_stage, nblk - blk0);
        const int64_t k0 = blk0 * PF_LANES;
        const int32_t Kc = (int32_t)std::min<int64_t>(nb * PF_LANES, K - k0);
        const size_t L8 = sizeof(double) * (size_t)PF_LANES;
        PF_CUDA(cudaMemcpyAsync(b.y[s], y + blk0 * d.n_var * PF_LANES, L8 * nb * d.n_var,
                                cudaMemcpyHostToDevice, st));
        if (pq_p)
            PF_CUDA(cudaMemcpyAsync(b.pq_p[s], pq_p + blk0 * d.P * PF_LANES, L8 * nb * d.P,
                                    cudaMemcpyHostToDevice, st));
        if (pq_q)
            PF_CUDA(cudaMemcpyAsync(b.pq_q[s], pq_q + blk0 * d.P * PF_LANES, L8 * nb * d.P,
                                    cudaMemcpyHostToDevice, st));
        if (pv_p)
            PF_CUDA(cudaMemcpyAsync(b.pv_p[s], pv_p + blk0 * d.G * PF_LANES, L8 * nb * d.G,
                                    cudaMemcpyHostToDevice, st));
        if (outage)
            PF_CUDA(cudaMemcpyAsync(b.outage[s], outage + k0, sizeof(int32_t) * (size_t)Kc,
                                    cudaMemcpyHostToDevice, st));
        PF_CUDA(pf::launch_eval_batched(d, Kc, b.y[s], pq_p ? b.pq_p[s] : nullptr,
                                        pq_q ? b.pq_q[s] : nullptr, pv_p ? b.pv_p[s] : nullptr,
                                        outage ? b.outage[s] : nullptr, g ? b.g[s] : nullptr,
                                        jval ? b.j[s] : nullptr, norms ? b.norms[s] : nullptr, st));
        if (g)
            PF_CUDA(cudaMemcpyAsync(g + blk0 * d.n_var * PF_LANES, b.g[s], L8 * nb * d.n_var,
                                    cudaMemcpyDeviceToHost, st));
        if (jval)
            PF_CUDA(cudaMemcpyAsync(jval + blk0 * (int64_t)d.nnz * PF_LANES, b.j[s],
                                    L8 * nb * (size_t)d.nnz, cudaMemcpyDeviceToHost, st));
        if (norms)
            PF_CUDA(cudaMemcpyAsync(norms + k0, b.norms[s], sizeof(double) * (size_t)Kc,
                                    cudaMemcpyDeviceToHost, st));
    }
    for (int s = 0; s < b.n_streams; ++s) PF_CUDA(cudaStreamSynchronize(b.streams[s]));
    return PF_OK;
}

int pf_line_injections(const pf_plan* p, const double* y, double* ph, double* pk, double* qh,
                       double* qk, void* stream) {
    if (!p || !y || !ph || !pk || !qh || !qk) return pf::invalid("NULL argument");
    PF_CUDA(pf::launch_line_injections(p->d, y, ph, pk, qh, qk, (cudaStream_t)stream));
    return PF_OK;
}

int pf_line_jacobian_slots(const pf_plan* p, const double* y, double* slots, void* stream) {
    if (!p || !y || !slots) return pf::invalid("NULL argument");
    PF_CUDA(pf::launch_line_jac_slots(p->d, y, slots, (cudaStream_t)stream));
    return PF_OK;
}

int pf_device_injections(const pf_plan* p, const double* y, double* pool, void* stream) {
    if (!p || !y || !pool) return pf::invalid("NULL argument");
    PF_CUDA(pf::launch_device_injections(p->d, y, pool, (cudaStream_t)stream));
    return PF_OK;
}

int pf_device_jacobian_slots(const pf_plan* p, const double* y, double* slots, void* stream) {
    if (!p || !y || !slots) return pf::invalid("NULL argument");
    PF_CUDA(pf::launch_device_jac_slots(p->d, y, slots, (cudaStream_t)stream));
    return PF_OK;
}

int pf_join_rows(int32_t n, const int32_t* ptr, const int32_t* split, const int32_t* idx,
                 const double* pool, double* out, void* stream) {
    if (n < 0) return pf::invalid("n < 0");
    if (n > 0 && (!ptr || !split || !out)) return pf::invalid("NULL argument");
    PF_CUDA(pf::launch_join_rows(n, ptr, split, idx, pool, out, (cudaStream_t)stream));
    return PF_OK;
}

int pf_gather_sum(int32_t n, const int32_t* ptr, const int32_t* idx, const double* vals,
                  double* out, void* stream) {
    if (n < 0) return pf::invalid("n < 0");
    if (n > 0 && (!ptr || !out)) return pf::invalid("NULL argument");
    PF_CUDA(pf::launch_gather_sum(n, ptr, idx, vals, out, (cudaStream_t)stream));
    return PF_OK;
}

int pf_sincos(int64_t n, const double* x, double* s, double* c, void* stream) {
    if (n < 0) return pf::invalid("n < 0");
    if (n > 0 && (!x || !s || !c)) return pf::invalid("NULL argument");
    PF_CUDA(pf::launch_sincos(n, x, s, c, (cudaStream_t)stream));
    return PF_OK;
}

}  // extern "C"
