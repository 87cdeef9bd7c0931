// pf_eval.cu - fp64 evaluation kernels for sm_100a.
//
// Compiled with -fmad=false: every product and sum is rounded exactly where
// the reference's wf1 rounds it (numba njit without fastmath, pflow
// kernels.py:79-282), so the only deviation from the CPU oracle is the last
// rounding of sin/cos: pf_trig.h is correctly rounded except in rare
// near-midpoint cases, and glibc 2.39 is not correctly rounded in ~0.3% of
// power-flow angles, so the two agree on >99.7% of arguments.
//
// Fused kernel k_eval (the product path): one thread per (bus, scenario).
// A bus walks its incidence list -- branches with h = bus ascending, then
// branches with k = bus ascending -- which is exactly the association order of
// the reference's join (residual.py:79-125) and CSC assembly
// (jacobian.py:50-72, kernels.py:277-282).  So the bus-balance sums and the
// summed Jacobian entries come out in the reference's order with no atomics
// and no contribution pool: each residual row and each Jacobian value is
// written exactly once (a parallel branch re-reads its own earlier write).
//
// Batched mode maps the 32 lanes of a warp to 32 scenarios of the same bus:
// topology loads are warp-uniform broadcasts and every state load / output
// store is one fully coalesced 256-byte transaction (PF_LANES-blocked layout).
#include <cuda_runtime.h>

#include "pf_internal.cuh"
#include "pf_trig.h"

namespace pf {
namespace {

constexpr int RES = 1, JAC = 2, NORM = 4;

// The one trig routine every kernel uses (fused, per-model, test surface):
// near-correctly-rounded table sin/cos (pf_trig.h), table staged in shared
// memory because lanes index it divergently.
__device__ __forceinline__ void pf_sincos(double x, const double* tab, double* s, double* c) {
    pf_sincos_tab(x, tab, s, c);
}

__device__ __forceinline__ const double* stage_trig_table(double* smem) {
    for (int t = threadIdx.x; t < PF_TRIG_N * 4; t += blockDim.x) smem[t] = pf_trig_tab[t];
    __syncthreads();
    return smem;
}

__device__ __forceinline__ double4 ldg4(const double4* p) {
    const double2* q = reinterpret_cast<const double2*>(p);
    double2 a = __ldg(q), b = __ldg(q + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ unsigned long long abs_bits(double x) {
    // |x| as an ordered integer; NaN sorts above +inf like numpy's max
    return static_cast<unsigned long long>(__double_as_longlong(fabs(x)));
}

template <bool BATCH>
struct Addr {
    int64_t y0, j0, pq0, pv0;  // element offset of entry 0 of this scenario
    __device__ __forceinline__ int64_t y(int64_t e) const { return BATCH ? y0 + e * PF_LANES : e; }
    __device__ __forceinline__ int64_t j(int64_t e) const { return BATCH ? j0 + e * PF_LANES : e; }
    __device__ __forceinline__ int64_t pq(int64_t e) const { return pq0 + e * PF_LANES; }
    __device__ __forceinline__ int64_t pv(int64_t e) const { return pv0 + e * PF_LANES; }
};

template <int MODE>
__device__ __forceinline__ void put_offdiag(double* __restrict__ jv, int64_t at, bool first,
                                            double v) {
    // reference assembly: acc = 0.0; acc += slot ... (kernels.py:277-282)
    if (first) jv[at] = 0.0 + v;
    else jv[at] = jv[at] + v;
}

template <int MODE, bool BATCH>
__device__ __forceinline__ unsigned long long eval_bus(
    const DevicePlan& d, const double* tab, const int32_t i, const Addr<BATCH>& A,
    const int32_t out_l,
    const double* __restrict__ y, const double* __restrict__ pq_p,
    const double* __restrict__ pq_q, const double* __restrict__ pv_p,
    double* __restrict__ g, double* __restrict__ jv) {
    const int32_t N = d.N;
    const double th_i = y[A.y(i)];
    const double v_i = y[A.y(N + i)];
    const int4 br = __ldg(d.bus_row + i);
    const int64_t rp = br.x, rq = br.y, nb = br.z;
    const int32_t pos_i = br.w & POS_MASK;
    const bool vdiag = (br.w & VDIAG) != 0;

    double acc_p = 0.0, acc_q = 0.0;
    double d_pt = 0.0, d_pv = 0.0, d_qt = 0.0, d_qv = 0.0;
    unsigned long long nrm = 0;

    const int32_t e1 = __ldg(d.inc_ptr + i + 1);
    for (int32_t e = __ldg(d.inc_ptr + i); e < e1; ++e) {
        const int4 m = __ldg(d.inc_meta + e);
        double4 c = ldg4(d.inc_coef + e);
        if (BATCH && m.y == out_l) c = make_double4(0.0, 0.0, 0.0, 0.0);  // outage
        const int32_t jb = m.x;
        const bool kside = (m.z & KSIDE) != 0;
        const double th_j = y[A.y(jb)];
        const double w = y[A.y(N + jb)];
        const double u = v_i;
        // thk = theta_h - theta_k (kernels.py:86)
        const double thk = kside ? (th_j - th_i) : (th_i - th_j);
        double si, ci;
        pf_sincos(thk, tab, &si, &ci);
        const double ab = u * w;
        // h side: t1h = gl ci + bl si, t2h = gl si - bl ci.  k side with
        // b1 = -bl2: t1k = gl2 ci - bl2 si, and t2s = -t2k.  Sign flips are
        // exact, so every term below is bit-identical to kernels.py:90-163.
        const double t1 = c.x * ci + c.y * si;
        const double t2 = c.x * si - c.y * ci;
        const double t2s = kside ? -t2 : t2;
        const double fp = u * u * c.z - ab * t1;     // ph / pk
        const double fq = -u * u * c.w - ab * t2s;   // qh / qk
        acc_p -= fp;
        acc_q -= fq;
        if (MODE & JAC) {
            d_pt += -ab * t2s;                     // gph_thh | gpk_thk
            d_pv += -(2.0 * u * c.z - w * t1);     // gph_vh  | gpk_vk
            d_qt += ab * t1;                       // gqh_thh | gqk_thk
            d_qv += 2.0 * u * c.w + w * t2s;       // gqh_vh  | gqk_vk
            const bool first = (m.z & FIRST) != 0;
            const int64_t pos = m.z & POS_MASK;
            put_offdiag<MODE>(jv, A.j(rp + pos), first, ab * t2s);        // gph_thk | gpk_thh
            put_offdiag<MODE>(jv, A.j(rp + nb + pos), first, u * t1);     // gph_vk  | gpk_vh
            put_offdiag<MODE>(jv, A.j(rq + pos), first, -ab * t1);        // gqh_thk | gqk_thh
            put_offdiag<MODE>(jv, A.j(rq + nb + pos), first, u * t2s);    // gqh_vk  | gqk_vh
        }
    }

    // devices in pool-segment order: PQ, PV, Slack, Shunt (residual.py:57, 91-109)
    const int32_t t1e = __ldg(d.dev_ptr + i + 1);
    for (int32_t t = __ldg(d.dev_ptr + i); t < t1e; ++t) {
        const int4 dv = __ldg(d.dev_list + t);
        const int32_t k = dv.y;
        if (dv.x == DEV_PQ) {
            const double p0 = (BATCH && pq_p) ? pq_p[A.pq(k)] : __ldg(d.pq_p0 + k);
            const double q0 = (BATCH && pq_q) ? pq_q[A.pq(k)] : __ldg(d.pq_q0 + k);
            acc_p += -p0;
            acc_q += -q0;
        } else if (dv.x == DEV_PV) {
            const double p0 = (BATCH && pv_p) ? pv_p[A.pv(k)] : __ldg(d.pv_p0 + k);
            const int32_t q = __ldg(d.pv_qg + k);
            const int64_t row = 2 * (int64_t)N + q;
            acc_p += p0;
            acc_q += y[A.y(row)];
            if (MODE & (RES | NORM)) {
                const double gv = 0.0 + (v_i - __ldg(d.pv_v0 + k));
                if (MODE & RES) g[A.y(row)] = gv;
                nrm = max(nrm, abs_bits(gv));
            }
            if (MODE & JAC) {
                jv[A.j(dv.z)] = 1.0;   // (g_q[i], Q_g)   kernels.py:244-247
                jv[A.j(dv.w)] = 1.0;   // (g_V, V_i)
            }
        } else if (dv.x == DEV_SLACK) {
            const int32_t q = __ldg(d.sl_qg + k);
            const int32_t ps = __ldg(d.sl_ps + k);
            const int64_t row_v = 2 * (int64_t)N + q;
            const int64_t row_t = 2 * (int64_t)N + d.n_gen + ps;
            acc_p += y[A.y(row_t)];
            acc_q += y[A.y(row_v)];
            if (MODE & (RES | NORM)) {
                const double gv = 0.0 + (v_i - __ldg(d.sl_v0 + k));
                const double gt = 0.0 + (th_i - __ldg(d.sl_th0 + k));
                if (MODE & RES) {
                    g[A.y(row_v)] = gv;
                    g[A.y(row_t)] = gt;
                }
                nrm = max(nrm, max(abs_bits(gv), abs_bits(gt)));
            }
            if (MODE & JAC) {
                jv[A.j(dv.z)] = 1.0;                                   // (g_p, P_s)
                jv[A.j(dv.w)] = 1.0;                                   // (g_q, Q_g)
                jv[A.j(__ldg(d.gen_row_pos + q))] = 1.0;               // (g_V, V)
                jv[A.j(__ldg(d.gen_row_pos + d.n_gen + ps))] = 1.0;    // (g_theta, theta)
            }
        } else {  // DEV_SHUNT (kernels.py:236-241, 258-262)
            const double gsh = __ldg(d.sh_g + k), bsh = __ldg(d.sh_b + k);
            const double v2 = v_i * v_i;
            acc_p += -gsh * v2;
            acc_q += bsh * v2;
            if (MODE & JAC) {
                d_pv += -2.0 * gsh * v_i;
                d_qv += 2.0 * bsh * v_i;
            }
        }
    }

    if (MODE & RES) {
        g[A.y(i)] = acc_p;
        g[A.y(N + i)] = acc_q;
    }
    nrm = max(nrm, max(abs_bits(acc_p), abs_bits(acc_q)));
    if (MODE & JAC) {
        if (nb > 0) {
            jv[A.j(rp + pos_i)] = d_pt;
            jv[A.j(rq + pos_i)] = d_qt;
        }
        if (vdiag) {
            jv[A.j(rp + nb + pos_i)] = d_pv;
            jv[A.j(rq + nb + pos_i)] = d_qv;
        }
    }
    return nrm;
}

// Batched: blockDim = 32 * W, warp w of block (x, y) = bus x*W + w of
// scenario block y; lane = scenario within the block.
template <int MODE, int W>
__global__ void __launch_bounds__(32 * W) k_eval_batched(
    const DevicePlan d, const int32_t K, const double* __restrict__ y,
    const double* __restrict__ pq_p, const double* __restrict__ pq_q,
    const double* __restrict__ pv_p, const int32_t* __restrict__ outage,
    double* __restrict__ g, double* __restrict__ jv, unsigned long long* __restrict__ norms) {
    __shared__ unsigned long long red[W][32];
    __shared__ double s_tab[PF_TRIG_N * 4];
    const double* tab = stage_trig_table(s_tab);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t bus = blockIdx.x * W + warp;
    const int64_t blk = blockIdx.y;
    const int32_t s = (int32_t)(blk * PF_LANES + lane);
    unsigned long long nrm = 0;
    if (bus < d.N && s < K) {
        Addr<true> A;
        A.y0 = blk * (int64_t)d.n_var * PF_LANES + lane;
        A.j0 = blk * (int64_t)d.nnz * PF_LANES + lane;
        A.pq0 = blk * (int64_t)d.P * PF_LANES + lane;
        A.pv0 = blk * (int64_t)d.G * PF_LANES + lane;
        const int32_t out_l = outage ? __ldg(outage + s) : -1;
        nrm = eval_bus<MODE, true>(d, tab, bus, A, out_l, y, pq_p, pq_q, pv_p, g, jv);
    }
    if (MODE & NORM) {
        red[warp][lane] = nrm;
        __syncthreads();
        if (warp == 0) {
            unsigned long long m = red[0][lane];
#pragma unroll
            for (int w = 1; w < W; ++w) m = max(m, red[w][lane]);
            if (s < K && m) atomicMax(norms + s, m);
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(128) k_eval_single(const DevicePlan d,
                                                     const double* __restrict__ y,
                                                     double* __restrict__ g,
                                                     double* __restrict__ jv,
                                                     unsigned long long* __restrict__ norm) {
    __shared__ unsigned long long red[4];
    __shared__ double s_tab[PF_TRIG_N * 4];
    const double* tab = stage_trig_table(s_tab);
    const int32_t bus = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long nrm = 0;
    if (bus < d.N) {
        Addr<false> A{0, 0, 0, 0};
        nrm = eval_bus<MODE, false>(d, tab, bus, A, -1, y, nullptr, nullptr, nullptr, g, jv);
    }
    if (MODE & NORM) {
        for (int o = 16; o > 0; o >>= 1) nrm = max(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long m = max(max(red[0], red[1]), max(red[2], red[3]));
            if (m) atomicMax(norm, m);
        }
    }
}

// ---- per-model kernels (unit parity with pflow kernels) -------------------

// kernels.py:79-97, same expressions
__global__ void k_line_injections(const DevicePlan d, const double* __restrict__ y,
                                  double* ph, double* pk, double* qh, double* qk) {
    __shared__ double s_tab[PF_TRIG_N * 4];
    const double* tab = stage_trig_table(s_tab);
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d.L) return;
    const int32_t h = d.bus_h[i], k = d.bus_k[i], nb = d.N;
    const double a = y[nb + h];
    const double b = y[nb + k];
    const double thk = y[h] - y[k];
    double si, ci;
    pf_sincos(thk, tab, &si, &ci);
    const double ab = a * b;
    const double t1h = d.gl[i] * ci + d.bl[i] * si;
    const double t2h = d.gl[i] * si - d.bl[i] * ci;
    const double t1k = d.gl2[i] * ci - d.bl2[i] * si;
    const double t2k = d.gl2[i] * si + d.bl2[i] * ci;
    ph[i] = a * a * d.gsh[i] - ab * t1h;
    qh[i] = -a * a * d.bsh[i] - ab * t2h;
    pk[i] = b * b * d.gsk[i] - ab * t1k;
    qk[i] = -b * b * d.bsk[i] + ab * t2k;
}

// kernels.py:128-163; o = [16][L] in jacobian.py:31-36 order
__global__ void k_line_jac_slots(const DevicePlan d, const double* __restrict__ y, double* o) {
    __shared__ double s_tab[PF_TRIG_N * 4];
    const double* tab = stage_trig_table(s_tab);
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d.L) return;
    const int64_t L = d.L;
    const int32_t h = d.bus_h[i], k = d.bus_k[i], nb = d.N;
    const double a = y[nb + h];
    const double b = y[nb + k];
    const double thk = y[h] - y[k];
    double si, ci;
    pf_sincos(thk, tab, &si, &ci);
    const double ab = a * b;
    const double t1h = d.gl[i] * ci + d.bl[i] * si;
    const double t2h = d.gl[i] * si - d.bl[i] * ci;
    const double t1k = d.gl2[i] * ci - d.bl2[i] * si;
    const double t2k = d.gl2[i] * si + d.bl2[i] * ci;
    o[0 * L + i] = -ab * t2h;
    o[1 * L + i] = ab * t2h;
    o[2 * L + i] = -(2.0 * a * d.gsh[i] - b * t1h);
    o[3 * L + i] = a * t1h;
    o[4 * L + i] = ab * t1h;
    o[5 * L + i] = -ab * t1h;
    o[6 * L + i] = 2.0 * a * d.bsh[i] + b * t2h;
    o[7 * L + i] = a * t2h;
    o[8 * L + i] = -ab * t2k;
    o[9 * L + i] = ab * t2k;
    o[10 * L + i] = b * t1k;
    o[11 * L + i] = -(2.0 * b * d.gsk[i] - a * t1k);
    o[12 * L + i] = -ab * t1k;
    o[13 * L + i] = ab * t1k;
    o[14 * L + i] = -b * t2k;
    o[15 * L + i] = 2.0 * b * d.bsk[i] - a * t2k;
}

// kernels.py:215-241 into pool segments 4..14 of residual.py:57
__global__ void k_device_injections(const DevicePlan d, const double* __restrict__ y,
                                    double* pool) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t P = d.P, G = d.G, S = d.S, H = d.H, nb = d.N;
    double* pq_p = pool;
    double* pq_q = pq_p + P;
    double* pv_p = pq_q + P;
    double* pv_q = pv_p + G;
    double* pv_v = pv_q + G;
    double* sl_p = pv_v + G;
    double* sl_q = sl_p + S;
    double* sl_v = sl_q + S;
    double* sl_t = sl_v + S;
    double* sh_p = sl_t + S;
    double* sh_q = sh_p + H;
    if (t < P) {
        pq_p[t] = -d.pq_p0[t];
        pq_q[t] = -d.pq_q0[t];
        return;
    }
    t -= P;
    if (t < G) {
        pv_p[t] = d.pv_p0[t];
        pv_q[t] = y[2 * nb + d.pv_qg[t]];
        pv_v[t] = y[nb + d.pv_bus[t]] - d.pv_v0[t];
        return;
    }
    t -= G;
    if (t < S) {
        sl_p[t] = y[2 * nb + d.n_gen + d.sl_ps[t]];
        sl_q[t] = y[2 * nb + d.sl_qg[t]];
        sl_v[t] = y[nb + d.sl_bus[t]] - d.sl_v0[t];
        sl_t[t] = y[d.sl_bus[t]] - d.sl_th0[t];
        return;
    }
    t -= S;
    if (t < H) {
        const double vi = y[nb + d.sh_bus[t]];
        const double v2 = vi * vi;
        sh_p[t] = -d.sh_g[t] * v2;
        sh_q[t] = d.sh_b[t] * v2;
    }
}

// kernels.py:244-262 into the device sections of jacobian.py:200-207
__global__ void k_device_jac_slots(const DevicePlan d, const double* __restrict__ y, double* o) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t G = d.G, S = d.S, H = d.H, nb = d.N;
    if (t < G) {
        o[t] = 1.0;
        o[G + t] = 1.0;
        return;
    }
    t -= G;
    if (t < S) {
        o[2 * G + t] = 1.0;
        o[2 * G + S + t] = 1.0;
        o[2 * G + 2 * S + t] = 1.0;
        o[2 * G + 3 * S + t] = 1.0;
        return;
    }
    t -= S;
    if (t < H) {
        const double vi = y[nb + d.sh_bus[t]];
        o[2 * G + 4 * S + t] = -2.0 * d.sh_g[t] * vi;
        o[2 * G + 4 * S + H + t] = 2.0 * d.sh_b[t] * vi;
    }
}

// kernels.py:265-274
__global__ void k_join_rows(int32_t n, const int32_t* __restrict__ ptr,
                            const int32_t* __restrict__ split, const int32_t* __restrict__ idx,
                            const double* __restrict__ pool, double* __restrict__ out) {
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    double acc = 0.0;
    for (int32_t j = ptr[r]; j < split[r]; ++j) acc -= pool[idx[j]];
    for (int32_t j = split[r]; j < ptr[r + 1]; ++j) acc += pool[idx[j]];
    out[r] = acc;
}

// kernels.py:277-282
__global__ void k_gather_sum(int32_t n, const int32_t* __restrict__ ptr,
                             const int32_t* __restrict__ idx, const double* __restrict__ vals,
                             double* __restrict__ out) {
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    double acc = 0.0;
    for (int32_t j = ptr[r]; j < ptr[r + 1]; ++j) acc += vals[idx[j]];
    out[r] = acc;
}

// CSR -> reference CSC order; batched: one lane per scenario of a block
__global__ void k_jac_to_csc(int32_t nnz, int32_t nblk, const int32_t* __restrict__ perm,
                             const double* __restrict__ src, double* __restrict__ dst,
                             bool batched) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (!batched) {
        if (t < nnz) dst[t] = src[__ldg(perm + t)];
        return;
    }
    const int64_t q = t >> 5, lane = t & 31;
    const int64_t blk = blockIdx.y;
    if (q >= nnz) return;
    const int64_t base = blk * (int64_t)nnz * PF_LANES + lane;
    dst[base + q * PF_LANES] = src[base + (int64_t)__ldg(perm + q) * PF_LANES];
}

// array sin/cos test surface (pflow kernels.py:66-72 exposes the same)
__global__ void k_sincos(int64_t n, const double* __restrict__ x, double* __restrict__ s,
                         double* __restrict__ c) {
    __shared__ double s_tab[PF_TRIG_N * 4];
    const double* tab = stage_trig_table(s_tab);
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) pf_sincos(x[i], tab, s + i, c + i);
}

inline unsigned grid_for(int64_t n, int threads) {
    return (unsigned)((n + threads - 1) / threads);
}

}  // namespace

// ---- launchers --------------------------------------------------------------

template <int MODE>
static void launch_single_mode(const DevicePlan& d, const double* y, double* g, double* j,
                               double* norm, cudaStream_t st) {
    k_eval_single<MODE><<<grid_for(d.N, 128), 128, 0, st>>>(
        d, y, g, j, reinterpret_cast<unsigned long long*>(norm));
}

cudaError_t launch_eval_single(const DevicePlan& d, const double* y, double* g, double* j,
                               double* norm, cudaStream_t st) {
    if (norm) {
        cudaError_t e = cudaMemsetAsync(norm, 0, sizeof(double), st);
        if (e != cudaSuccess) return e;
    }
    if (d.N == 0) return cudaSuccess;
    const int mode = (g ? RES : 0) | (j ? JAC : 0) | (norm ? NORM : 0);
    switch (mode) {
        case RES: launch_single_mode<RES>(d, y, g, j, norm, st); break;
        case JAC: launch_single_mode<JAC>(d, y, g, j, norm, st); break;
        case RES | JAC: launch_single_mode<RES | JAC>(d, y, g, j, norm, st); break;
        case NORM: launch_single_mode<NORM>(d, y, g, j, norm, st); break;
        case RES | NORM: launch_single_mode<RES | NORM>(d, y, g, j, norm, st); break;
        case JAC | NORM: launch_single_mode<JAC | NORM>(d, y, g, j, norm, st); break;
        case RES | JAC | NORM: launch_single_mode<RES | JAC | NORM>(d, y, g, j, norm, st); break;
        default: return cudaSuccess;
    }
    count_launch();
    return cudaGetLastError();
}

constexpr int BATCH_W = 8;

template <int MODE>
static void launch_batched_mode(const DevicePlan& d, int32_t K, const double* y,
                                const double* pq_p, const double* pq_q, const double* pv_p,
                                const int32_t* outage, double* g, double* j, double* norms,
                                cudaStream_t st) {
    dim3 grid(grid_for(d.N, BATCH_W), grid_for(K, PF_LANES));
    k_eval_batched<MODE, BATCH_W><<<grid, 32 * BATCH_W, 0, st>>>(
        d, K, y, pq_p, pq_q, pv_p, outage, g, j, reinterpret_cast<unsigned long long*>(norms));
}

cudaError_t launch_eval_batched(const DevicePlan& d, int32_t K, const double* y,
                                const double* pq_p, const double* pq_q, const double* pv_p,
                                const int32_t* outage, double* g, double* j, double* norms,
                                cudaStream_t st) {
    if (norms) {
        cudaError_t e = cudaMemsetAsync(norms, 0, sizeof(double) * (size_t)K, st);
        if (e != cudaSuccess) return e;
    }
    if (d.N == 0 || K == 0) return cudaSuccess;
    const int mode = (g ? RES : 0) | (j ? JAC : 0) | (norms ? NORM : 0);
#define PF_B(M) launch_batched_mode<M>(d, K, y, pq_p, pq_q, pv_p, outage, g, j, norms, st)
    switch (mode) {
        case RES: PF_B(RES); break;
        case JAC: PF_B(JAC); break;
        case RES | JAC: PF_B(RES | JAC); break;
        case NORM: PF_B(NORM); break;
        case RES | NORM: PF_B(RES | NORM); break;
        case JAC | NORM: PF_B(JAC | NORM); break;
        case RES | JAC | NORM: PF_B(RES | JAC | NORM); break;
        default: return cudaSuccess;
    }
#undef PF_B
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_jac_to_csc(const DevicePlan& d, int32_t K, const double* jcsr, double* jcsc,
                              cudaStream_t st) {
    if (d.nnz == 0) return cudaSuccess;
    if (K <= 0) {
        k_jac_to_csc<<<grid_for(d.nnz, 256), 256, 0, st>>>(d.nnz, 1, d.csc_perm, jcsr, jcsc,
                                                           false);
    } else {
        dim3 grid(grid_for((int64_t)d.nnz * PF_LANES, 256), grid_for(K, PF_LANES));
        k_jac_to_csc<<<grid, 256, 0, st>>>(d.nnz, grid.y, d.csc_perm, jcsr, jcsc, true);
    }
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_line_injections(const DevicePlan& d, const double* y, double* ph, double* pk,
                                   double* qh, double* qk, cudaStream_t st) {
    if (d.L == 0) return cudaSuccess;
    k_line_injections<<<grid_for(d.L, 256), 256, 0, st>>>(d, y, ph, pk, qh, qk);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_line_jac_slots(const DevicePlan& d, const double* y, double* slots,
                                  cudaStream_t st) {
    if (d.L == 0) return cudaSuccess;
    k_line_jac_slots<<<grid_for(d.L, 256), 256, 0, st>>>(d, y, slots);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_device_injections(const DevicePlan& d, const double* y, double* pool,
                                     cudaStream_t st) {
    const int64_t n = (int64_t)d.P + d.G + d.S + d.H;
    if (n == 0) return cudaSuccess;
    k_device_injections<<<grid_for(n, 256), 256, 0, st>>>(d, y, pool);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_device_jac_slots(const DevicePlan& d, const double* y, double* slots,
                                    cudaStream_t st) {
    const int64_t n = (int64_t)d.G + d.S + d.H;
    if (n == 0) return cudaSuccess;
    k_device_jac_slots<<<grid_for(n, 256), 256, 0, st>>>(d, y, slots);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_join_rows(int32_t n, const int32_t* ptr, const int32_t* split,
                             const int32_t* idx, const double* pool, double* out,
                             cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_join_rows<<<grid_for(n, 256), 256, 0, st>>>(n, ptr, split, idx, pool, out);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_gather_sum(int32_t n, const int32_t* ptr, const int32_t* idx,
                              const double* vals, double* out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_gather_sum<<<grid_for(n, 256), 256, 0, st>>>(n, ptr, idx, vals, out);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_sincos(int64_t n, const double* x, double* s, double* c, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_sincos<<<grid_for(n, 256), 256, 0, st>>>(n, x, s, c);
    count_launch();
    return cudaGetLastError();
}

}  // namespace pf
