// pf_eval.cu - fp64 evaluation kernels for sm_100a.
//
// Compiled with -fmad=false: every product and sum is rounded exactly where
// the reference's wf1 rounds it (numba njit without fastmath, pflow
// kernels.py:79-282), so the only deviation from the CPU oracle is the last
// rounding of sin/cos -- and pf_trig.h restates glibc 2.39's sin/cos bit for
// bit (checked against the live libm on 2e9 arguments), so there is none.
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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "pf_internal.cuh"
#include "pf_trig.h"

namespace pf {
namespace {

constexpr int RES = 1, JAC = 2, NORM = 4;

// The one trig routine every kernel uses (fused, per-model, test surface):
// glibc-identical table sin/cos (pf_trig.h), table staged in shared memory
// because lanes index it divergently.
__device__ __forceinline__ void pf_sincos(double x, const double* tab, double* s, double* c) {
    pf_sincos_tab(x, tab, s, c);
}

__device__ __forceinline__ const double* stage_trig_table(double* smem) {
    for (int t = threadIdx.x; t < PF_TRIG_N * 4; t += blockDim.x) smem[t] = __ldg(pf_trig_tab + t);
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

// Per-thread view of one scenario: base pointers already offset to the
// thread's scenario block and lane, so entry e sits at base[e * S] with
// S = PF_LANES (batched) or 1 (single grid).  Offsets stay 32-bit
// (pf_plan_create checks nnz * PF_LANES < 2^31).
template <int S>
struct Scen {
    const double* __restrict__ y;
    const double* __restrict__ pq_p;
    const double* __restrict__ pq_q;
    const double* __restrict__ pv_p;
    double* __restrict__ g;
    double* __restrict__ j;
    int32_t out_l;
};

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Stage the next item of this warp: pull the scenario-block data bus `i`'s
// evaluation will read (its own state, every neighbour's state, each
// device's per-scenario parameters: 256 B = 2 lines per entry) from HBM into
// L2 while the current item computes, and touch its incidence / device
// records (real loads, so they land in L1).  The lanes split the incidence
// and device lists, so one pass issues every line at once.  Measured on B200
// (config 3): 0.778 -> 0.732 ms per K=256 launch; an L1 prefetch or a
// two-items-ahead distance measured no better.
template <int S>
__device__ __forceinline__ void stage_next_bus(const DevicePlan& d, const Scen<S>& A,
                                               const int32_t i, const int4 rng, const int lane) {
    const int32_t N = d.N;
    const double* y = A.y;
    if (lane < 4) {
        const int64_t e = (lane < 2) ? i : N + i;
        prefetch_l2(y + e * S + (lane & 1) * 16);
    }
    for (int32_t e = rng.x + lane; e < rng.y; e += 32) {
        const int32_t j = __ldg(&d.inc_meta[e].x);
        prefetch_l2(y + (int64_t)j * S);
        prefetch_l2(y + (int64_t)j * S + 16);
        prefetch_l2(y + (int64_t)(N + j) * S);
        prefetch_l2(y + (int64_t)(N + j) * S + 16);
    }
    for (int32_t t = rng.z + lane; t < rng.w; t += 32) {
        const int4 dv = __ldg(d.dev_list + t);
        const double* a = nullptr;
        const double* b = nullptr;
        if (dv.x == DEV_PQ) {
            a = A.pq_p ? A.pq_p + (int64_t)dv.y * S : nullptr;
            b = A.pq_q ? A.pq_q + (int64_t)dv.y * S : nullptr;
        } else if (dv.x == DEV_PV) {
            a = A.pv_p ? A.pv_p + (int64_t)dv.y * S : nullptr;
            b = y + (int64_t)(2 * N + dv.y) * S;   // Q_g (pv_qg = index)
        }
        if (a) {
            prefetch_l2(a);
            prefetch_l2(a + 16);
        }
        if (b) {
            prefetch_l2(b);
            prefetch_l2(b + 16);
        }
    }
}

// Outputs are written once and never re-read by the kernel (except the rare
// parallel-branch update): no L1 allocation.  In L2 they keep the default
// policy: an evict-first policy (createpolicy) measured 12 % slower on
// config 3 and `.cs` no faster than plain stores (config 4: 0.535 -> 0.531).
__device__ __forceinline__ void st_out(double* p, double v) {
    asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

template <int S>
__device__ __forceinline__ void put_offdiag(double* __restrict__ jv, int32_t at, bool first,
                                            double v) {
    // reference assembly: acc = 0.0; acc += slot ... (kernels.py:277-282)
    if (first) st_out(jv + at * S, 0.0 + v);
    else st_out(jv + at * S, jv[at * S] + v);
}

// One incidence of bus i (kernels.py:79-163 restated for one terminal):
// adds the flow to the bus balance, the partials to the four diagonal
// accumulators, and writes the four off-diagonal values of this neighbour.
// The ten per-incidence quantities of one bus terminal (kernels.py:79-163
// restated for one side): the two flows and the eight residual-row partials.
struct IncVals {
    double fp, fq;                 // ph / pk, qh / qk
    double pt, pv, qt, qv;         // diagonal partials (theta_i, V_i) of rows g_p[i], g_q[i]
    double opt, opv, oqt, oqv;     // off-diagonal partials (theta_j, V_j)
};

// The ten values of one terminal, from sin/cos of d = theta_i - theta_j
// (bus i, neighbour j), the terminal's coefficients c and u = V_i, w = V_j.
// h side (i = h): c = {gl, bl, gsh, bsh} and d = thk (kernels.py:86), so
// t1 = gl ci + bl si = t1h, t2 = gl si - bl ci = t2h.  k side (i = k):
// c = {gl2, bl2, gsk, bsk} and d = -thk, so sin d = -sin thk (pf_trig is odd
// bit for bit) and t1 = gl2 ci - bl2 sin thk = t1k, t2 = -(gl2 sin thk +
// bl2 ci) = -t2k.  Negations are exact and rounding is sign-symmetric, so
// every term is bit-identical to kernels.py:90-163 (t2s is t2h | -t2k).
__device__ __forceinline__ IncVals inc_terms(const double sd, const double ci, const double4 c,
                                             const double u, const double w) {
    const double ab = u * w;
    const double t1 = c.x * ci + c.y * sd;
    const double t2s = c.x * sd - c.y * ci;
    const double uu = u * u;                     // (-u)*u == -(u*u) exactly
    IncVals v;
    v.fp = uu * c.z - ab * t1;                   // ph | pk
    v.fq = -(uu * c.w) - ab * t2s;               // qh | qk
    v.pt = -ab * t2s;                            // gph_thh | gpk_thk
    v.pv = -(2.0 * u * c.z - w * t1);            // gph_vh  | gpk_vk
    v.qt = ab * t1;                              // gqh_thh | gqk_thk
    v.qv = 2.0 * u * c.w + w * t2s;              // gqh_vh  | gqk_vk
    v.opt = ab * t2s;                            // gph_thk | gpk_thh
    v.opv = u * t1;                              // gph_vk  | gpk_vh
    v.oqt = -ab * t1;                            // gqh_thk | gqk_thh
    v.oqv = u * t2s;                             // gqh_vk  | gqk_vh
    return v;
}

// One incidence of bus i against neighbour j (theta_i, u = V_i, theta_j, w = V_j).
template <int S>
__device__ __forceinline__ IncVals inc_vals(const double* tab, const int4 m, double4 c,
                                            const double th_i, const double u,
                                            const double th_j, const double w,
                                            const int32_t out_l, const bool ochk = true) {
    constexpr bool BATCH = S > 1;
    // outaged branch in some lane's scenario: rare, so test warp-wide first
    // (ochk: a warp-uniform pre-test per bus, see k_eval_staged)
    if (BATCH && ochk) {
        const bool hit = m.y == out_l;
        if (__any_sync(__activemask(), hit) && hit) c = make_double4(0.0, 0.0, 0.0, 0.0);
    }
    double sd, ci;
    pf_sincos(th_i - th_j, tab, &sd, &ci);
    return inc_terms(sd, ci, c, u, w);
}

// Fold one incidence into the bus's sums, in list order.
template <int MODE>
__device__ __forceinline__ void inc_fold(const IncVals& v, double& acc_p, double& acc_q,
                                         double& d_pt, double& d_pv, double& d_qt,
                                         double& d_qv) {
    acc_p -= v.fp;
    acc_q -= v.fq;
    if (MODE & JAC) {
        d_pt += v.pt;
        d_pv += v.pv;
        d_qt += v.qt;
        d_qv += v.qv;
    }
}

// Jacobian writers.  GlobalJ stores straight to the value array (batched:
// lane stride S); StagedJ (single grid) keeps the rows g_p, g_q of the CTA's
// buses in shared memory and writes other rows (g_V, g_theta) through.
// Writers take the row kind: p (row g_p[i] of the bus being evaluated), q
// (row g_q[i]) or x (any other row: g_V, g_theta).
template <int S>
struct GlobalJ {
    double* __restrict__ jv;
    __device__ __forceinline__ void put(int32_t at, double v) const { st_out(jv + at * S, v); }
    __device__ __forceinline__ void put_p(int32_t at, double v) const { put(at, v); }
    __device__ __forceinline__ void put_q(int32_t at, double v) const { put(at, v); }
    __device__ __forceinline__ void put_x(int32_t at, double v) const { put(at, v); }
    // reference assembly: acc = 0.0; acc += slot ... (kernels.py:277-282)
    __device__ __forceinline__ void add_p(int32_t at, bool first, double v) const {
        put_offdiag<S>(jv, at, first, v);
    }
    __device__ __forceinline__ void add_q(int32_t at, bool first, double v) const {
        put_offdiag<S>(jv, at, first, v);
    }
};

// The chunk's rows g_p[b0..b1) and g_q[b0..b1) are staged, so p / q
// entries of its buses go to shared memory without a range test.
struct StagedJ {
    double* jp;                   // staged rows g_p[b0..b1): jp[k] is jv[p0 + k]
    double* jq;                   // staged rows g_q[b0..b1): jq[k] is jv[q0 + k]
    double* __restrict__ jv;
    int32_t p0, q0;
    __device__ __forceinline__ void put_p(int32_t at, double v) const { jp[at - p0] = v; }
    __device__ __forceinline__ void put_q(int32_t at, double v) const { jq[at - q0] = v; }
    __device__ __forceinline__ void put_x(int32_t at, double v) const { jv[at] = v; }
    __device__ __forceinline__ void add_p(int32_t at, bool first, double v) const {
        double* p = jp + (at - p0);
        *p = first ? 0.0 + v : *p + v;
    }
    __device__ __forceinline__ void add_q(int32_t at, bool first, double v) const {
        double* p = jq + (at - q0);
        *p = first ? 0.0 + v : *p + v;
    }
};

// Write the four off-diagonal Jacobian values of one incidence.
template <class JW>
__device__ __forceinline__ void inc_offdiag(const IncVals& v, const int4 m, const JW& jw,
                                            const int32_t rp, const int32_t rq, const int32_t nb) {
    const bool first = (m.z & FIRST) != 0;
    const int32_t pos = m.z & POS_MASK;
    // one (warp-uniform) branch per incidence: the common first-neighbour
    // stores, or the rare parallel-branch read-modify-writes
    if (first) {
        jw.add_p(rp + pos, true, v.opt);
        jw.add_p(rp + nb + pos, true, v.opv);
        jw.add_q(rq + pos, true, v.oqt);
        jw.add_q(rq + nb + pos, true, v.oqv);
    } else {
        jw.add_p(rp + pos, false, v.opt);
        jw.add_p(rp + nb + pos, false, v.opv);
        jw.add_q(rq + pos, false, v.oqt);
        jw.add_q(rq + nb + pos, false, v.oqv);
    }
}

// Sources whose incidence values were computed beforehand (the single-grid
// incidence phase) set kSplit; the others compute them in place.
template <class Src, class = void>
struct SplitIncidences {
    static constexpr bool value = false;
};
template <class Src>
struct SplitIncidences<Src, decltype(void(Src::kSplit))> {
    static constexpr bool value = Src::kSplit;
};

// Sources that hold a bus's first incidences and devices in shared memory
// (the staged batched kernel) set kStaged.
template <class Src, class = void>
struct StagedPrefix {
    static constexpr bool value = false;
};
template <class Src>
struct StagedPrefix<Src, decltype(void(Src::kStaged))> {
    static constexpr bool value = Src::kStaged;
};

// Sources holding a bus's first two devices in registers (the single-grid
// source) set kRegDev: those two are evaluated without the generic device
// loop's index selects.
template <class Src, class = void>
struct RegDevices {
    static constexpr bool value = false;
};
template <class Src>
struct RegDevices<Src, decltype(void(Src::kRegDev))> {
    static constexpr bool value = Src::kRegDev;
};

// Staged sources that can reuse their slot for the incidences past the
// staged prefix (chunks of the prefix's size) set kChunked.
template <class Src, class = void>
struct ChunkedOverflow {
    static constexpr bool value = false;
};
template <class Src>
struct ChunkedOverflow<Src, decltype(void(Src::kChunked))> {
    static constexpr bool value = Src::kChunked;
};

// Operand source of the global-memory path: every read goes to HBM/L2/L1.
template <int S>
struct GlobalSrc {
    const DevicePlan& d;
    const Scen<S>& A;               // block base pointers (shared memory when batched)
    const double* __restrict__ y;   // this lane's scenario view of the state
    int32_t i, ln;
    __device__ __forceinline__ int4 hdr0() const { return __ldg(d.bus_row + 2 * i); }
    __device__ __forceinline__ int4 hdr1() const { return __ldg(d.bus_row + 2 * i + 1); }
    __device__ __forceinline__ double th_i() const { return __ldg(y + i * S); }
    __device__ __forceinline__ double v_i() const { return __ldg(y + (d.N + i) * S); }
    __device__ __forceinline__ int4 meta(int32_t e, int32_t) const { return __ldg(d.inc_meta + e); }
    __device__ __forceinline__ double4 coef(int32_t e, int32_t) const { return ldg4(d.inc_coef + e); }
    __device__ __forceinline__ double th_j(int32_t j, int32_t) const { return __ldg(y + j * S); }
    __device__ __forceinline__ double v_j(int32_t j, int32_t) const {
        return __ldg(y + (d.N + j) * S);
    }
    __device__ __forceinline__ int4 dev(int32_t t, int32_t) const { return __ldg(d.dev_list + t); }
    // per-scenario device operands: (a, b) = PQ (p0, q0), PV (p0, Q_g), Slack (P_s, Q_g)
    __device__ __forceinline__ double dev_a(const int4 dv, int32_t) const {
        const int32_t k = dv.y;
        if (dv.x == DEV_PQ)
            return (S > 1 && A.pq_p) ? __ldg(A.pq_p + k * S + ln) : __ldg(d.pq_p0 + k);
        if (dv.x == DEV_PV)
            return (S > 1 && A.pv_p) ? __ldg(A.pv_p + k * S + ln) : __ldg(d.pv_p0 + k);
        return __ldg(y + (2 * d.N + d.n_gen + k) * S);   // P_s (sl_ps = index)
    }
    __device__ __forceinline__ double dev_b(const int4 dv, int32_t) const {
        const int32_t k = dv.y;
        if (dv.x == DEV_PQ)
            return (S > 1 && A.pq_q) ? __ldg(A.pq_q + k * S + ln) : __ldg(d.pq_q0 + k);
        if (dv.x == DEV_PV) return __ldg(y + (2 * d.N + k) * S);       // Q_g (pv_qg = index)
        return __ldg(y + (2 * d.N + d.G + k) * S);                     // Q_g (sl_qg = G + index)
    }
    // device constants (c, d) = PV (v0, -), Slack (v0, theta0), Shunt (g, b)
    __device__ __forceinline__ double dev_c(const int4 dv, int32_t) const {
        if (dv.x == DEV_PV) return __ldg(d.pv_v0 + dv.y);
        if (dv.x == DEV_SLACK) return __ldg(d.sl_v0 + dv.y);
        return __ldg(d.sh_g + dv.y);
    }
    __device__ __forceinline__ double dev_d(const int4 dv, int32_t) const {
        if (dv.x == DEV_SLACK) return __ldg(d.sl_th0 + dv.y);
        return __ldg(d.sh_b + dv.y);
    }
};

// One bus for one scenario (S = PF_LANES: batched lane; S = 1: single grid),
// operands from `src` (global memory or a shared-memory staging slot).
template <int MODE, int S, class Src, class JW>
__device__ __forceinline__ unsigned long long eval_bus_src(const DevicePlan& d, const double* tab,
                                                           const int32_t i, const Src& src,
                                                           const Scen<S>& A, const int32_t ln,
                                                           const int32_t out_l, const JW& jw,
                                                           const bool ochk = true) {
    const int32_t N = d.N;
    const int4 br = src.hdr0();
    const int4 rng = src.hdr1();
    const int32_t rp = br.x, rq = br.y, nb = br.z;
    const int32_t pos_i = br.w & POS_MASK;
    const bool vdiag = (br.w & VDIAG) != 0;
    const double th_i = src.th_i();
    const double v_i = src.v_i();

    double acc_p = 0.0, acc_q = 0.0;
    double d_pt = 0.0, d_pv = 0.0, d_qt = 0.0, d_qv = 0.0;
    unsigned long long nrm = 0;

    if constexpr (SplitIncidences<Src>::value) {
        // values from the incidence phase; it already wrote the off-diagonals
        // of every SOLO incidence, parallel branches are summed here in order
        const bool dups = (MODE & JAC) && (br.w & DUPS);
        for (int32_t e = rng.x; e < rng.y; ++e) {
            inc_fold<MODE>(src.vals(e), acc_p, acc_q, d_pt, d_pv, d_qt, d_qv);
            if (dups) {
                const int4 m = src.meta(e, e - rng.x);
                if (!(m.z & SOLO)) inc_offdiag(src.dup(e), m, jw, rp, rq, nb);
            }
        }
    } else {
        auto inc_step = [&](const int4 m, const double4 c, const double tj, const double wj) {
            const IncVals v = inc_vals<S>(tab, m, c, th_i, v_i, tj, wj, out_l, ochk);
            inc_fold<MODE>(v, acc_p, acc_q, d_pt, d_pv, d_qt, d_qv);
            if (MODE & JAC) inc_offdiag(v, m, jw, rp, rq, nb);
        };
        int32_t e0 = rng.x;
        if constexpr (StagedPrefix<Src>::value) {   // operands in shared memory
            const int32_t ns = src.n_inc_staged();
            for (int32_t t = 0; t < ns; ++t)
                inc_step(src.smeta(t), src.scoef(t), src.sth(t), src.sv(t));
            e0 += ns;
            if constexpr (ChunkedOverflow<Src>::value) {
                // the rest in chunks of ns through the same slot space (a
                // hub's 48 overflow incidences cost two round trips per
                // chunk instead of two to three each)
                if (ns > 0) {
                    for (int32_t c0 = e0; c0 < rng.y; c0 += ns) {
                        const int32_t n = min(ns, rng.y - c0);
                        src.load_chunk(c0, n);
                        for (int32_t t = 0; t < n; ++t)
                            inc_step(src.smeta(t), src.scoef(t), src.sth(t), src.sv(t));
                    }
                    e0 = rng.y;
                }
            }
        }
        for (int32_t e = e0; e < rng.y; ++e) {
            const int32_t t = e - rng.x;
            const int4 m = src.meta(e, t);
            inc_step(m, src.coef(e, t), src.th_j(m.x, t), src.v_j(m.x, t));
        }
    }

    // devices in pool-segment order: PQ, PV, Slack, Shunt (residual.py:57, 91-109);
    // ga..gd fetch the device's operands (a, b) and constants (c, d) lazily
    auto dev_step = [&](const int4 dv, auto ga, auto gb, auto gc, auto gd) {
        const int32_t k = dv.y;
        if (dv.x == DEV_PQ) {
            acc_p += -ga();
            acc_q += -gb();
        } else if (dv.x == DEV_PV) {
            const int32_t row = 2 * N + k;   // g_V row of the gen (pv_qg = index, plan-checked)
            acc_p += ga();
            acc_q += gb();
            if (MODE & (RES | NORM)) {
                const double gv = 0.0 + (v_i - gc());
                if (MODE & RES) st_out(A.g + ln + row * S, gv);
                nrm = max(nrm, abs_bits(gv));
            }
            if (MODE & JAC) {
                jw.put_q(dv.z, 1.0);   // (g_q[i], Q_g)   kernels.py:244-247
                jw.put_x(dv.w, 1.0);   // (g_V, V_i)
            }
        } else if (dv.x == DEV_SLACK) {
            const int32_t q = d.G + k;    // sl_qg, sl_ps are aranges (plan-checked)
            const int32_t ps = k;
            const int32_t row_v = 2 * N + q;
            const int32_t row_t = 2 * N + d.n_gen + ps;
            acc_p += ga();   // P_s
            acc_q += gb();   // Q_g
            if (MODE & (RES | NORM)) {
                const double gv = 0.0 + (v_i - gc());
                const double gt = 0.0 + (th_i - gd());
                if (MODE & RES) {
                    st_out(A.g + ln + row_v * S, gv);
                    st_out(A.g + ln + row_t * S, gt);
                }
                nrm = max(nrm, max(abs_bits(gv), abs_bits(gt)));
            }
            if (MODE & JAC) {
                jw.put_p(dv.z, 1.0);                                   // (g_p, P_s)
                jw.put_q(dv.w, 1.0);                                   // (g_q, Q_g)
                jw.put_x(__ldg(d.gen_row_pos + q), 1.0);               // (g_V, V)
                jw.put_x(__ldg(d.gen_row_pos + d.n_gen + ps), 1.0);    // (g_theta, theta)
            }
        } else {  // DEV_SHUNT (kernels.py:236-241, 258-262)
            const double gsh = gc(), bsh = gd();
            const double v2 = v_i * v_i;
            acc_p += -gsh * v2;
            acc_q += bsh * v2;
            if (MODE & JAC) {
                d_pv += -2.0 * gsh * v_i;
                d_qv += 2.0 * bsh * v_i;
            }
        }
    };
    int32_t t0 = rng.z;
    if constexpr (StagedPrefix<Src>::value) {
        const int32_t nv = src.n_dev_staged();
        for (int32_t u = 0; u < nv; ++u) {
            const int4 dv = src.sdev(u);
            dev_step(dv, [&] { return src.sdev_a(dv, u); }, [&] { return src.sdev_b(dv, u); },
                     [&] { return src.sdev_c(u); }, [&] { return src.sdev_d(u); });
        }
        t0 += nv;
    }
    if constexpr (RegDevices<Src>::value) {
        const int32_t nd = rng.w - rng.z;
        if (nd > 0)
            dev_step(src.dv0, [&] { return src.a0; }, [&] { return src.b0; },
                     [&] { return src.c0; }, [&] { return src.d0; });
        if (nd > 1)
            dev_step(src.dv1, [&] { return src.a1; }, [&] { return src.b1; },
                     [&] { return src.c1; }, [&] { return src.d1; });
        t0 += min(nd, 2);
    }
    for (int32_t t = t0; t < rng.w; ++t) {
        const int32_t u = t - rng.z;
        const int4 dv = src.dev(t, u);
        dev_step(dv, [&] { return src.dev_a(dv, u); }, [&] { return src.dev_b(dv, u); },
                 [&] { return src.dev_c(dv, u); }, [&] { return src.dev_d(dv, u); });
    }

    if (MODE & RES) {
        st_out(A.g + ln + i * S, acc_p);
        st_out(A.g + ln + (N + i) * S, acc_q);
    }
    nrm = max(nrm, max(abs_bits(acc_p), abs_bits(acc_q)));
    if (MODE & JAC) {
        if (nb > 0) {
            jw.put_p(rp + pos_i, d_pt);
            jw.put_q(rq + pos_i, d_qt);
        }
        if (vdiag) {
            jw.put_p(rp + nb + pos_i, d_pv);
            jw.put_q(rq + nb + pos_i, d_qv);
        }
    }
    return nrm;
}

template <int MODE, int S>
__device__ __forceinline__ unsigned long long eval_bus(const DevicePlan& d, const double* tab,
                                                       const int32_t i, const Scen<S>& A,
                                                       const int32_t ln, const int32_t out_l) {
    GlobalSrc<S> src{d, A, A.y + ln, i, ln};
    return eval_bus_src<MODE, S>(d, tab, i, src, A, ln, out_l,
                                 GlobalJ<S>{A.j ? A.j + ln : nullptr});
}

// Batched, persistent: gridDim.x CTAs (a few per SM) stride over work items
// (scenario block b, group of W buses) in block-major order, so the whole
// GPU sweeps one 32-scenario block at a time and its states stay in L2.
// Warp w of an item evaluates bus (group * W + w) for the block's 32
// scenarios (lane = scenario).  Norms: per-lane running max per block,
// reduced across the CTA's warps and atomically max-ed into norms[s] only
// when the CTA moves to the next block (integer max of |g| bit patterns is
// exact and order-independent, NaN-propagating like numpy).
template <int MODE, int W, int MINB>
__global__ void __launch_bounds__(32 * W, MINB) k_eval_batched(
    const DevicePlan d, const int32_t K, const int32_t n_groups, const int32_t n_items,
    const double* __restrict__ y, const double* __restrict__ pq_p,
    const double* __restrict__ pq_q, const double* __restrict__ pv_p,
    const int32_t* __restrict__ outage, double* __restrict__ g, double* __restrict__ jv,
    unsigned long long* __restrict__ norms) {
    __shared__ unsigned long long red[W][32];
    __shared__ double s_tab[PF_TRIG_N * 4];
    const double* tab = stage_trig_table(s_tab);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t cur = -1;
    unsigned long long nrm = 0;
    auto flush = [&](int32_t blk) {
        __syncthreads();  // every warp is done with the previous block
        if (MODE & NORM) {
            red[warp][lane] = nrm;
            __syncthreads();
            if (warp == 0) {
                unsigned long long mx = red[0][lane];
#pragma unroll
                for (int w = 1; w < W; ++w) mx = max(mx, red[w][lane]);
                const int32_t s = blk * PF_LANES + lane;
                if (s < K && mx) atomicMax(norms + s, mx);
            }
            __syncthreads();
        }
        nrm = 0;
    };
    // item = blk * n_groups + grp, walked with a stride of gridDim.x
    // (gridDim.x <= n_groups, so grp wraps at most once per step)
    int32_t blk = blockIdx.x / n_groups;
    int32_t grp = blockIdx.x - blk * n_groups;
    // block base pointers live in shared memory (one copy per CTA) so they
    // cost no registers across the incidence loop
    __shared__ Scen<PF_LANES> A;
    int32_t out_l = -1;
    for (int32_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        if (blk != cur) {
            if (cur >= 0) flush(cur);
            cur = blk;
            if (threadIdx.x == 0) {
                const int64_t b = blk;
                A.y = y + b * d.n_var * PF_LANES;
                A.g = g ? g + b * d.n_var * PF_LANES : nullptr;
                A.j = jv ? jv + b * d.nnz * PF_LANES : nullptr;
                A.pq_p = pq_p ? pq_p + b * d.P * PF_LANES : nullptr;
                A.pq_q = pq_q ? pq_q + b * d.P * PF_LANES : nullptr;
                A.pv_p = pv_p ? pv_p + b * d.G * PF_LANES : nullptr;
            }
            const int32_t s = blk * PF_LANES + lane;
            out_l = (outage && s < K) ? __ldg(outage + s) : -1;
            if ((uint32_t)out_l >= (uint32_t)d.L) out_l = -1;   // out of range: no outage
            __syncthreads();
        }
        // processing order: high-degree buses first, so they do not form a
        // straggler tail at the end of each block's sweep
        const int32_t slot = grp * W + warp;
        const int32_t bus = slot < d.N ? __ldg(d.bus_order + slot) : d.N;
        // stage the next item of this warp (same block only) behind this one
        const int32_t gn = grp + gridDim.x;
        const int32_t sn = gn * W + warp;
        const bool pre = gn < n_groups && sn < d.N;
        int32_t bn = 0;
        int4 rng_n = make_int4(0, 0, 0, 0);
        if (pre) {
            bn = __ldg(d.bus_order + sn);
            rng_n = __ldg(d.bus_row + 2 * bn + 1);
        }
        if (bus < d.N && blk * PF_LANES + lane < K)
            nrm = max(nrm, eval_bus<MODE, PF_LANES>(d, tab, bus, A, lane, out_l));
        // (staging before the evaluation measured slower: 0.773 vs 0.741 ms)
        if (pre) stage_next_bus<PF_LANES>(d, A, bn, rng_n, lane);
        grp += gridDim.x;
        while (grp >= n_groups) {
            grp -= n_groups;
            ++blk;
        }
    }
    if (cur >= 0) flush(cur);
}

// ---- staged batched kernel (the product batched path) ----------------------
//
// k_eval_staged: same items, order and arithmetic as k_eval_batched (one
// warp = one bus x 32 scenarios), but the operands of each item reach the
// evaluating warp through shared memory.  Every warp owns two 4 KB slots.
// While it evaluates item k from one slot, its cp.async copies of item k+1
// fill the other: the bus's packet (header, incidence and device records,
// device constants; plan-built, see pf_internal.cuh WS_ROWS) and its 256-byte
// scenario rows (own state, neighbour states, device operands), 16 B per
// lane and two rows per warp instruction, named by a 64-byte stage record
// that was loaded one item earlier still.  The dependent global loads of the
// old kernel's per-item chain (header -> records -> neighbour rows -> device
// rows) thus overlap the previous item's arithmetic.  Warps stay independent:
// no producer warp, no CTA barrier after the prologue (a producer-warp
// version with an mbarrier ring measured 1.23 ms against 0.79 for this
// scheme at the same stage of development).  Incidences and devices past
// the staged ones are read from global memory as before.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// L2 policy of the plan reads that every scenario block repeats (packets,
// stage records): evict-last when the plan keeps them (DevicePlan::ws_keep).
// Rows of the scenario states get no hint: evict-last on them measured
// slower (config 3 0.572 -> 0.589 with the packets kept, also at fractions
// 0.5 and 0.25; config 4 -1 to -2 %).
__device__ __forceinline__ uint64_t plan_policy(int32_t keep) {
    uint64_t p;
    if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void cp_async16_pol(uint32_t dst, const void* src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst),
                 "l"(src), "l"(pol)
                 : "memory");
}
constexpr int WS_ROW_BYTES = PF_LANES * 8;
constexpr int WS_SLOT_BYTES = WS_ROWS * WS_ROW_BYTES + 32 * 16;   // rows + packet

// Operand source reading a staged slot (rows + packet in shared memory,
// addressed through 32-bit shared-window addresses): the first ni incidences
// and nv devices of the bus; the rest (and the parallel-branch re-reads) go
// through the global-memory accessors.
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double2 lds_v2f64(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ int4 lds_v4s32(uint32_t a) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a));
    return v;
}

struct StagedSrc : GlobalSrc<PF_LANES> {
    static constexpr bool kStaged = true;
    static constexpr bool kChunked = true;   // B200 config 4: 0.548 -> 0.533 ms
    uint32_t rw;   // shared address of this lane's entry of row 0 (row r at + r * 256)
    uint32_t pk;   // shared address of the slot packet
    int32_t ni, nv;
    __device__ __forceinline__ double row(int32_t r) const { return lds_f64(rw + r * WS_ROW_BYTES); }
    __device__ __forceinline__ int4 hdr0() const { return lds_v4s32(pk); }
    __device__ __forceinline__ int4 hdr1() const { return lds_v4s32(pk + 16); }
    __device__ __forceinline__ double th_i() const { return row(0); }
    __device__ __forceinline__ double v_i() const { return row(1); }
    __device__ __forceinline__ int32_t n_inc_staged() const { return ni; }
    __device__ __forceinline__ int32_t n_dev_staged() const { return nv; }
    __device__ __forceinline__ int4 smeta(int32_t t) const { return lds_v4s32(pk + 16 * (3 + t)); }
    __device__ __forceinline__ double4 scoef(int32_t t) const {
        const uint32_t c = pk + 16 * (3 + ni + 2 * t);
        const double2 a = lds_v2f64(c), b = lds_v2f64(c + 16);
        return make_double4(a.x, a.y, b.x, b.y);
    }
    __device__ __forceinline__ double sth(int32_t t) const { return row(2 + 2 * t); }
    __device__ __forceinline__ double sv(int32_t t) const { return row(3 + 2 * t); }
    __device__ __forceinline__ int4 sdev(int32_t u) const {
        return lds_v4s32(pk + 16 * (3 + 3 * ni + u));
    }
    __device__ __forceinline__ double2 scd(int32_t u) const {
        return lds_v2f64(pk + 16 * (3 + 3 * ni + nv + u));
    }
    // rows a / b: PQ (pq_p, pq_q), PV (pv_p, Q_g), Slack (P_s, Q_g); a scenario
    // array the caller did not pass falls back to the plan constants
    // (packet: PQ {p0, q0}, PV {v0, p0}, Slack {v0, theta0}, Shunt {g, b})
    __device__ __forceinline__ double sdev_a(const int4 dv, int32_t u) const {
        if (dv.x == DEV_PQ && !A.pq_p) return scd(u).x;
        if (dv.x == DEV_PV && !A.pv_p) return scd(u).y;
        return row(2 + 2 * ni + 2 * u);
    }
    __device__ __forceinline__ double sdev_b(const int4 dv, int32_t u) const {
        if (dv.x == DEV_PQ && !A.pq_q) return scd(u).y;
        return row(3 + 2 * ni + 2 * u);
    }
    __device__ __forceinline__ double sdev_c(int32_t u) const { return scd(u).x; }
    __device__ __forceinline__ double sdev_d(int32_t u) const { return scd(u).y; }
    // Incidences [e, e + n), n <= ni, into the staged prefix's places (its
    // values are consumed): records and coefficients into packet units
    // 3 + t and 3 + ni + 2t, this lane's theta_j / V_j into rows 2 + 2t,
    // 3 + 2t.  The device rows and records behind them are untouched.  The
    // active lanes are 0 .. c-1 (scenarios below K), so lane t' < c copies
    // records t', t' + c, ...
    __device__ __forceinline__ void load_chunk(int32_t e, int32_t n) const {
        const unsigned mask = __activemask();
        const int32_t c = __popc(mask);
        __syncwarp(mask);   // every lane is done with the previous chunk
        for (int32_t t = ln; t < n; t += c) {
            const int4 m = __ldg(d.inc_meta + e + t);
            const double4 cf = ldg4(d.inc_coef + e + t);
            asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(pk + 16 * (3 + t)),
                         "r"(m.x), "r"(m.y), "r"(m.z), "r"(m.w) : "memory");
            const uint32_t ca = pk + 16 * (3 + ni + 2 * t);
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(ca), "d"(cf.x), "d"(cf.y)
                         : "memory");
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(ca + 16), "d"(cf.z), "d"(cf.w)
                         : "memory");
        }
        __syncwarp(mask);
        for (int32_t t = 0; t < n; ++t) {
            const int32_t j = smeta(t).x;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(rw + (2 + 2 * t) * WS_ROW_BYTES),
                         "l"(y + (int64_t)j * PF_LANES) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(rw + (3 + 2 * t) * WS_ROW_BYTES),
                         "l"(y + ((int64_t)d.N + j) * PF_LANES) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        // the slot is refilled by TMA (async proxy) two steps later
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
};

__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Issue the copies of one item into the slot at shared address sb.  Lane l
// holds word (l + 2) & 15 of the item's stage record in `rw`: lanes 0..13 the
// codes of rows 0..13, lanes 14 and 15 the packet offset and sizes.  Each
// lane decodes its own row's source address once; the packet goes 16 B per
// lane, the rows 16 lanes per row (two rows per instruction).  One commit
// group per item.
__device__ __forceinline__ void stage_item(const uint32_t sb, const int32_t rw,
                                           const int4* __restrict__ pkt,
                                           const double* const* base, const int32_t keep,
                                           const int lane) {
    const int32_t off = __shfl_sync(0xffffffffu, rw, 14);
    const int32_t meta = __shfl_sync(0xffffffffu, rw, 15);
    const int32_t units = meta & 0xffff, rows = meta >> 16;
    if (lane < units) {
        if (keep)
            cp_async16_pol(sb + WS_ROWS * WS_ROW_BYTES + lane * 16, pkt + off + lane, plan_policy(1));
        else
            cp_async16(sb + WS_ROWS * WS_ROW_BYTES + lane * 16, pkt + off + lane);
    }
    const double* src = nullptr;
    if (lane < rows && rw >= 0) {
        const double* bp = base[(uint32_t)rw >> 29];
        if (bp) src = bp + (int64_t)(rw & 0x1fffffff) * PF_LANES;
    }
    const int half = lane >> 4, chunk = lane & 15;
    for (int rr0 = 0; rr0 < rows; rr0 += 2) {
        const int rr = rr0 + half;
        const double* p = reinterpret_cast<const double*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(src), rr));
        if (rr < rows && p) cp_async16(sb + rr * WS_ROW_BYTES + chunk * 16, p + chunk * 2);
    }
    cp_async_commit();
}

// ---- TMA staging (Blackwell tile::gather4) --------------------------------
//
// The same slot contents, moved by the tensor-memory accelerator instead of
// per-lane cp.async: the scenario rows are rows of one 2-D tensor map
// [rows x 32 doubles] whose base is the lowest of the launch's y / pq_p /
// pq_q / pv_p arrays (every array sits a whole number of 256-byte rows above
// it; launch_staged_kernel checks), so any four rows of the item, from any of
// the arrays, are one gather4.  Lane 0 issues the packet as one bulk copy
// and the rows as <= 3 gathers, all completing on the slot's mbarrier; rows
// 12 and 13 (buses with many staged incidences) go by cp.async, since a
// fourth gather would write past the rows into the packet.
// Opt-in (PF_STAGING=tma), not the default: it executes 4.7 % fewer
// instructions (config 3, ncu: 433 M against 454 M per launch) but measured
// slower on B200 -- config 3 0.581 against 0.574 ms, config 4 0.550 against
// 0.537 (profiles/r02_experiments.md): lane 0 issues every gather (the UTMALDG
// operands must be moved to uniform registers one item at a time) while the
// warp waits, and the kernel is not bound by the staging instructions.
__device__ __forceinline__ void mbar_init(uint32_t m) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(m) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(m) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t m, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "PF_MBW:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra PF_MBW;\n}" ::"r"(m),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t m, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(m), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* tm, uint32_t m,
                                        int4 r) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
        "l"(tm), "r"(m), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w)
        : "memory");
}
constexpr int WS_GATHER_ROWS = 12;   // rows moved by gather4 (3 x 4); the rest by cp.async

// Issue the copies of one item into the slot at sb (mbarrier mb).  rw as in
// stage_item; rb: this warp's row coordinate of entry 0 of each array of the
// staged block (-1: array not passed); crd: the warp's 12-entry coordinate
// scratch.  Rows of arrays not passed (the kernel reads plan constants for
// them) and the padding of the last gather repeat row 0 (theta_i).
__device__ __forceinline__ void stage_item_tma(const uint32_t sb, const uint32_t mb,
                                               const int32_t rw, const int4* __restrict__ pkt,
                                               const int32_t* rb, int32_t* crd,
                                               const CUtensorMap* tm,
                                               const double* const* tm_base,
                                               const int32_t keep, const int lane) {
    const int32_t off = __shfl_sync(0xffffffffu, rw, 14);
    const int32_t meta = __shfl_sync(0xffffffffu, rw, 15);
    const int32_t units = meta & 0xffff, rows = meta >> 16;
    int32_t c = -1;
    if (lane < rows && rw >= 0) {
        const int32_t b = rb[(uint32_t)rw >> 29];
        if (b >= 0) c = b + (rw & 0x1fffffff);
    }
    const int32_t c0 = __shfl_sync(0xffffffffu, c, 0);
    if (c < 0) c = c0;
    if (lane < WS_GATHER_ROWS) crd[lane] = c;
    __syncwarp();
    if (lane == 0) {
        const int32_t ng = (min(rows, WS_GATHER_ROWS) + 3) >> 2;
        mbar_expect_tx(mb, (uint32_t)(ng * 4 * WS_ROW_BYTES + units * 16));
        bulk_g2s(sb + WS_ROWS * WS_ROW_BYTES, pkt + off, (uint32_t)(units * 16), mb,
                 plan_policy(keep));
        const uint32_t ca = smem_u32(crd);
        for (int32_t q = 0; q < ng; ++q)
            gather4(sb + q * 4 * WS_ROW_BYTES, tm, mb, lds_v4s32(ca + 16 * q));
    }
    if (rows > WS_GATHER_ROWS) {   // rows 12, 13: lanes 0-15 and 16-31
        const int32_t r = WS_GATHER_ROWS + (lane >> 4);
        const int32_t cr = __shfl_sync(0xffffffffu, c, r);
        if (r < rows)
            cp_async16(sb + r * WS_ROW_BYTES + (lane & 15) * 16,
                       *tm_base + (int64_t)cr * PF_LANES + (lane & 15) * 2);
    }
    cp_async_commit();
}

// Each warp stages its own next item (no producer warp, no cross-warp
// coupling): at the start of item k it issues item k+1's copies into its
// other slot and loads item k+2's stage record, then waits for item k's
// copies (issued one item earlier) and evaluates from shared memory.
// TMA = true: the slots are filled by stage_item_tma (tensor map tm over the
// rows from tm_base; rb0: row coordinate of entry 0 of block 0 of y, pq_p,
// pq_q, pv_p, -1 for an array not passed), false: by per-lane cp.async.
template <int MODE, int W, int MINB, bool DYN, bool TMA, bool KEEP>
__global__ void __launch_bounds__(32 * W, MINB) k_eval_staged(
    const DevicePlan d, const int32_t K, const int32_t n_groups, const int32_t n_items,
    const double* __restrict__ y, const double* __restrict__ pq_p,
    const double* __restrict__ pq_q, const double* __restrict__ pv_p,
    const int32_t* __restrict__ outage, double* __restrict__ g, double* __restrict__ jv,
    unsigned long long* __restrict__ norms, const uint32_t fd_m, const uint32_t fd_l,
    const __grid_constant__ CUtensorMap tm, const double* __restrict__ tm_base, const int4 rb0) {
    extern __shared__ __align__(128) unsigned char ws_smem[];
    __shared__ __align__(8) unsigned long long s_mb[W][2];   // TMA: one mbarrier per slot
    __shared__ int32_t s_rb[W][4];                           // TMA: rb0 of the staged block
    __shared__ __align__(16) int32_t s_crd[W][WS_GATHER_ROWS];
    __shared__ const double* s_tmb;                          // TMA: tm_base
    if (TMA && threadIdx.x == 0) s_tmb = tm_base;
    if (TMA && (threadIdx.x & 31) == 0) {
        mbar_init(smem_u32(&s_mb[threadIdx.x >> 5][0]));
        mbar_init(smem_u32(&s_mb[threadIdx.x >> 5][1]));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __shared__ double s_tab[PF_TRIG_N * 4];
    __shared__ Scen<PF_LANES> As[W];   // per-warp block base pointers
    __shared__ int32_t s_ctr;          // dynamic mode: next slot claim of this CTA
    __shared__ int32_t s_total;        // dynamic mode: slots of this CTA
    if (DYN && threadIdx.x == 0) {
        s_ctr = 0;
        s_total = (int32_t)blockIdx.x < n_items
                      ? ((n_items - (int32_t)blockIdx.x + (int32_t)gridDim.x - 1) /
                         (int32_t)gridDim.x) * W
                      : 0;
    }
    const double* tab = stage_trig_table(s_tab);   // (its barrier publishes s_ctr, s_total)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Scen<PF_LANES>& A = As[warp];
    unsigned char* slots = ws_smem + (size_t)warp * 2 * WS_SLOT_BYTES;
    const uint32_t slots_u32 = smem_u32(slots);

    // Work: the CTA owns items blockIdx.x, blockIdx.x + G, ... (G =
    // gridDim.x), each a group of W consecutive bus slots; item -> (block,
    // group) by multiply-shift division (fd_m, fd_l: n_groups).
    //  * static (DYN = false): warp w takes slot w of each of the CTA's
    //    items, so a step's item is blockIdx.x + k G;
    //  * dynamic (DYN = true): the warps claim the CTA's slots in order from a
    //    shared counter (q = local item * W + slot), so a warp held up by an
    //    expensive bus (a hub with many incidences past the staged ones)
    //    claims fewer and the load balances inside the CTA.  Claims run two
    //    steps ahead (the staging pipeline) in a per-warp ring.
    // A step is named by x: the item (static) or the claim q (dynamic).
    const int32_t stride = gridDim.x;
    auto blk_of = [&](int32_t it) -> int32_t {
        return (int32_t)((__umulhi((uint32_t)it, fd_m) + (uint32_t)it) >> fd_l);
    };
    auto item_of = [&](int32_t x) -> int32_t {
        if constexpr (DYN) return (int32_t)blockIdx.x + (x / W) * stride;
        else return x;
    };
    auto sub_of = [&](int32_t x) -> int32_t {
        if constexpr (DYN) return x % W;
        else return warp;
    };
    auto live = [&](int32_t x) -> bool {
        if constexpr (DYN) return x < s_total;
        else return x < n_items;
    };
    auto rec_word = [&](int32_t x) -> int32_t {
        if (!live(x)) return -1;
        const int32_t it = item_of(x);
        const int32_t slot = (it - blk_of(it) * n_groups) * W + sub_of(x);
        if (slot >= d.N) return -1;
        const int32_t* rp = reinterpret_cast<const int32_t*>(d.ws_rec) + (int64_t)slot * WS_REC_WORDS +
                            ((lane + 2) & 15);
        if (!KEEP) return __ldg(rp);
        int32_t v;
        asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;"
                     : "=r"(v)
                     : "l"(rp), "l"(plan_policy(1)));
        return v;
    };
    // base pointers (y, pq_p, pq_q, pv_p) of the block being staged, per
    // warp in shared memory, refreshed when the staged block changes
    __shared__ const double* s_base[W][4];
    __shared__ int32_t s_sblk[W];
    if (lane == 0) s_sblk[warp] = -1;
    __syncwarp();
    auto issue = [&](int32_t x, int32_t rw, int s) {
        const uint32_t sb = slots_u32 + s * WS_SLOT_BYTES;
        const uint32_t mb = smem_u32(&s_mb[warp][s]);
        if (live(x) && __shfl_sync(0xffffffffu, rw, 14) >= 0) {
            const int32_t bb = blk_of(item_of(x));
            if (bb != s_sblk[warp]) {
                __syncwarp();
                if (lane == 0) s_sblk[warp] = bb;
                if (lane < 4) {
                    const int64_t n = lane == 0 ? d.n_var : lane == 3 ? d.G : d.P;
                    if constexpr (TMA) {
                        const int32_t r = lane == 0 ? rb0.x : lane == 1 ? rb0.y : lane == 2 ? rb0.z : rb0.w;
                        s_rb[warp][lane] = r >= 0 ? r + (int32_t)(bb * n) : -1;
                    } else {
                        const double* a = lane == 0 ? y : lane == 1 ? pq_p : lane == 2 ? pq_q : pv_p;
                        s_base[warp][lane] = a ? a + (int64_t)bb * n * PF_LANES : nullptr;
                    }
                }
                __syncwarp();
            }
            if constexpr (TMA)
                stage_item_tma(sb, mb, rw, d.ws_pkt, s_rb[warp], s_crd[warp], &tm, &s_tmb,
                               KEEP, lane);
            else
                stage_item(sb, rw, d.ws_pkt, s_base[warp], KEEP, lane);
        } else {
            if (TMA && lane == 0) mbar_arrive(mb);   // complete the slot's phase
            cp_async_commit();                       // keep one group per step
        }
    };

    // norms: each warp keeps a per-lane running max over its items of the
    // current scenario block and max-es it into norms[] when it moves to a
    // later block (a warp's blocks never go back, in either mode; integer
    // max of |g| bit patterns: exact, order-independent).  No CTA barrier:
    // warps cross block boundaries independently.  Per-lane state touched
    // once per item lives in shared memory, leaving the registers to the
    // evaluation (B200, config 3: 0.598 -> 0.593 ms).
    __shared__ unsigned long long s_nrm[W][32];
    __shared__ int32_t s_out[3][W][32];
    __shared__ int32_t s_cur[W][32];
    unsigned long long& nrm = s_nrm[warp][lane];
    int32_t& out_l = s_out[0][warp][lane];
    int32_t& out_h = s_out[1][warp][lane];
    int32_t& out_k = s_out[2][warp][lane];
    nrm = 0;
    out_l = out_h = out_k = -1;   // lane's outaged branch and its buses
    // the warp's current block: a register in static mode, shared memory in
    // dynamic mode (whose claim bookkeeping needs the register)
    int32_t cur_reg = -1;
    int32_t& cur = DYN ? s_cur[warp][lane] : cur_reg;
    cur = -1;
    auto flush = [&](int32_t blk) {
        if (MODE & NORM) {
            const int32_t s = blk * PF_LANES + lane;
            if (s < K && nrm) atomicMax(norms + s, nrm);
        }
        nrm = 0;
    };
    auto enter_block = [&](int32_t blk) {
        if (cur >= 0) flush(cur);
        cur = blk;
        if (lane == 0) {
            const int64_t b = blk;
            A.y = y + b * d.n_var * PF_LANES;
            A.g = g ? g + b * d.n_var * PF_LANES : nullptr;
            A.j = jv ? jv + b * d.nnz * PF_LANES : nullptr;
            A.pq_p = pq_p ? pq_p + b * d.P * PF_LANES : nullptr;
            A.pq_q = pq_q ? pq_q + b * d.P * PF_LANES : nullptr;
            A.pv_p = pv_p ? pv_p + b * d.G * PF_LANES : nullptr;
        }
        const int32_t s = blk * PF_LANES + lane;
        out_l = (outage && s < K) ? __ldg(outage + s) : -1;
        // an index outside [0, L) (rejected by the host paths) reads no memory
        if ((uint32_t)out_l >= (uint32_t)d.L) out_l = -1;
        out_h = out_l >= 0 ? __ldg(d.bus_h + out_l) : -1;
        out_k = out_l >= 0 ? __ldg(d.bus_k + out_l) : -1;
        __syncwarp();
    };
    // evaluate step k (slot `slot` of block `blk`) from its staging slot
    auto evaluate = [&](int32_t k, int32_t blk, int32_t slot) {
        if constexpr (TMA) mbar_wait(smem_u32(&s_mb[warp][k & 1]), (uint32_t)(k >> 1) & 1);
        cp_async_wait<1>();   // this step's group has landed (own lanes)
        __syncwarp();         // ... and every lane's
        unsigned char* sb = slots + (k & 1) * WS_SLOT_BYTES;
        const int4* pk = reinterpret_cast<const int4*>(sb + WS_ROWS * WS_ROW_BYTES);
        const int4 cnt = pk[2];
        // does any lane's outaged branch end at this bus?  (usually not: then
        // the per-incidence outage test is skipped)
        const bool ochk = __any_sync(0xffffffffu, slot < d.N && (cnt.z == out_h || cnt.z == out_k));
        if (slot < d.N && blk * PF_LANES + lane < K) {
            const uint32_t sbu = slots_u32 + (k & 1) * WS_SLOT_BYTES;
            const StagedSrc src{{d, A, A.y + lane, cnt.z, lane}, sbu + lane * 8,
                                sbu + WS_ROWS * WS_ROW_BYTES, cnt.x, cnt.y};
            // (the running max is read from shared memory after the bus, not
            // held in registers through it)
            const unsigned long long r = eval_bus_src<MODE, PF_LANES>(
                d, tab, cnt.z, src, A, lane, out_l,
                GlobalJ<PF_LANES>{A.j ? A.j + lane : nullptr}, ochk);
            nrm = max(nrm, r);
        }
        __syncwarp();         // slot reads done before it is refilled
    };

    if constexpr (DYN) {
        __shared__ int32_t s_q[W][4];      // claims of steps k .. k+2 (ring)
        auto claim = [&]() -> int32_t {
            int32_t q = 0;
            if (lane == 0) q = atomicAdd(&s_ctr, 1);
            return __shfl_sync(0xffffffffu, q, 0);
        };
        {   // prologue: step 0's copies in flight, step 1's record in a register
            const int32_t q0 = claim();
            issue(q0, rec_word(q0), 0);
            const int32_t q1 = claim();
            if (lane == 0) {
                s_q[warp][0] = q0;
                s_q[warp][1] = q1;
            }
        }
        __syncwarp();
        int32_t rw_next = rec_word(s_q[warp][1]);
        for (int32_t k = 0;; ++k) {
            const int32_t q = s_q[warp][k & 3];
            if (!live(q)) break;
            const int32_t item = item_of(q);
            const int32_t blk = blk_of(item);
            if (blk != cur) enter_block(blk);
            // claim step k+2; start step k+1's copies into the other slot
            // (its previous contents, step k-1, were consumed in the previous
            // iteration); load step k+2's record
            const int32_t q2 = claim();
            if (lane == 0) s_q[warp][(k + 2) & 3] = q2;
            issue(s_q[warp][(k + 1) & 3], rw_next, (k + 1) & 1);
            rw_next = rec_word(q2);
            evaluate(k, blk, (item - blk * n_groups) * W + q % W);
        }
    } else {
        // prologue: item 0's copies in flight, item 1's record in a register
        issue(blockIdx.x, rec_word(blockIdx.x), 0);
        int32_t rw_next = rec_word(blockIdx.x + stride);
        int32_t k = 0;
        for (int32_t item = blockIdx.x; item < n_items; item += stride, ++k) {
            const int32_t blk = blk_of(item);
            if (blk != cur) enter_block(blk);
            // next item's copies into the other slot (its previous contents,
            // item k-1, were consumed in the previous iteration), then the
            // record of the item after it
            issue(item + stride, rw_next, (k + 1) & 1);
            rw_next = rec_word(item + 2 * stride);
            evaluate(k, blk, (item - blk * n_groups) * W + warp);
        }
    }
    cp_async_wait<0>();
    if (cur >= 0) flush(cur);
}

// Single grid: one CTA per chunk of consecutive buses (plan-built so that
// its incidences, Jacobian rows and parallel-branch slots fit the shared-memory
// caps), in three phases:
//   0: one thread per bus loads its header, state and first two devices
//      (registers) and publishes theta, V and the theta-block width;
//   A: one thread per incidence computes the ten values of its terminal
//      (pflow kernels.py:79-163) into shared memory and writes its four
//      off-diagonal Jacobian values into the CTA's staged rows (0.0 + v,
//      the reference's assembly) unless a parallel branch shares them;
//   B: each bus thread folds its incidences in list order (the reference's
//      join and assembly association), adds the parallel-branch values in
//      order and its devices, and writes g and its diagonal / device values;
// then the CTA copies its staged rows g_p[b0..b1), g_q[b0..b1) out with two
// TMA bulk copies.  A chunk whose single bus exceeds the caps (a hub) is
// evaluated serially by one thread from global memory.  Launched with
// programmatic stream serialisation (launch_single_mode): plan data is read
// before griddepcontrol.wait, the state and every output after it.
struct SingleSrc : GlobalSrc<1> {
    static constexpr bool kSplit = true;
    static constexpr bool kRegDev = true;
    const double* fold;                // [n_inc of chunk][6] {fp, fq, pt, pv, qt, qv}
    const double* dupv;                // [dup slots][4] {opt, opv, oqt, oqv}
    int32_t E0;
    int4 h0, h1;
    double thi, vi;
    int4 dv0, dv1;                     // first two devices
    double a0, b0, c0, d0, a1, b1, c1, d1;
    __device__ __forceinline__ int4 hdr0() const { return h0; }
    __device__ __forceinline__ int4 hdr1() const { return h1; }
    __device__ __forceinline__ double th_i() const { return thi; }
    __device__ __forceinline__ double v_i() const { return vi; }
    __device__ __forceinline__ IncVals vals(int32_t e) const {
        const double2* p = reinterpret_cast<const double2*>(fold + 6 * (e - E0));
        const double2 a = p[0], b = p[1], c = p[2];
        IncVals v;
        v.fp = a.x; v.fq = a.y;
        v.pt = b.x; v.pv = b.y;
        v.qt = c.x; v.qv = c.y;
        return v;
    }
    __device__ __forceinline__ IncVals dup(int32_t e) const {
        const int32_t slot = (__ldg(&d.sg_inc[e].y) >> SG_DUP_SHIFT) & SG_FIELD_MASK;
        const double2* p = reinterpret_cast<const double2*>(dupv + 4 * slot);
        const double2 a = p[0], b = p[1];
        IncVals v;
        v.opt = a.x; v.opv = a.y;
        v.oqt = b.x; v.oqv = b.y;
        return v;
    }
    __device__ __forceinline__ int4 dev(int32_t t, int32_t u) const {
        return u == 0 ? dv0 : u == 1 ? dv1 : GlobalSrc<1>::dev(t, u);
    }
    __device__ __forceinline__ double dev_a(const int4 dv, int32_t u) const {
        return u == 0 ? a0 : u == 1 ? a1 : GlobalSrc<1>::dev_a(dv, u);
    }
    __device__ __forceinline__ double dev_b(const int4 dv, int32_t u) const {
        return u == 0 ? b0 : u == 1 ? b1 : GlobalSrc<1>::dev_b(dv, u);
    }
    __device__ __forceinline__ double dev_c(const int4 dv, int32_t u) const {
        return u == 0 ? c0 : u == 1 ? c1 : GlobalSrc<1>::dev_c(dv, u);
    }
    __device__ __forceinline__ double dev_d(const int4 dv, int32_t u) const {
        return u == 0 ? d0 : u == 1 ? d1 : GlobalSrc<1>::dev_d(dv, u);
    }
};

// Device u's record and operands into registers, in two steps: the record
// and the plan constants (PQ p0 / q0, PV p0 / v0, Slack v0 / theta0, Shunt
// g / b) may be read before the programmatic-launch wait; the operands that
// live in y (PV Q_g, Slack P_s / Q_g) only after it.  Types a device does
// not use are left untouched: no out-of-range reads.
__device__ __forceinline__ void single_dev_plan(const GlobalSrc<1>& gs, const DevicePlan& d,
                                                int32_t t, bool have, int4& dv, double& a,
                                                double& b, double& c, double& dd) {
    dv = have ? __ldg(d.dev_list + t) : make_int4(-1, 0, 0, 0);
    a = b = c = dd = 0.0;
    if (dv.x == DEV_PQ) {
        a = gs.dev_a(dv, 0);
        b = gs.dev_b(dv, 0);
    } else if (dv.x == DEV_PV) {
        a = gs.dev_a(dv, 0);
    }
    if (dv.x == DEV_PV || dv.x == DEV_SLACK || dv.x == DEV_SHUNT) c = gs.dev_c(dv, 0);
    if (dv.x == DEV_SLACK || dv.x == DEV_SHUNT) dd = gs.dev_d(dv, 0);
}

__device__ __forceinline__ void single_dev_state(const GlobalSrc<1>& gs, const int4 dv, double& a,
                                                 double& b) {
    if (dv.x == DEV_PV) {
        b = gs.dev_b(dv, 0);
    } else if (dv.x == DEV_SLACK) {
        a = gs.dev_a(dv, 0);
        b = gs.dev_b(dv, 0);
    }
}

// shared-memory layout of k_eval_single (doubles, then ints)
constexpr int SG_SMEM_FOLD = 0;
constexpr int SG_SMEM_DUP = SG_SMEM_FOLD + 6 * SG_CAP_INC;
constexpr int SG_SMEM_J = SG_SMEM_DUP + 4 * SG_CAP_DUP;
constexpr int SG_SMEM_TH = SG_SMEM_J + SG_CAP_J + 2;   // +2: 16-byte phase shifts
constexpr int SG_SMEM_V = SG_SMEM_TH + SG_CAP_BUS;
constexpr int SG_SMEM_DOUBLES = SG_SMEM_V + SG_CAP_BUS;
constexpr size_t SG_SMEM_BYTES = 8 * (size_t)SG_SMEM_DOUBLES + 4 * (size_t)SG_CAP_BUS;

// Copy n doubles from shared to global memory: the 16-byte aligned middle
// with one TMA bulk copy (cp.async.bulk), a misaligned head / odd tail with
// plain stores.  src and dst share their 16-byte phase (see the staging).
__device__ __forceinline__ void bulk_out(double* dst, const double* src, int32_t n) {
    int32_t k0 = (int32_t)((reinterpret_cast<uintptr_t>(dst) >> 3) & 1);
    if (k0 > n) k0 = n;
    if (k0) dst[0] = src[0];
    const int32_t pairs = (n - k0) >> 1;
    if ((n - k0) & 1) dst[n - 1] = src[n - 1];
    if (pairs > 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t saddr = static_cast<uint32_t>(__cvta_generic_to_shared(src + k0));
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     :: "l"(dst + k0), "r"(saddr), "r"(16 * pairs) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
}

__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// CTA max -> one integer atomicMax of the |g| bit pattern into the plan's
// accumulator (exact, order-independent); the last CTA moves it to *norm and
// re-arms accumulator and counter for the next launch.  Two steps: every
// warp posts its max to red[] (norm_post), and after a barrier one thread
// publishes (norm_publish); release / acquire atomics order the max before
// the count.  (A memset of *norm before the launch plus a plain atomicMax
// measured 2.5 us slower per evaluation inside a CUDA graph.)
__device__ __forceinline__ void norm_post(unsigned long long nrm, unsigned long long* red) {
    // warp max of a 64-bit value with two 32-bit reductions (REDUX): the
    // high words first, then the low words of the lanes holding that high
    const unsigned hi = (unsigned)(nrm >> 32);
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? (unsigned)nrm : 0u);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ((unsigned long long)mh << 32) | ml;
}
__device__ __forceinline__ void norm_publish(const DevicePlan& d, const unsigned long long* red,
                                             unsigned long long* norm) {
    {
        unsigned long long mx = red[0];
        for (int w = 1; w < SG_THREADS / 32; ++w) mx = max(mx, red[w]);
        atomicMax(d.sg_acc, mx);
        unsigned int done;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                     : "=r"(done) : "l"(d.sg_count) : "memory");
        if (done == gridDim.x - 1) {
            unsigned long long v;
            asm volatile("atom.acquire.gpu.global.exch.b64 %0, [%1], 0;"
                         : "=l"(v) : "l"(d.sg_acc) : "memory");
            *norm = v;
            *d.sg_count = 0;
        }
    }
}

#ifdef PF_X_TRACE
// dev probe (scripts/dbg/sg_trace.py): %globaltimer at phase boundaries of
// every CTA, thread 0's view (after each barrier every thread is there)
__device__ unsigned long long g_sg_trace[4096 * 8];
__device__ __forceinline__ void sg_stamp(int k) {
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_sg_trace[blockIdx.x * 8 + k] = t;
    }
}
#define SG_STAMP(k) sg_stamp(k)
#else
#define SG_STAMP(k)
#endif

template <int MODE>
__global__ void __launch_bounds__(SG_THREADS, SG_MINB) k_eval_single(const DevicePlan d,
                                                            const double* __restrict__ y,
                                                            double* __restrict__ g,
                                                            double* __restrict__ jv,
                                                            unsigned long long* __restrict__ norm) {
    extern __shared__ __align__(16) double sg[];
    __shared__ unsigned long long red[SG_THREADS / 32];
    __shared__ double s_tab[PF_TRIG_N * 4];
    const int32_t N = d.N;
    const int t = threadIdx.x;
    // Programmatic dependent launch (launch_single_mode): the next kernel in
    // the stream may start while this one runs; it reads only plan data until
    // its griddepcontrol.wait, after which everything the preceding kernel
    // wrote (y included, whoever produced it) is visible.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    SG_STAMP(0);
    // Every global access is a ~0.5 us round trip here (one wave, one
    // dependent chain per CTA), so loads are issued level by level: chunk
    // record and trig table first, then everything that depends only on
    // the chunk record, and the table reaches shared memory at the first
    // barrier (it is not read before).
    const int4 c0 = __ldg(d.sg_chunk + 2 * blockIdx.x);
    const int4 c1 = __ldg(d.sg_chunk + 2 * blockIdx.x + 1);
    constexpr int TAB16 = PF_TRIG_N * 4 / 2;
    static_assert(TAB16 <= 2 * SG_THREADS, "trig table staging");
// trig table: two 16-byte loads per thread into registers now, stored to
    // shared memory before the first barrier (cp.async staging instead cost
    // 1.4 us per evaluation in the graph: its completion wait lands after
    // griddepcontrol.wait, on the critical path)
    double2 tv[2];
    for (int r = 0; r < 2; ++r)
        tv[r] = t + r * SG_THREADS < TAB16
                    ? __ldg(reinterpret_cast<const double2*>(pf_trig_tab) + t + r * SG_THREADS)
                    : make_double2(0.0, 0.0);
    const double* tab = s_tab;
    const int32_t b0 = c0.x, b1 = c0.y & ~SG_BIG, E0 = c0.z, E1 = c0.w;
    const Scen<1> A{y, nullptr, nullptr, nullptr, g, jv, -1};
    unsigned long long nrm = 0;
    if (c0.y & SG_BIG) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int r = 0; r < 2; ++r)
            if (t + r * SG_THREADS < TAB16)
                reinterpret_cast<double2*>(s_tab)[t + r * SG_THREADS] = tv[r];
        __syncthreads();
        if (t == 0) nrm = eval_bus<MODE, 1>(d, tab, b0, A, 0, -1);
    } else {
        double* fold = sg + SG_SMEM_FOLD;
        double* dupv = sg + SG_SMEM_DUP;
        // Staged rows keep the 16-byte phase of their global destination, so
        // the copy-out is one TMA bulk copy per range (plus a lone head /
        // tail value).  jp / jq start at element 0 or 1 of their slot.
        const int32_t lp = c1.y - c1.x, lq = c1.w - c1.z;
        const int32_t sp = (int32_t)((reinterpret_cast<uintptr_t>(jv + c1.x) >> 3) & 1);
        const int32_t sq0 = sp + lp;
        const int32_t sq = sq0 + ((sq0 ^ (int32_t)(reinterpret_cast<uintptr_t>(jv + c1.z) >> 3)) & 1);
        double* jpb = sg + SG_SMEM_J + sp;
        double* jqb = sg + SG_SMEM_J + sq;
        double* bth = sg + SG_SMEM_TH;
        double* bv = sg + SG_SMEM_V;
        int32_t* bnb = reinterpret_cast<int32_t*>(sg + SG_SMEM_DOUBLES);
        const int32_t i = b0 + t;
        const bool own = i < b1;
        // plan data: the first incidence's record, the bus header, the first
        // two devices and their constant operands
        // (chunks hold at most 2 SG_THREADS incidences: two per thread)
        static_assert(SG_CAP_INC <= 2 * SG_THREADS, "two incidences per thread");
        const int32_t ea = E0 + t, eb = ea + SG_THREADS;
        int4 ra = make_int4(0, 0, 0, 0), rb = make_int4(0, 0, 0, 0);
        double4 ca = make_double4(0.0, 0.0, 0.0, 0.0);
        if (ea < E1) {
            ra = __ldg(d.sg_inc + ea);
            ca = ldg4(d.inc_coef + ea);
        }
        double4 cb_reg = make_double4(0.0, 0.0, 0.0, 0.0);
        if (eb < E1) {
            rb = __ldg(d.sg_inc + eb);
            cb_reg = ldg4(d.inc_coef + eb);
        }
        SingleSrc src{{d, A, y, i, 0}, fold, dupv, E0, make_int4(0, 0, 0, 0),
                      make_int4(0, 0, 0, 0), 0.0, 0.0};
        if (own) {
            src.h0 = __ldg(d.bus_row + 2 * i);
            src.h1 = __ldg(d.bus_row + 2 * i + 1);
            const int32_t t0 = src.h1.z, nd = src.h1.w - src.h1.z;
            single_dev_plan(src, d, t0, nd > 0, src.dv0, src.a0, src.b0, src.c0, src.d0);
            single_dev_plan(src, d, t0 + 1, nd > 1, src.dv1, src.a1, src.b1, src.c1, src.d1);
        }
        for (int r = 0; r < 2; ++r)
            if (t + r * SG_THREADS < TAB16)
                reinterpret_cast<double2*>(s_tab)[t + r * SG_THREADS] = tv[r];
        // the second incidence's coefficients wait in its own fold slot (free
        // until phase A writes it): loaded now, before griddepcontrol.wait,
        // instead of a global round trip inside phase A
        if (eb < E1) {
            double2* cs = reinterpret_cast<double2*>(fold + 6 * (eb - E0));
            cs[0] = make_double2(cb_reg.x, cb_reg.y);
            cs[1] = make_double2(cb_reg.z, cb_reg.w);
        }
        // state: after the preceding kernel's writes are visible
        SG_STAMP(1);
        asm volatile("griddepcontrol.wait;" ::: "memory");
        SG_STAMP(2);
        double tja = 0.0, wja = 0.0, tjb = 0.0, wjb = 0.0;
        if (ea < E1) {
            tja = __ldg(y + ra.x);
            wja = __ldg(y + N + ra.x);
        }
        if (eb < E1) {
            tjb = __ldg(y + rb.x);
            wjb = __ldg(y + N + rb.x);
        }
        if (own) {
            src.thi = __ldg(y + i);
            src.vi = __ldg(y + N + i);
            single_dev_state(src, src.dv0, src.a0, src.b0);
            single_dev_state(src, src.dv1, src.a1, src.b1);
            bth[t] = src.thi;
            bv[t] = src.vi;
            bnb[t] = src.h0.z;
        }
        __syncthreads();
        SG_STAMP(3);
        auto incidence = [&](int32_t e, int4 r, double4 c, double tj, double wj) {   // phase A
            const int32_t o = r.y & SG_FIELD_MASK;
            const int4 m = make_int4(r.x, -1, r.y & KSIDE, 0);
            const IncVals v = inc_vals<1>(tab, m, c, bth[o], bv[o], tj, wj, -1);
            double2* f = reinterpret_cast<double2*>(fold + 6 * (e - E0));
            if (MODE & (RES | NORM)) f[0] = make_double2(v.fp, v.fq);
            if (MODE & JAC) {
                f[1] = make_double2(v.pt, v.pv);
                f[2] = make_double2(v.qt, v.qv);
                if (r.y & SOLO) {
                    const int32_t w = bnb[o];
                    jpb[r.z] = 0.0 + v.opt;
                    jpb[r.z + w] = 0.0 + v.opv;
                    jqb[r.w] = 0.0 + v.oqt;
                    jqb[r.w + w] = 0.0 + v.oqv;
                } else {
                    double2* u = reinterpret_cast<double2*>(
                        dupv + 4 * ((r.y >> SG_DUP_SHIFT) & SG_FIELD_MASK));
                    u[0] = make_double2(v.opt, v.opv);
                    u[1] = make_double2(v.oqt, v.oqv);
                }
            }
        };
        if (ea < E1) incidence(ea, ra, ca, tja, wja);
        if (eb < E1) {
            const double2* cs = reinterpret_cast<const double2*>(fold + 6 * (eb - E0));
            const double2 c01 = cs[0], c23 = cs[1];
            incidence(eb, rb, make_double4(c01.x, c01.y, c23.x, c23.y), tjb, wjb);
        }
        __syncthreads();
        SG_STAMP(4);
        if (own)   // phase B
            nrm = eval_bus_src<MODE, 1>(d, tab, i, src, A, 0, -1,
                                        StagedJ{jpb, jqb, jv, c1.x, c1.z});
        if (MODE & NORM) norm_post(nrm, red);
        if (MODE & (JAC | NORM)) __syncthreads();
        SG_STAMP(5);
        // three warps in parallel: the two staged row ranges out by TMA bulk
        // copies (warps 0, 1) and the norm protocol (warp 2); B200 graph of
        // 100 evaluations: config 0 5.03 -> 4.87 us, config 2 7.66 -> 7.60
        static_assert(SG_THREADS >= 96, "warps 0-2 split the epilogue");
        if (MODE & JAC) {
            if (t == 0) bulk_out(jv + c1.x, jpb, lp);
            if (t == 32) bulk_out(jv + c1.z, jqb, lq);
        }
        if (MODE & NORM) {
            if (t == 64) norm_publish(d, red, norm);
        }
        SG_STAMP(6);
        if (MODE & JAC) {
            if (t == 0 || t == 32) bulk_wait();   // smem must outlive the copy's reads
        }
        SG_STAMP(7);
        return;
    }
    if (MODE & NORM) {
        __syncthreads();
        norm_post(nrm, red);
        __syncthreads();
        if (t == 0) norm_publish(d, red, norm);
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

// Blocked <-> scenario-major transposes through a 32 x 33 shared tile:
// both the 256-byte blocked rows and the scenario-major rows move coalesced.
// Tile (blockIdx.x: 32 entries, blockIdx.y: scenario block).
__global__ void k_batch_unblock(int32_t K, int32_t n_e, const double* __restrict__ src,
                                double* __restrict__ dst, double alpha) {
    __shared__ double tile[32][33];
    const int32_t e0 = blockIdx.x * 32, blk = blockIdx.y;
    const int lane = threadIdx.x & 31, row = threadIdx.x >> 5;   // 8 warps
    const double* sb = src + (int64_t)blk * n_e * PF_LANES;
    for (int r = row; r < 32; r += 8) {
        const int32_t e = e0 + r;
        tile[r][lane] = e < n_e ? sb[(int64_t)e * PF_LANES + lane] : 0.0;
    }
    __syncthreads();
    for (int r = row; r < 32; r += 8) {
        const int32_t s = blk * PF_LANES + r, e = e0 + lane;
        if (s < K && e < n_e) dst[(int64_t)s * n_e + e] = alpha * tile[lane][r];
    }
}

__global__ void k_batch_update(int32_t K, int32_t n_e, double* __restrict__ y,
                               const double* __restrict__ dx, const int32_t* __restrict__ active) {
    __shared__ double tile[32][33];
    const int32_t e0 = blockIdx.x * 32, blk = blockIdx.y;
    const int lane = threadIdx.x & 31, row = threadIdx.x >> 5;
    for (int r = row; r < 32; r += 8) {
        const int32_t s = blk * PF_LANES + r, e = e0 + lane;
        tile[r][lane] = (s < K && e < n_e) ? dx[(int64_t)s * n_e + e] : 0.0;
    }
    __syncthreads();
    double* yb = y + (int64_t)blk * n_e * PF_LANES;
    const int32_t s = blk * PF_LANES + lane;
    const bool on = s < K && (!active || __ldg(active + s));
    for (int r = row; r < 32; r += 8) {
        const int32_t e = e0 + r;
        if (on && e < n_e) yb[(int64_t)e * PF_LANES + lane] += tile[lane][r];
    }
}

inline unsigned grid_for(int64_t n, int threads) {
    return (unsigned)((n + threads - 1) / threads);
}

}  // namespace

// ---- launchers --------------------------------------------------------------

// Per-device launch configuration of one kernel instantiation: the
// dynamic-shared-memory opt-in (a per-context function attribute), the SM
// count and the occupancy, set up once per device ordinal (std::call_once:
// concurrent first launches from several host threads are safe), with the
// CUDA status kept and returned on every launch.
constexpr int PF_MAX_DEVICES = 64;
struct DevLaunchCfg {
    std::once_flag once;
    cudaError_t err = cudaSuccess;
    int ctas = 1;
    int sms = 1;
};

template <class Kern>
static cudaError_t device_cfg(DevLaunchCfg (&tab)[PF_MAX_DEVICES], Kern kern, int threads,
                              size_t dyn_smem, const DevLaunchCfg** out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= PF_MAX_DEVICES) return cudaErrorInvalidDevice;
    DevLaunchCfg& c = tab[dev];
    std::call_once(c.once, [&] {
        c.err = cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
        if (c.err == cudaSuccess && dyn_smem > 48 * 1024)
            c.err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)dyn_smem);
        if (c.err == cudaSuccess)
            c.err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.ctas, kern, threads,
                                                                  dyn_smem);
        if (c.ctas < 1) c.ctas = 1;
    });
    *out = &c;
    return c.err;
}

template <int MODE>
static cudaError_t launch_single_mode(const DevicePlan& d, const double* y, double* g, double* j,
                                      double* norm, cudaStream_t st) {
    static DevLaunchCfg tab[PF_MAX_DEVICES];
    const DevLaunchCfg* dc = nullptr;
    cudaError_t e = device_cfg(tab, k_eval_single<MODE>, SG_THREADS, SG_SMEM_BYTES, &dc);
    if (e != cudaSuccess) return e;
    // programmatic stream serialisation: see k_eval_single
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(d.sg_chunks);
    cfg.blockDim = dim3(SG_THREADS);
    cfg.dynamicSmemBytes = SG_SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_eval_single<MODE>, d, y, g, j,
                              reinterpret_cast<unsigned long long*>(norm));
}

cudaError_t launch_eval_single(const DevicePlan& d, const double* y, double* g, double* j,
                               double* norm, cudaStream_t st) {
    if (d.N == 0) {
        if (norm) return cudaMemsetAsync(norm, 0, sizeof(double), st);
        return cudaSuccess;
    }
    const int mode = (g ? RES : 0) | (j ? JAC : 0) | (norm ? NORM : 0);
#define PF_S(M) launch_single_mode<M>(d, y, g, j, norm, st)
    cudaError_t e = cudaSuccess;
    switch (mode) {
        case RES: e = PF_S(RES); break;
        case JAC: e = PF_S(JAC); break;
        case RES | JAC: e = PF_S(RES | JAC); break;
        case NORM: e = PF_S(NORM); break;
        case RES | NORM: e = PF_S(RES | NORM); break;
        case JAC | NORM: e = PF_S(JAC | NORM); break;
        case RES | JAC | NORM: e = PF_S(RES | JAC | NORM); break;
        default: return cudaSuccess;
    }
#undef PF_S
    if (e != cudaSuccess) return e;
    count_launch();
    return cudaGetLastError();
}

// 12 warps per CTA, 2 CTAs per SM: 24 warps at 80 registers, no spills.
// Measured on B200 (config 3, ms per K=256 launch): 12x2 0.735, 8x3 0.739,
// 6x4 0.740, 4x6 0.743, 24x1 0.736, 16x1 (98 registers) 0.924; fewer
// registers (8x4, 64 registers, spills) 0.80; more (8x2, 108) 0.96.
constexpr int BATCH_W = 12;
constexpr int BATCH_MINB = 2;
template <int MODE>
static cudaError_t launch_batched_mode(const DevicePlan& d, int32_t K, const double* y,
                                       const double* pq_p, const double* pq_q,
                                       const double* pv_p, const int32_t* outage, double* g,
                                       double* j, double* norms, cudaStream_t st) {
    static DevLaunchCfg tab[PF_MAX_DEVICES];
    const DevLaunchCfg* dc = nullptr;
    cudaError_t e = device_cfg(tab, k_eval_batched<MODE, BATCH_W, BATCH_MINB>, 32 * BATCH_W, 0,
                               &dc);
    if (e != cudaSuccess) return e;
    const int ctas = dc->ctas, sms = dc->sms;
    const int32_t n_groups = (d.N + BATCH_W - 1) / BATCH_W;
    const int64_t n_items64 = (int64_t)n_groups * ((K + PF_LANES - 1) / PF_LANES);
    if (n_items64 >= (1ll << 31)) return cudaErrorInvalidValue;
    const int32_t n_items = (int32_t)n_items64;
    const int grid = (int)std::min<int64_t>(std::min<int64_t>(n_items, n_groups),
                                            (int64_t)ctas * sms);
    k_eval_batched<MODE, BATCH_W, BATCH_MINB><<<grid, 32 * BATCH_W, 0, st>>>(
        d, K, n_groups, n_items, y, pq_p, pq_q, pv_p, outage, g, j,
        reinterpret_cast<unsigned long long*>(norms));
    return cudaSuccess;
}

// Staged kernel shape (pf_internal.cuh WS_W, WS_MINB): two 4 KB slots per
// warp in dynamic shared memory.
constexpr size_t WS_SMEM = (size_t)WS_W * 2 * WS_SLOT_BYTES;

// The row tensor map of a launch (stage_item_tma): base = the lowest of the
// arrays passed, every array a whole number of 256-byte rows above it, all
// rows addressable with int32 coordinates.  Encoded on the host per launch
// (a pure host call, ~1 us); false when the arrays do not qualify or the
// driver lacks the entry point, and the launch uses cp.async staging.
static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

static bool use_tma_staging() {
    static const bool v = [] {
        const char* e = getenv("PF_STAGING");
        return e && e[0] == 't';   // "tma": gather4 staging (opt-in, see k_eval_staged)
    }();
    return v;
}

static bool row_tensor_map(const DevicePlan& d, int32_t K, const double* y, const double* pq_p,
                           const double* pq_q, const double* pv_p, CUtensorMap* tm,
                           const double** base, int4* rb0) {
    if (!use_tma_staging()) return false;
    const auto enc = tma_encoder();
    if (!enc || !y) return false;
    const int64_t nblk = (K + PF_LANES - 1) / PF_LANES;
    const double* arr[4] = {y, pq_p, pq_q, pv_p};
    const int64_t len[4] = {d.n_var, d.P, d.P, d.G};
    uintptr_t lo = UINTPTR_MAX;
    for (int a = 0; a < 4; ++a)
        if (arr[a]) lo = std::min(lo, reinterpret_cast<uintptr_t>(arr[a]));
    if (lo % 16) return false;
    int32_t r[4];
    int64_t rows = 1;
    for (int a = 0; a < 4; ++a) {
        r[a] = -1;
        if (!arr[a]) continue;
        const uintptr_t off = reinterpret_cast<uintptr_t>(arr[a]) - lo;
        if (off % WS_ROW_BYTES) return false;
        const int64_t r0 = (int64_t)(off / WS_ROW_BYTES), end = r0 + nblk * len[a];
        if (end >= (1ll << 31)) return false;
        r[a] = (int32_t)r0;
        rows = std::max(rows, end);
    }
    cuuint64_t gdim[2] = {(cuuint64_t)PF_LANES, (cuuint64_t)rows};
    cuuint64_t gstr[1] = {(cuuint64_t)WS_ROW_BYTES};
    cuuint32_t box[2] = {(cuuint32_t)PF_LANES, 1};
    cuuint32_t es[2] = {1, 1};
    if (enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, reinterpret_cast<void*>(lo), gdim, gstr, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    *base = reinterpret_cast<const double*>(lo);
    *rb0 = make_int4(r[0], r[1], r[2], r[3]);
    return true;
}

template <int MODE, bool DYN, bool TMA, bool KEEP>
static cudaError_t launch_staged_kernel(const DevicePlan& d, int32_t K, const double* y,
                                      const double* pq_p, const double* pq_q,
                                      const double* pv_p, const int32_t* outage, double* g,
                                      double* j, double* norms, const CUtensorMap& tm,
                                      const double* tm_base, int4 rb0, cudaStream_t st) {
    auto kern = k_eval_staged<MODE, WS_W, WS_MINB, DYN, TMA, KEEP>;
    static DevLaunchCfg tab[PF_MAX_DEVICES];
    const DevLaunchCfg* dc = nullptr;
    cudaError_t e = device_cfg(tab, kern, 32 * WS_W, WS_SMEM, &dc);
    if (e != cudaSuccess) return e;
    const int ctas = dc->ctas, sms = dc->sms;
    const int32_t n_groups = (d.N + WS_W - 1) / WS_W;
    const int64_t n_items64 = (int64_t)n_groups * ((K + PF_LANES - 1) / PF_LANES);
    if (n_items64 >= (1ll << 31)) return cudaErrorInvalidValue;
    const int32_t n_items = (int32_t)n_items64;
    const int grid = (int)std::min<int64_t>(std::min<int64_t>(n_items, n_groups),
                                            (int64_t)ctas * sms);
    // n_groups as a multiply-shift divisor (Granlund-Montgomery, round-up form)
    uint32_t fd_l = 0;
    while ((1ll << fd_l) < n_groups) ++fd_l;
    const uint32_t fd_m =
        (uint32_t)(((1ull << 32) * ((1ull << fd_l) - (uint64_t)n_groups)) / (uint64_t)n_groups + 1);
    kern<<<grid, 32 * WS_W, WS_SMEM, st>>>(d, K, n_groups, n_items, y, pq_p, pq_q, pv_p,
                                           outage, g, j,
                                           reinterpret_cast<unsigned long long*>(norms), fd_m,
                                           fd_l, tm, tm_base, rb0);
    return cudaSuccess;
}

// Dynamic claiming when high-degree buses make the per-bus cost uneven
// (>= 0.5 % of buses with degree >= HUB_DEG; B200, ms per launch, static /
// dynamic: config 4 0.620 / 0.555, config 3 0.594 / 0.608).
template <int MODE>
static cudaError_t launch_staged_mode(const DevicePlan& d, int32_t K, const double* y,
                                      const double* pq_p, const double* pq_q,
                                      const double* pv_p, const int32_t* outage, double* g,
                                      double* j, double* norms, cudaStream_t st) {
    // PF_SCHEDULE=static|dynamic overrides the choice (A/B, tests); read once
    // (a C++11 function-local static initialiser is thread-safe)
    static const int forced = [] {
        const char* e = getenv("PF_SCHEDULE");
        return !e ? -1 : (e[0] == 'd' ? 1 : (e[0] == 's' ? 0 : -1));
    }();
    const bool dyn = forced >= 0 ? forced == 1 : (int64_t)d.n_hubs * 200 >= d.N;
    CUtensorMap tm;
    std::memset(&tm, 0, sizeof tm);
    const double* base = nullptr;
    int4 rb0 = make_int4(-1, -1, -1, -1);
    const bool tma = row_tensor_map(d, K, y, pq_p, pq_q, pv_p, &tm, &base, &rb0);
#define PF_K(D, T, KP) \
    launch_staged_kernel<MODE, D, T, KP>(d, K, y, pq_p, pq_q, pv_p, outage, g, j, norms, tm, base, rb0, st)
    // (the plan's L2 policy is a template parameter: no per-item branch)
    if (tma) return dyn ? PF_K(true, true, false) : PF_K(false, true, false);
    if (d.ws_keep) return dyn ? PF_K(true, false, true) : PF_K(false, false, true);
    return dyn ? PF_K(true, false, false) : PF_K(false, false, false);
#undef PF_K
}

static bool use_staged() {
    static const bool v = [] {
        const char* e = getenv("PF_BATCHED_KERNEL");
        return !(e && e[0] == 'o');   // "old": the single-role kernel (A/B timing)
    }();
    return v;
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
#define PF_B(M)                                                                         \
    (use_staged() ? launch_staged_mode<M>(d, K, y, pq_p, pq_q, pv_p, outage, g, j, norms, st) \
                  : launch_batched_mode<M>(d, K, y, pq_p, pq_q, pv_p, outage, g, j, norms, st))
    cudaError_t e = cudaSuccess;
    switch (mode) {
        case RES: e = PF_B(RES); break;
        case JAC: e = PF_B(JAC); break;
        case RES | JAC: e = PF_B(RES | JAC); break;
        case NORM: e = PF_B(NORM); break;
        case RES | NORM: e = PF_B(RES | NORM); break;
        case JAC | NORM: e = PF_B(JAC | NORM); break;
        case RES | JAC | NORM: e = PF_B(RES | JAC | NORM); break;
        default: return cudaSuccess;
    }
    if (e != cudaSuccess) return e;
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

cudaError_t launch_batch_unblock(int32_t K, int32_t n_e, const double* src, double* dst,
                                 double alpha, cudaStream_t st) {
    if (K <= 0 || n_e <= 0) return cudaSuccess;
    const dim3 grid(grid_for(n_e, 32), (unsigned)((K + PF_LANES - 1) / PF_LANES));
    k_batch_unblock<<<grid, 256, 0, st>>>(K, n_e, src, dst, alpha);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_batch_update(int32_t K, int32_t n_e, double* y, const double* dx,
                                const int32_t* active, cudaStream_t st) {
    if (K <= 0 || n_e <= 0) return cudaSuccess;
    const dim3 grid(grid_for(n_e, 32), (unsigned)((K + PF_LANES - 1) / PF_LANES));
    k_batch_update<<<grid, 256, 0, st>>>(K, n_e, y, dx, active);
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

#ifdef PF_X_TRACE
extern "C" __attribute__((visibility("default"))) int pf_debug_sg_trace(unsigned long long* host) {
    return (int)cudaMemcpyFromSymbol(host, pf::g_sg_trace, sizeof(unsigned long long) * 4096 * 8);
}
#endif
