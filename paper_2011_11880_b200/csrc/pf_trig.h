/* pf_trig.h - near-correctly-rounded fp64 sin/cos shared by the CUDA kernels
 * (device) and a CPU twin (host C, tests only).
 *
 * Why: the reference's oracle workflow evaluates sin/cos with glibc 2.39
 * (pflow kernels.py:87-88 -> @llvm.sin/cos.f64 -> libm), whose results are
 * correctly rounded for all but ~0.3% (sin) / ~0.05% (cos) of arguments in
 * the power-flow angle range.  CUDA's sincos() differs from glibc in ~5-6% of
 * arguments (1 ulp).  A near-correctly-rounded sin/cos therefore agrees with
 * the oracle far more often, which keeps cancelling bus-balance sums inside
 * the 1e-12 / 1e-14 parity bound.
 *
 * Method (own restatement of the classic table + double-double scheme):
 *   1. k = rint(x 2/pi); r = x - k pi/2 as a double-double using a 3-part
 *      pi/2 and exact FMA products (Cody-Waite; valid for |x| < 2^20).
 *   2. |r| = X_i + d, X_i = i/64 from a 52-entry table of double-double
 *      sin/cos values, |d| <= 1/128.
 *   3. sin(X_i + d) = S + C d + [C (sin d - d) + S (cos d - 1) + low parts],
 *      cos(X_i + d) = C - S d + [...]: the leading product is split exactly
 *      with an FMA, the bracket (< 2^-14 of the result) is plain double, and
 *      one final rounding gives an error below 0.5 + 2^-12 ulp.
 *   4. quadrant selection by k mod 4.  |x| >= 2^20, inf, NaN: library call.
 * Every operation is written explicitly (fma() where fused), so the CUDA
 * build (-fmad=false) and the C build (-ffp-contract=off) are bit-identical.
 */
#ifndef PF_TRIG_H
#define PF_TRIG_H

#include "pf_trig_table.h"

#ifdef __CUDACC__
#define PF_HD __device__ __forceinline__
#else
#include <math.h>
#include <stdbool.h>
#define PF_HD static inline
#endif

/* polynomial coefficients; on the device they sit in the constant bank so the
 * FP64 instructions take them as operands instead of materialising
 * immediates every call */
#ifdef __CUDACC__
__device__ __constant__
#else
static
#endif
const double pf_trig_k[6] = {-1.0 / 6.0, 1.0 / 120.0, -1.0 / 5040.0,
                             -0.5, 1.0 / 24.0, -1.0 / 720.0};
#define PF_S3 pf_trig_k[0]
#define PF_S5 pf_trig_k[1]
#define PF_S7 pf_trig_k[2]
#define PF_C2 pf_trig_k[3]
#define PF_C4 pf_trig_k[4]
#define PF_C6 pf_trig_k[5]

#ifdef __CUDACC__
/* huge / non-finite arguments: out of line so the hot path stays small;
 * returned by value so the caller needs no stack slot */
__device__ __noinline__ static double2 pf_sincos_slow(double x) {
    double2 r;
    sincos(x, &r.x, &r.y);
    return r;
}
#endif

PF_HD void pf_two_sum(double a, double b, double* s, double* e) {
    double ss = a + b;
    double bb = ss - a;
    *e = (a - (ss - bb)) + (b - bb);
    *s = ss;
}

/* tab: PF_TRIG_N * 4 doubles {Sh, Ch, Sl, Cl} (pf_trig_tab, possibly staged
 * in shared memory by the caller). */
PF_HD void pf_sincos_tab(double x, const double* tab, double* sp, double* cp) {
    /* 1. r = x - k pi/2 in double-double.  |x| <= pi/4 (the usual power-flow
     * angle difference) has k = 0, for which the reduction is the identity
     * bit for bit, so it is skipped.  Everything else (NaN included) is
     * tested further inside the rare branch, so the common path pays one
     * comparison. */
    double kf = 0.0, rh = x, rl = 0.0;
    const bool reduce = !(fabs(x) <= 0.78539816339744828);
    if (reduce) {
        if (!(fabs(x) < 1048576.0)) {
            /* huge, infinite or NaN: evaluated at |x| so that, like the
             * fast path, sin is odd and cos even bit for bit (the kernels
             * evaluate one branch terminal at -thk, pf_eval.cu inc_terms) */
#ifdef __CUDA_ARCH__
            const double2 r = pf_sincos_slow(fabs(x));
            *sp = x < 0.0 ? -r.x : r.x;
            *cp = r.y;
#else
            *sp = x < 0.0 ? -sin(-x) : sin(x);
            *cp = cos(fabs(x));
#endif
            return;
        }
        kf = rint(x * PF_TWO_OVER_PI);
        const double ph = kf * PF_PIO2_1;
        const double pl = fma(kf, PF_PIO2_1, -ph);
        const double t = x - ph; /* exact (Sterbenz) */
        const double qh = kf * PF_PIO2_2;
        const double ql = fma(kf, PF_PIO2_2, -qh);
        double s1, e1, s2, e2;
        pf_two_sum(t, -pl, &s1, &e1);
        pf_two_sum(s1, -qh, &s2, &e2);
        const double rl0 = ((e1 + e2) - ql) - kf * PF_PIO2_3;
        rh = s2 + rl0;
        rl = rl0 - (rh - s2);
    }
    /* 2. |r| = X_i + d */
    const bool neg = rh < 0.0;
    const double a = fabs(rh);
    const double al = neg ? -rl : rl;
    const double fi = rint(a * 64.0);
    const int i = (int)fi;
    const double dh = a - fi * 0.015625; /* exact */
    const double z = dh * dh;
    /* sin d - dh and cos d - 1 (Horner with explicit FMAs) */
    const double sd = fma(dh * z, fma(z, fma(z, PF_S7, PF_S5), PF_S3), al);
    const double cm1 = fma(z, fma(z, fma(z, PF_C6, PF_C4), PF_C2), -(dh * al));
    const double Sh = tab[4 * i], Ch = tab[4 * i + 1], Sl = tab[4 * i + 2], Cl = tab[4 * i + 3];
    /* 3. sin and cos of |r|: leading sum split exactly (Fast2Sum is valid:
     * |Sh| >= |Ch dh| for i >= 1, and Sh = 0 for i = 0; |Ch| >= |Sh dh|) */
    const double P = Ch * dh;
    const double Pl = fma(Ch, dh, -P);
    double h = Sh + P;
    double e = P - (h - Sh);
    double s = h + (e + (Pl + (Sl + fma(Ch, sd, fma(Cl, dh, Sh * cm1)))));
    const double Q = Sh * dh;
    const double Ql = fma(Sh, dh, -Q);
    h = Ch - Q;
    e = (Ch - h) - Q;
    const double c = h + (e + (Cl - fma(Sh, sd, fma(Sl, dh, fma(-Ch, cm1, Ql)))));
    s = neg ? -s : s;
    /* 4. quadrant (k = 0 without reduction) */
    double so = s, co = c;
    if (reduce) {
        const int q = (int)((long long)kf & 3);
        so = (q & 1) ? c : s;
        co = (q & 1) ? s : c;
        so = (q & 2) ? -so : so;
        co = ((q + 1) & 2) ? -co : co;
    }
    *sp = (x == 0.0) ? x : so; /* keep the sign of -0.0 */
    *cp = co;
}

#endif /* PF_TRIG_H */
