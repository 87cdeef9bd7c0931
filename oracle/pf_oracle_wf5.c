/*
 * pf_oracle_wf5.c - restatement of pflow's vectorised (wf5) line kernels.
 *
 * TEST INFRASTRUCTURE (see pf_oracle.h); also the fastest single-thread
 * CPU path used by the CPU baseline.  Compiled with FMA contraction and
 * x86-64-v3 so the loops pack, as numba fastmath={"contract","nsz"} does
 * for the reference (kernels.py:28-30).  Not bit-exact with pflow wf5
 * (contraction choices are compiler-specific); checked within tolerance.
 */
#include <math.h>
#include <stdint.h>

#include "pf_oracle_impl.h"

/* kernels.py:32-46 */
#define TWO_OVER_PI 0.63661977236758134308
#define PIO2_HI 1.57079632673412561417e+00
#define PIO2_LO 6.07710050650619224932e-11
#define S1 -1.66666666666666324348e-01
#define S2 8.33333333332248946124e-03
#define S3 -1.98412698298579493134e-04
#define S4 2.75573137070700676789e-06
#define S5 -2.50507602534068634195e-08
#define S6 1.58969099521155010221e-10
#define C1 4.16666666666666019037e-02
#define C2 -1.38888888888741095749e-03
#define C3 2.48015872894767294178e-05
#define C4 -2.75573143513906633035e-07
#define C5 2.08757232129817482790e-09
#define C6 -1.13596475577881948265e-11

/* kernels.py:49-63: rounded-quadrant Cody-Waite reduction + minimax polys */
static inline void sincos_poly(double x, double* s_out, double* c_out) {
    double kf = rint(x * TWO_OVER_PI);
    int64_t k = (int64_t)kf;
    double r = (x - kf * PIO2_HI) - kf * PIO2_LO;
    double z = r * r;
    double sp = r + r * z * (S1 + z * (S2 + z * (S3 + z * (S4 + z * (S5 + z * S6)))));
    double cp = 1.0 - 0.5 * z + z * z * (C1 + z * (C2 + z * (C3 + z * (C4 + z * (C5 + z * C6)))));
    int64_t q = k & 3;
    int swap = (q & 1) == 1;
    double sv = swap ? cp : sp;
    double cv = swap ? sp : cp;
    *s_out = ((q & 2) == 2) ? -sv : sv;
    *c_out = (((q + 1) & 2) == 2) ? -cv : cv;
}

void orc_sincos_poly(const double* x, double* s, double* c, int64_t n) {
    for (int64_t i = 0; i < n; ++i) sincos_poly(x[i], &s[i], &c[i]);
}

/* kernels.py:111-125 */
void orc_line_res_simd(int64_t n, const double* restrict thk, const double* restrict vh,
                       const double* restrict vk, double* const* c, double* restrict ph,
                       double* restrict pk, double* restrict qh, double* restrict qk) {
    const double* restrict gl = c[0];
    const double* restrict bl = c[1];
    const double* restrict gl2 = c[2];
    const double* restrict bl2 = c[3];
    const double* restrict gsh = c[4];
    const double* restrict bsh = c[5];
    const double* restrict gsk = c[6];
    const double* restrict bsk = c[7];
    for (int64_t i = 0; i < n; ++i) {
        double si, ci;
        sincos_poly(thk[i], &si, &ci);
        double a = vh[i];
        double b = vk[i];
        double ab = a * b;
        double t1h = gl[i] * ci + bl[i] * si;
        double t2h = gl[i] * si - bl[i] * ci;
        double t1k = gl2[i] * ci - bl2[i] * si;
        double t2k = gl2[i] * si + bl2[i] * ci;
        ph[i] = a * a * gsh[i] - ab * t1h;
        qh[i] = -a * a * bsh[i] - ab * t2h;
        pk[i] = b * b * gsk[i] - ab * t1k;
        qk[i] = -b * b * bsk[i] + ab * t2k;
    }
}

/* kernels.py:171-188 */
void orc_line_jac_simd_h(int64_t n, const double* restrict thk, const double* restrict vh,
                         const double* restrict vk, const double* restrict gl,
                         const double* restrict bl, const double* restrict gsh,
                         const double* restrict bsh, double* const* o) {
    double* restrict o0 = o[0]; double* restrict o1 = o[1];
    double* restrict o2 = o[2]; double* restrict o3 = o[3];
    double* restrict o4 = o[4]; double* restrict o5 = o[5];
    double* restrict o6 = o[6]; double* restrict o7 = o[7];
    for (int64_t i = 0; i < n; ++i) {
        double si, ci;
        sincos_poly(thk[i], &si, &ci);
        double a = vh[i];
        double b = vk[i];
        double ab = a * b;
        double t1h = gl[i] * ci + bl[i] * si;
        double t2h = gl[i] * si - bl[i] * ci;
        o0[i] = -ab * t2h;
        o1[i] = ab * t2h;
        o2[i] = -(2.0 * a * gsh[i] - b * t1h);
        o3[i] = a * t1h;
        o4[i] = ab * t1h;
        o5[i] = -ab * t1h;
        o6[i] = 2.0 * a * bsh[i] + b * t2h;
        o7[i] = a * t2h;
    }
}

/* kernels.py:191-208 */
void orc_line_jac_simd_k(int64_t n, const double* restrict thk, const double* restrict vh,
                         const double* restrict vk, const double* restrict gl2,
                         const double* restrict bl2, const double* restrict gsk,
                         const double* restrict bsk, double* const* o) {
    double* restrict o0 = o[0]; double* restrict o1 = o[1];
    double* restrict o2 = o[2]; double* restrict o3 = o[3];
    double* restrict o4 = o[4]; double* restrict o5 = o[5];
    double* restrict o6 = o[6]; double* restrict o7 = o[7];
    for (int64_t i = 0; i < n; ++i) {
        double si, ci;
        sincos_poly(thk[i], &si, &ci);
        double a = vh[i];
        double b = vk[i];
        double ab = a * b;
        double t1k = gl2[i] * ci - bl2[i] * si;
        double t2k = gl2[i] * si + bl2[i] * ci;
        o0[i] = -ab * t2k;
        o1[i] = ab * t2k;
        o2[i] = b * t1k;
        o3[i] = -(2.0 * b * gsk[i] - a * t1k);
        o4[i] = -ab * t1k;
        o5[i] = ab * t1k;
        o6[i] = -b * t2k;
        o7[i] = 2.0 * b * bsk[i] - a * t2k;
    }
}
