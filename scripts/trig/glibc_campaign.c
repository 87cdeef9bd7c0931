#define _GNU_SOURCE
/* glibc_campaign.c - checks pf_trig.h (host build) against the live libm's
 * sin/cos bit for bit over many seeded arguments.  Dev/validation tool:
 *   gcc -O2 -fopenmp -ffp-contract=off scripts/trig/glibc_campaign.c -lm
 *   ./a.out N_PER_DIST SEED
 * Distributions (each N arguments): power-flow angle differences
 * N(0, 0.2*sqrt(2)) and N(0, 1); uniform on (-4, 4), (-100, 100), (-1e6, 1e6)
 * and (-1e8, 1e8); random bit patterns below 1.05e8 in magnitude (mostly
 * tiny); and the neighbourhoods of the range limits and of k/128. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../paper_2011_11880_b200/csrc/pf_trig.h"

static inline uint64_t next(uint64_t* s) {
    uint64_t x = *s;
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    return *s = x;
}
static inline double unif(uint64_t* s) { return (double)(next(s) >> 11) * 0x1p-53; }

static double draw(int dist, uint64_t* s) {
    switch (dist) {
    case 0:
    case 1: {
        const double sd = dist == 0 ? 0.28284271247461906 : 1.0;
        const double u1 = unif(s) + 1e-300, u2 = unif(s);
        return sd * sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    }
    case 2: return (2.0 * unif(s) - 1.0) * 4.0;
    case 3: return (2.0 * unif(s) - 1.0) * 100.0;
    case 4: return (2.0 * unif(s) - 1.0) * 1e6;
    case 5: return (2.0 * unif(s) - 1.0) * 1e8;
    case 6: {
        for (;;) {
            uint64_t b = next(s);
            double x;
            memcpy(&x, &b, 8);
            if (fabs(x) < 1.05e8) return x;
        }
    }
    default: {  /* near a limit or a table node: +-2^20 ulp */
        static const double lim[] = {0x1p-27, 0x1p-26, 0x1.020c49ba5e354p-3, 0.85546875,
                                     0x1.368fdp+1, 0x1.921fbp+26, 1.5707963267948966};
        double base;
        const uint64_t r = next(s);
        if (r % 3 == 0) base = lim[(r >> 8) % 7];
        else base = (double)((r >> 8) % 110) / 128.0 + (double)((r >> 20) % 2) / 256.0;
        int64_t b;
        memcpy(&b, &base, 8);
        b += (int64_t)(next(s) % (2u << 20)) - (1 << 20);
        double x;
        memcpy(&x, &b, 8);
        return (r >> 40) & 1 ? -x : x;
    }
    }
}

/* called through volatile pointers: a direct sin(x); cos(x) pair is fused
 * into one sincos() call by GCC, and pflow's wf1 (LLVM without fast-math on
 * a GNU target) calls sin and cos separately */
static double (*volatile libm_sin)(double) = sin;
static double (*volatile libm_cos)(double) = cos;
static void (*volatile libm_sincos)(double, double*, double*) = sincos;

int main(int argc, char** argv) {
    const long n = argc > 1 ? atol(argv[1]) : 1000000;
    const uint64_t seed = argc > 2 ? strtoull(argv[2], 0, 10) : 1;
    long total = 0, bad = 0;
    for (int dist = 0; dist < 8; ++dist) {
        long bs = 0, bc = 0, bq = 0;
#pragma omp parallel reduction(+ : bs, bc, bq)
        {
#ifdef _OPENMP
            extern int omp_get_thread_num(void);
            uint64_t st = seed * 0x9E3779B97F4A7C15ull + (uint64_t)(dist * 1000 + omp_get_thread_num() + 1) * 0xD1B54A32D192ED03ull;
#else
            uint64_t st = seed * 0x9E3779B97F4A7C15ull + (uint64_t)(dist * 1000 + 1) * 0xD1B54A32D192ED03ull;
#endif
#pragma omp for schedule(static)
            for (long i = 0; i < n; ++i) {
                const double x = draw(dist, &st);
                double s, c;
                pf_sincos_tab(x, pf_trig_tab, &s, &c);
                const double gs = libm_sin(x), gc = libm_cos(x);
                double s2, c2;
                libm_sincos(x, &s2, &c2);
                if (memcmp(&s2, &gs, 8) || memcmp(&c2, &gc, 8)) {
                    if (bq < 3) printf("  sincos(%a) != sin, cos\n", x);
                    ++bq;
                }
                if (memcmp(&s, &gs, 8)) {
                    if (bs < 3) printf("  sin(%a): %a, libm %a\n", x, s, gs);
                    ++bs;
                }
                if (memcmp(&c, &gc, 8)) {
                    if (bc < 3) printf("  cos(%a): %a, libm %a\n", x, c, gc);
                    ++bc;
                }
            }
        }
        printf("dist %d: %ld arguments, sin mismatches %ld, cos mismatches %ld (libm sincos vs sin/cos: %ld)\n",
               dist, n, bs, bc, bq);
        total += n;
        bad += bs + bc;
    }
    printf("TOTAL %ld arguments (x2 functions), %ld mismatches\n", total, bad);
    return bad != 0;
}
