/*
 * pf_oracle.c - CPU restatement of pflow's workspaces and wf1 kernels.
 *
 * TEST INFRASTRUCTURE (see pf_oracle.h).  Compiled with -ffp-contract=off
 * and libm sin/cos so every operation matches the reference's wf1
 * (numba njit without fastmath) in order and rounding.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#include "pf_oracle_impl.h"

#define ALLOC(T, n) ((T*)calloc((size_t)((n) > 0 ? (n) : 1), sizeof(T)))

static int32_t* dup_i32(const int32_t* a, int64_t n) {
    int32_t* r = ALLOC(int32_t, n);
    if (n && a) memcpy(r, a, (size_t)n * sizeof(int32_t));
    return r;
}
static double* dup_f64(const double* a, int64_t n) {
    double* r = ALLOC(double, n);
    if (n && a) memcpy(r, a, (size_t)n * sizeof(double));
    return r;
}

/* ------------------------------------------------------------------ */
/* wf1 kernels: pflow/kernels.py, same expressions, same order          */
/* ------------------------------------------------------------------ */

/* kernels.py:79-97 */
static void line_res_scalar(int64_t lo, int64_t hi, const int32_t* bus_h, const int32_t* bus_k,
                            double* const* c, const double* y, int32_t nb,
                            double* ph, double* pk, double* qh, double* qk) {
    const double *gl = c[0], *bl = c[1], *gl2 = c[2], *bl2 = c[3];
    const double *gsh = c[4], *bsh = c[5], *gsk = c[6], *bsk = c[7];
    for (int64_t i = lo; i < hi; ++i) {
        int32_t h = bus_h[i], k = bus_k[i];
        double a = y[nb + h];
        double b = y[nb + k];
        double thk = y[h] - y[k];
        double ci = cos(thk);
        double si = sin(thk);
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

/* kernels.py:128-163; out[16] in jacobian.py:31-36 section order */
static void line_jac_scalar(int64_t lo, int64_t hi, const int32_t* bus_h, const int32_t* bus_k,
                            double* const* c, const double* y, int32_t nb, double* const* o) {
    const double *gl = c[0], *bl = c[1], *gl2 = c[2], *bl2 = c[3];
    const double *gsh = c[4], *bsh = c[5], *gsk = c[6], *bsk = c[7];
    for (int64_t i = lo; i < hi; ++i) {
        int32_t h = bus_h[i], k = bus_k[i];
        double a = y[nb + h];
        double b = y[nb + k];
        double thk = y[h] - y[k];
        double ci = cos(thk);
        double si = sin(thk);
        double ab = a * b;
        double t1h = gl[i] * ci + bl[i] * si;
        double t2h = gl[i] * si - bl[i] * ci;
        double t1k = gl2[i] * ci - bl2[i] * si;
        double t2k = gl2[i] * si + bl2[i] * ci;
        o[0][i] = -ab * t2h;
        o[1][i] = ab * t2h;
        o[2][i] = -(2.0 * a * gsh[i] - b * t1h);
        o[3][i] = a * t1h;
        o[4][i] = ab * t1h;
        o[5][i] = -ab * t1h;
        o[6][i] = 2.0 * a * bsh[i] + b * t2h;
        o[7][i] = a * t2h;
        o[8][i] = -ab * t2k;
        o[9][i] = ab * t2k;
        o[10][i] = b * t1k;
        o[11][i] = -(2.0 * b * gsk[i] - a * t1k);
        o[12][i] = -ab * t1k;
        o[13][i] = ab * t1k;
        o[14][i] = -b * t2k;
        o[15][i] = 2.0 * b * bsk[i] - a * t2k;
    }
}

/* kernels.py:100-108 */
static void line_gather(int64_t lo, int64_t hi, const int32_t* bus_h, const int32_t* bus_k,
                        const double* y, int32_t nb, double* thk, double* vh, double* vk) {
    for (int64_t i = lo; i < hi; ++i) {
        int32_t h = bus_h[i], k = bus_k[i];
        thk[i] = y[h] - y[k];
        vh[i] = y[nb + h];
        vk[i] = y[nb + k];
    }
}

/* kernels.py:215-241 */
static void pq_res(int64_t lo, int64_t hi, const double* p0, const double* q0, double* op,
                   double* oq) {
    for (int64_t i = lo; i < hi; ++i) {
        op[i] = -p0[i];
        oq[i] = -q0[i];
    }
}
static void pv_res(int64_t lo, int64_t hi, const int32_t* bus, const double* p0, const double* v0,
                   const int32_t* qg_addr, const double* y, int32_t nb, double* op, double* oq,
                   double* ov) {
    for (int64_t i = lo; i < hi; ++i) {
        op[i] = p0[i];
        oq[i] = y[qg_addr[i]];
        ov[i] = y[nb + bus[i]] - v0[i];
    }
}
static void slack_res(int64_t n, const int32_t* bus, const double* v0, const double* th0,
                      const int32_t* qg_addr, const int32_t* ps_addr, const double* y, int32_t nb,
                      double* op, double* oq, double* ov, double* oth) {
    for (int64_t i = 0; i < n; ++i) {
        op[i] = y[ps_addr[i]];
        oq[i] = y[qg_addr[i]];
        ov[i] = y[nb + bus[i]] - v0[i];
        oth[i] = y[bus[i]] - th0[i];
    }
}
static void shunt_res(int64_t lo, int64_t hi, const int32_t* bus, const double* g,
                      const double* b, const double* y, int32_t nb, double* op, double* oq) {
    for (int64_t i = lo; i < hi; ++i) {
        double vi = y[nb + bus[i]];
        double v2 = vi * vi;
        op[i] = -g[i] * v2;
        oq[i] = b[i] * v2;
    }
}
/* kernels.py:244-262 */
static void pv_jac(int64_t n, double* gq_qg, double* gv_v) {
    for (int64_t i = 0; i < n; ++i) {
        gq_qg[i] = 1.0;
        gv_v[i] = 1.0;
    }
}
static void slack_jac(int64_t n, double* a, double* b, double* c, double* d) {
    for (int64_t i = 0; i < n; ++i) {
        a[i] = 1.0;
        b[i] = 1.0;
        c[i] = 1.0;
        d[i] = 1.0;
    }
}
static void shunt_jac(int64_t lo, int64_t hi, const int32_t* bus, const double* g, const double* b,
                      const double* y, int32_t nb, double* gp_v, double* gq_v) {
    for (int64_t i = lo; i < hi; ++i) {
        double vi = y[nb + bus[i]];
        gp_v[i] = -2.0 * g[i] * vi;
        gq_v[i] = 2.0 * b[i] * vi;
    }
}
/* kernels.py:265-274 */
static void join_rows(int64_t lo, int64_t hi, const int32_t* ptr, const int32_t* split,
                      const int32_t* idx, const double* pool, double* out) {
    for (int64_t r = lo; r < hi; ++r) {
        double acc = 0.0;
        for (int32_t j = ptr[r]; j < split[r]; ++j) acc -= pool[idx[j]];
        for (int32_t j = split[r]; j < ptr[r + 1]; ++j) acc += pool[idx[j]];
        out[r] = acc;
    }
}
/* kernels.py:277-282 */
static void gather_sum(int64_t lo, int64_t hi, const int32_t* ptr, const int32_t* idx,
                       const double* vals, double* out) {
    for (int64_t r = lo; r < hi; ++r) {
        double acc = 0.0;
        for (int32_t j = ptr[r]; j < ptr[r + 1]; ++j) acc += vals[idx[j]];
        out[r] = acc;
    }
}

/* ------------------------------------------------------------------ */
/* plan: pool layout, join CSR, slots, CSC (residual.py:49-125,        */
/* jacobian.py:42-72, 179-208)                                         */
/* ------------------------------------------------------------------ */

static void build_join(orc_plan* p) {
    const int32_t N = p->N, n = p->n_var;
    const int64_t* off = p->off;
    int32_t* nminus = ALLOC(int32_t, n);
    int32_t* nplus = ALLOC(int32_t, n);
    /* pass 1: counts (gp_of_bus = b, gq_of_bus = N + b, gv_of_gen = 2N + q,
       gtheta_of_slack = 2N + n_gen + ps) */
    for (int32_t i = 0; i < p->L; ++i) {
        nminus[p->bus_h[i]]++; nminus[p->bus_k[i]]++;
        nminus[N + p->bus_h[i]]++; nminus[N + p->bus_k[i]]++;
    }
    for (int32_t j = 0; j < p->P; ++j) { nplus[p->pq_bus[j]]++; nplus[N + p->pq_bus[j]]++; }
    for (int32_t i = 0; i < p->G; ++i) {
        nplus[p->pv_bus[i]]++; nplus[N + p->pv_bus[i]]++; nplus[2 * N + p->pv_qg[i]]++;
    }
    for (int32_t s = 0; s < p->S; ++s) {
        nplus[p->sl_bus[s]]++; nplus[N + p->sl_bus[s]]++;
        nplus[2 * N + p->sl_qg[s]]++; nplus[2 * N + p->n_gen + p->sl_ps[s]]++;
    }
    for (int32_t j = 0; j < p->H; ++j) { nplus[p->sh_bus[j]]++; nplus[N + p->sh_bus[j]]++; }
    p->join_ptr = ALLOC(int32_t, n + 1);
    p->join_split = ALLOC(int32_t, n);
    for (int32_t r = 0; r < n; ++r) {
        p->join_split[r] = p->join_ptr[r] + nminus[r];
        p->join_ptr[r + 1] = p->join_split[r] + nplus[r];
    }
    p->join_idx = ALLOC(int32_t, p->join_ptr[n]);
    /* pass 2: fill in ascending pool index, so each row's minus and plus
       lists come out sorted exactly as sorted(minus[r]) / sorted(plus[r]) */
    int32_t* cm = ALLOC(int32_t, n);
    int32_t* cp = ALLOC(int32_t, n);
    for (int32_t r = 0; r < n; ++r) { cm[r] = p->join_ptr[r]; cp[r] = p->join_split[r]; }
#define MINUS(row, slot) p->join_idx[cm[(row)]++] = (int32_t)(slot)
#define PLUS(row, slot) p->join_idx[cp[(row)]++] = (int32_t)(slot)
    for (int32_t i = 0; i < p->L; ++i) MINUS(p->bus_h[i], off[0] + i);
    for (int32_t i = 0; i < p->L; ++i) MINUS(p->bus_k[i], off[1] + i);
    for (int32_t i = 0; i < p->L; ++i) MINUS(N + p->bus_h[i], off[2] + i);
    for (int32_t i = 0; i < p->L; ++i) MINUS(N + p->bus_k[i], off[3] + i);
    for (int32_t j = 0; j < p->P; ++j) PLUS(p->pq_bus[j], off[4] + j);
    for (int32_t j = 0; j < p->P; ++j) PLUS(N + p->pq_bus[j], off[5] + j);
    for (int32_t i = 0; i < p->G; ++i) PLUS(p->pv_bus[i], off[6] + i);
    for (int32_t i = 0; i < p->G; ++i) PLUS(N + p->pv_bus[i], off[7] + i);
    for (int32_t i = 0; i < p->G; ++i) PLUS(2 * N + p->pv_qg[i], off[8] + i);
    for (int32_t s = 0; s < p->S; ++s) PLUS(p->sl_bus[s], off[9] + s);
    for (int32_t s = 0; s < p->S; ++s) PLUS(N + p->sl_bus[s], off[10] + s);
    for (int32_t s = 0; s < p->S; ++s) PLUS(2 * N + p->sl_qg[s], off[11] + s);
    for (int32_t s = 0; s < p->S; ++s) PLUS(2 * N + p->n_gen + p->sl_ps[s], off[12] + s);
    for (int32_t j = 0; j < p->H; ++j) PLUS(p->sh_bus[j], off[13] + j);
    for (int32_t j = 0; j < p->H; ++j) PLUS(N + p->sh_bus[j], off[14] + j);
#undef MINUS
#undef PLUS
    free(cm); free(cp); free(nminus); free(nplus);
}

/* stable counting sort of perm[] by key[perm[.]] in [0, range) */
static void stable_sort_by(int32_t* perm, int64_t n, const int32_t* key, int32_t range) {
    int64_t* cnt = ALLOC(int64_t, (int64_t)range + 1);
    int32_t* tmp = ALLOC(int32_t, n);
    for (int64_t i = 0; i < n; ++i) cnt[key[perm[i]] + 1]++;
    for (int32_t r = 0; r < range; ++r) cnt[r + 1] += cnt[r];
    for (int64_t i = 0; i < n; ++i) tmp[cnt[key[perm[i]]]++] = perm[i];
    memcpy(perm, tmp, (size_t)n * sizeof(int32_t));
    free(cnt); free(tmp);
}

static void build_slots(orc_plan* p) {
    const int32_t N = p->N, L = p->L, n = p->n_var;
    int64_t sizes[24];
    for (int i = 0; i < 16; ++i) sizes[i] = L;
    sizes[16] = p->G; sizes[17] = p->G;
    sizes[18] = p->S; sizes[19] = p->S; sizes[20] = p->S; sizes[21] = p->S;
    sizes[22] = p->H; sizes[23] = p->H;
    p->sec[0] = 0;
    for (int i = 0; i < 24; ++i) p->sec[i + 1] = p->sec[i] + sizes[i];
    p->n_slots = p->sec[24];
    p->rows = ALLOC(int32_t, p->n_slots);
    p->cols = ALLOC(int32_t, p->n_slots);
    /* _LINE_SECTIONS (jacobian.py:31-36): row kind gp_h,gq_h,gp_k,gq_k x
       col kind th_h,th_k,v_h,v_k */
    for (int s = 0; s < 16; ++s) {
        int rk = s / 4, ck = s % 4;
        int32_t* R = p->rows + p->sec[s];
        int32_t* C = p->cols + p->sec[s];
        for (int32_t i = 0; i < L; ++i) {
            int32_t h = p->bus_h[i], k = p->bus_k[i];
            R[i] = (rk == 0) ? h : (rk == 1) ? N + h : (rk == 2) ? k : N + k;
            C[i] = (ck == 0) ? h : (ck == 1) ? k : (ck == 2) ? N + h : N + k;
        }
    }
    for (int32_t i = 0; i < p->G; ++i) {
        p->rows[p->sec[16] + i] = N + p->pv_bus[i];
        p->cols[p->sec[16] + i] = 2 * N + p->pv_qg[i];
        p->rows[p->sec[17] + i] = 2 * N + p->pv_qg[i];
        p->cols[p->sec[17] + i] = N + p->pv_bus[i];
    }
    for (int32_t s = 0; s < p->S; ++s) {
        int32_t b = p->sl_bus[s];
        p->rows[p->sec[18] + s] = b;
        p->cols[p->sec[18] + s] = 2 * N + p->n_gen + p->sl_ps[s];
        p->rows[p->sec[19] + s] = N + b;
        p->cols[p->sec[19] + s] = 2 * N + p->sl_qg[s];
        p->rows[p->sec[20] + s] = 2 * N + p->sl_qg[s];
        p->cols[p->sec[20] + s] = N + b;
        p->rows[p->sec[21] + s] = 2 * N + p->n_gen + p->sl_ps[s];
        p->cols[p->sec[21] + s] = b;
    }
    for (int32_t j = 0; j < p->H; ++j) {
        int32_t b = p->sh_bus[j];
        p->rows[p->sec[22] + j] = b;
        p->cols[p->sec[22] + j] = N + b;
        p->rows[p->sec[23] + j] = N + b;
        p->cols[p->sec[23] + j] = N + b;
    }
    /* order = lexsort((rows, cols)): by col, then row, then slot (stable) */
    int64_t ns = p->n_slots;
    int32_t* order = ALLOC(int32_t, ns);
    for (int64_t i = 0; i < ns; ++i) order[i] = (int32_t)i;
    stable_sort_by(order, ns, p->rows, n);
    stable_sort_by(order, ns, p->cols, n);
    p->slot_to_csc = order;
    int32_t nnz = 0;
    for (int64_t i = 0; i < ns; ++i) {
        if (i == 0 || p->rows[order[i]] != p->rows[order[i - 1]] ||
            p->cols[order[i]] != p->cols[order[i - 1]])
            nnz++;
    }
    p->nnz = nnz;
    p->gather_ptr = ALLOC(int32_t, nnz + 1);
    p->csc_indices = ALLOC(int32_t, nnz);
    p->csc_indptr = ALLOC(int32_t, n + 1);
    int32_t q = 0;
    for (int64_t i = 0; i < ns; ++i) {
        if (i == 0 || p->rows[order[i]] != p->rows[order[i - 1]] ||
            p->cols[order[i]] != p->cols[order[i - 1]]) {
            p->gather_ptr[q] = (int32_t)i;
            p->csc_indices[q] = p->rows[order[i]];
            p->csc_indptr[p->cols[order[i]] + 1]++;
            q++;
        }
    }
    p->gather_ptr[nnz] = (int32_t)ns;
    for (int32_t c = 0; c < n; ++c) p->csc_indptr[c + 1] += p->csc_indptr[c];
}

orc_plan* orc_plan_create(const pf_topology* t) {
    orc_plan* p = (orc_plan*)calloc(1, sizeof(orc_plan));
    p->N = t->n_bus; p->L = t->n_line; p->P = t->n_pq; p->G = t->n_pv; p->S = t->n_slack;
    p->H = t->n_shunt;
    p->n_gen = p->G + p->S;
    p->n_var = 2 * p->N + p->G + 2 * p->S;
    p->bus_h = dup_i32(t->bus_h, p->L);
    p->bus_k = dup_i32(t->bus_k, p->L);
    const double* src[8] = {t->gl, t->bl, t->gl2, t->bl2, t->g_self_h, t->b_self_h,
                            t->g_self_k, t->b_self_k};
    for (int i = 0; i < 8; ++i) p->coef[i] = dup_f64(src[i], p->L);
    p->pq_bus = dup_i32(t->pq_bus, p->P);
    p->pq_p0 = dup_f64(t->pq_p0, p->P);
    p->pq_q0 = dup_f64(t->pq_q0, p->P);
    p->pv_bus = dup_i32(t->pv_bus, p->G);
    p->pv_p0 = dup_f64(t->pv_p0, p->G);
    p->pv_v0 = dup_f64(t->pv_v0, p->G);
    p->pv_qg = dup_i32(t->pv_qg, p->G);
    p->sl_bus = dup_i32(t->sl_bus, p->S);
    p->sl_v0 = dup_f64(t->sl_v0, p->S);
    p->sl_th0 = dup_f64(t->sl_th0, p->S);
    p->sl_qg = dup_i32(t->sl_qg, p->S);
    p->sl_ps = dup_i32(t->sl_ps, p->S);
    p->sh_bus = dup_i32(t->sh_bus, p->H);
    p->sh_g = dup_f64(t->sh_g, p->H);
    p->sh_b = dup_f64(t->sh_b, p->H);
    /* qg_addr = addr.qg_of_gen[qg], ps_addr = addr.ps_of_slack[ps] (residual.py:70-72) */
    p->qg_addr_pv = ALLOC(int32_t, p->G);
    for (int32_t i = 0; i < p->G; ++i) p->qg_addr_pv[i] = 2 * p->N + p->pv_qg[i];
    p->qg_addr_sl = ALLOC(int32_t, p->S);
    p->ps_addr_sl = ALLOC(int32_t, p->S);
    for (int32_t s = 0; s < p->S; ++s) {
        p->qg_addr_sl[s] = 2 * p->N + p->sl_qg[s];
        p->ps_addr_sl[s] = 2 * p->N + p->n_gen + p->sl_ps[s];
    }
    int64_t sizes[15] = {p->L, p->L, p->L, p->L, p->P, p->P, p->G, p->G, p->G,
                         p->S, p->S, p->S, p->S, p->H, p->H};
    p->off[0] = 0;
    for (int i = 0; i < 15; ++i) p->off[i + 1] = p->off[i] + sizes[i];
    p->n_pool = p->off[15];
    build_join(p);
    build_slots(p);
    return p;
}

void orc_plan_destroy(orc_plan* p) {
    if (!p) return;
    free(p->bus_h); free(p->bus_k);
    for (int i = 0; i < 8; ++i) free(p->coef[i]);
    free(p->pq_bus); free(p->pq_p0); free(p->pq_q0);
    free(p->pv_bus); free(p->pv_p0); free(p->pv_v0); free(p->pv_qg); free(p->qg_addr_pv);
    free(p->sl_bus); free(p->sl_v0); free(p->sl_th0); free(p->sl_qg); free(p->sl_ps);
    free(p->qg_addr_sl); free(p->ps_addr_sl);
    free(p->sh_bus); free(p->sh_g); free(p->sh_b);
    free(p->join_ptr); free(p->join_split); free(p->join_idx);
    free(p->rows); free(p->cols); free(p->slot_to_csc); free(p->gather_ptr);
    free(p->csc_indptr); free(p->csc_indices);
    free(p);
}

int64_t orc_plan_info(const orc_plan* p, int what) {
    switch (what) {
        case ORC_NVAR: return p->n_var;
        case ORC_NNZ: return p->nnz;
        case ORC_NSLOTS: return p->n_slots;
        case ORC_NPOOL: return p->n_pool;
        case ORC_NJOIN: return p->join_ptr[p->n_var];
    }
    return -1;
}

void orc_plan_pattern(const orc_plan* p, int32_t* indptr, int32_t* indices) {
    memcpy(indptr, p->csc_indptr, (size_t)(p->n_var + 1) * sizeof(int32_t));
    memcpy(indices, p->csc_indices, (size_t)p->nnz * sizeof(int32_t));
}

void orc_plan_join(const orc_plan* p, int32_t* ptr, int32_t* split, int32_t* idx) {
    memcpy(ptr, p->join_ptr, (size_t)(p->n_var + 1) * sizeof(int32_t));
    memcpy(split, p->join_split, (size_t)p->n_var * sizeof(int32_t));
    memcpy(idx, p->join_idx, (size_t)p->join_ptr[p->n_var] * sizeof(int32_t));
}

void orc_plan_slots(const orc_plan* p, int32_t* rows, int32_t* cols, int32_t* slot_to_csc,
                    int32_t* gather_ptr) {
    memcpy(rows, p->rows, (size_t)p->n_slots * sizeof(int32_t));
    memcpy(cols, p->cols, (size_t)p->n_slots * sizeof(int32_t));
    memcpy(slot_to_csc, p->slot_to_csc, (size_t)p->n_slots * sizeof(int32_t));
    memcpy(gather_ptr, p->gather_ptr, (size_t)(p->nnz + 1) * sizeof(int32_t));
}

orc_ws* orc_ws_create(const orc_plan* p) {
    orc_ws* w = (orc_ws*)calloc(1, sizeof(orc_ws));
    w->p = p;
    for (int i = 0; i < 8; ++i) w->coef[i] = dup_f64(p->coef[i], p->L);
    w->pq_p0 = dup_f64(p->pq_p0, p->P);
    w->pq_q0 = dup_f64(p->pq_q0, p->P);
    w->pv_p0 = dup_f64(p->pv_p0, p->G);
    w->pool = ALLOC(double, p->n_pool);
    w->vals = ALLOC(double, p->n_slots);
    w->data = ALLOC(double, p->nnz);
    w->thk = ALLOC(double, p->L);
    w->vh = ALLOC(double, p->L);
    w->vk = ALLOC(double, p->L);
    w->y = ALLOC(double, p->n_var);
    w->g = ALLOC(double, p->n_var);
    return w;
}

void orc_ws_destroy(orc_ws* w) {
    if (!w) return;
    for (int i = 0; i < 8; ++i) free(w->coef[i]);
    free(w->pq_p0); free(w->pq_q0); free(w->pv_p0);
    free(w->pool); free(w->vals); free(w->data); free(w->thk); free(w->vh); free(w->vk);
    free(w->y); free(w->g);
    free(w);
}

const double* orc_ws_pool(const orc_ws* w) { return w->pool; }
const double* orc_ws_vals(const orc_ws* w) { return w->vals; }

/* ------------------------------------------------------------------ */
/* residual / Jacobian drivers (residual.py:244-255, jacobian.py:173-176) */
/* ------------------------------------------------------------------ */

static void residual_models(orc_ws* w, int wf, const double* y) {
    const orc_plan* p = w->p;
    double* pool = w->pool;
    const int64_t* off = p->off;
    /* serial inter-model order PQ, PV, Slack, Line, Shunt (residual.py:237-238) */
    pq_res(0, p->P, w->pq_p0, w->pq_q0, pool + off[4], pool + off[5]);
    pv_res(0, p->G, p->pv_bus, w->pv_p0, p->pv_v0, p->qg_addr_pv, y, p->N, pool + off[6],
           pool + off[7], pool + off[8]);
    slack_res(p->S, p->sl_bus, p->sl_v0, p->sl_th0, p->qg_addr_sl, p->ps_addr_sl, y, p->N,
              pool + off[9], pool + off[10], pool + off[11], pool + off[12]);
    if (wf == 5) {
        line_gather(0, p->L, p->bus_h, p->bus_k, y, p->N, w->thk, w->vh, w->vk);
        orc_line_res_simd(p->L, w->thk, w->vh, w->vk, w->coef, pool + off[0], pool + off[1],
                          pool + off[2], pool + off[3]);
    } else {
        line_res_scalar(0, p->L, p->bus_h, p->bus_k, w->coef, y, p->N, pool + off[0],
                        pool + off[1], pool + off[2], pool + off[3]);
    }
    shunt_res(0, p->H, p->sh_bus, p->sh_g, p->sh_b, y, p->N, pool + off[13], pool + off[14]);
}

void orc_residual(orc_ws* w, int wf, const double* y, double* g) {
    residual_models(w, wf, y);
    const orc_plan* p = w->p;
    join_rows(0, p->n_var, p->join_ptr, p->join_split, p->join_idx, w->pool, g);
}

static void jacobian_models(orc_ws* w, int wf, const double* y) {
    const orc_plan* p = w->p;
    double* o[24];
    for (int s = 0; s < 24; ++s) o[s] = w->vals + p->sec[s];
    pv_jac(p->G, o[16], o[17]);
    slack_jac(p->S, o[18], o[19], o[20], o[21]);
    if (wf == 5) {
        line_gather(0, p->L, p->bus_h, p->bus_k, y, p->N, w->thk, w->vh, w->vk);
        orc_line_jac_simd_h(p->L, w->thk, w->vh, w->vk, w->coef[0], w->coef[1], w->coef[4],
                            w->coef[5], o);
        orc_line_jac_simd_k(p->L, w->thk, w->vh, w->vk, w->coef[2], w->coef[3], w->coef[6],
                            w->coef[7], o + 8);
    } else {
        line_jac_scalar(0, p->L, p->bus_h, p->bus_k, w->coef, y, p->N, o);
    }
    shunt_jac(0, p->H, p->sh_bus, p->sh_g, p->sh_b, y, p->N, o[22], o[23]);
}

void orc_jacobian(orc_ws* w, int wf, const double* y, double* csc_data) {
    jacobian_models(w, wf, y);
    const orc_plan* p = w->p;
    gather_sum(0, p->nnz, p->gather_ptr, p->slot_to_csc, w->vals, csc_data);
}

void orc_line_injections(orc_ws* w, int wf, const double* y, double* ph, double* pk,
                         double* qh, double* qk) {
    const orc_plan* p = w->p;
    if (wf == 5) {
        line_gather(0, p->L, p->bus_h, p->bus_k, y, p->N, w->thk, w->vh, w->vk);
        orc_line_res_simd(p->L, w->thk, w->vh, w->vk, w->coef, ph, pk, qh, qk);
    } else {
        line_res_scalar(0, p->L, p->bus_h, p->bus_k, w->coef, y, p->N, ph, pk, qh, qk);
    }
}

/* wf3: every model's device range in contiguous static chunks over the
   worker threads (workflow.py:185-197, residual.py:33-43) */
void orc_eval_threaded(orc_ws* w, const double* y, double* g, double* csc_data, int nthreads) {
    const orc_plan* p = w->p;
    double* pool = w->pool;
    const int64_t* off = p->off;
    double* o[24];
    for (int s = 0; s < 24; ++s) o[s] = w->vals + p->sec[s];
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel num_threads(nthreads)
    {
        int t = omp_get_thread_num(), T = omp_get_num_threads();
#define CHUNK(n) int64_t lo = ((int64_t)(n) * t) / T, hi = ((int64_t)(n) * (t + 1)) / T
        if (g) {
            { CHUNK(p->P); pq_res(lo, hi, w->pq_p0, w->pq_q0, pool + off[4], pool + off[5]); }
            { CHUNK(p->G); pv_res(lo, hi, p->pv_bus, w->pv_p0, p->pv_v0, p->qg_addr_pv, y, p->N,
                                  pool + off[6], pool + off[7], pool + off[8]); }
            if (t == 0)
                slack_res(p->S, p->sl_bus, p->sl_v0, p->sl_th0, p->qg_addr_sl, p->ps_addr_sl, y,
                          p->N, pool + off[9], pool + off[10], pool + off[11], pool + off[12]);
            { CHUNK(p->L); line_res_scalar(lo, hi, p->bus_h, p->bus_k, w->coef, y, p->N,
                                           pool + off[0], pool + off[1], pool + off[2],
                                           pool + off[3]); }
            { CHUNK(p->H); shunt_res(lo, hi, p->sh_bus, p->sh_g, p->sh_b, y, p->N,
                                     pool + off[13], pool + off[14]); }
#pragma omp barrier
            { CHUNK(p->n_var); join_rows(lo, hi, p->join_ptr, p->join_split, p->join_idx, pool,
                                         g); }
        }
        if (csc_data) {
            if (t == 0) {
                pv_jac(p->G, o[16], o[17]);
                slack_jac(p->S, o[18], o[19], o[20], o[21]);
            }
            { CHUNK(p->L); line_jac_scalar(lo, hi, p->bus_h, p->bus_k, w->coef, y, p->N, o); }
            { CHUNK(p->H); shunt_jac(lo, hi, p->sh_bus, p->sh_g, p->sh_b, y, p->N, o[22],
                                     o[23]); }
#pragma omp barrier
            { CHUNK(p->nnz); gather_sum(lo, hi, p->gather_ptr, p->slot_to_csc, w->vals,
                                        csc_data); }
        }
#undef CHUNK
    }
}

void orc_libm_sincos(const double* x, double* s, double* c, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        s[i] = sin(x[i]);
        c[i] = cos(x[i]);
    }
}

/* ------------------------------------------------------------------ */
/* scenario batch (SURVEY.md §8c batched oracle)                        */
/* ------------------------------------------------------------------ */

static inline int64_t blk(int64_t n_e, int64_t e, int64_t s) {
    return ((s / PF_LANES) * n_e + e) * PF_LANES + (s % PF_LANES);
}

/* max |x| with NaN propagation (np.abs(g).max()) */
static double inf_norm(const double* g, int64_t n) {
    uint64_t best = 0;
    for (int64_t i = 0; i < n; ++i) {
        double a = fabs(g[i]);
        uint64_t u;
        memcpy(&u, &a, sizeof u);
        if (u > best) best = u;
    }
    double r;
    memcpy(&r, &best, sizeof r);
    return r;
}

int orc_eval_scenarios(const orc_plan* p, int wf, int32_t K, const double* y,
                       const double* pq_p, const double* pq_q, const double* pv_p,
                       const int32_t* outage, double* g, double* jcsc, double* norms,
                       int nthreads) {
    if (nthreads < 1) nthreads = 1;
    const int64_t nv = p->n_var, nnz = p->nnz;
#pragma omp parallel num_threads(nthreads)
    {
        orc_ws* w = orc_ws_create(p);
#pragma omp for schedule(dynamic, 1)
        for (int32_t s = 0; s < K; ++s) {
            for (int64_t e = 0; e < nv; ++e) w->y[e] = y[blk(nv, e, s)];
            for (int32_t j = 0; j < p->P; ++j) {
                w->pq_p0[j] = pq_p ? pq_p[blk(p->P, j, s)] : p->pq_p0[j];
                w->pq_q0[j] = pq_q ? pq_q[blk(p->P, j, s)] : p->pq_q0[j];
            }
            for (int32_t j = 0; j < p->G; ++j) w->pv_p0[j] = pv_p ? pv_p[blk(p->G, j, s)] : p->pv_p0[j];
            int32_t l = outage ? outage[s] : -1;
            double saved[8];
            if (l >= 0 && l < p->L)
                for (int c = 0; c < 8; ++c) { saved[c] = w->coef[c][l]; w->coef[c][l] = 0.0; }
            orc_residual(w, wf, w->y, w->g);
            orc_jacobian(w, wf, w->y, w->data);
            if (l >= 0 && l < p->L)
                for (int c = 0; c < 8; ++c) w->coef[c][l] = saved[c];
            if (norms) norms[s] = inf_norm(w->g, nv);
            if (g) for (int64_t e = 0; e < nv; ++e) g[blk(nv, e, s)] = w->g[e];
            if (jcsc) for (int64_t e = 0; e < nnz; ++e) jcsc[blk(nnz, e, s)] = w->data[e];
        }
        orc_ws_destroy(w);
    }
    return 0;
}
