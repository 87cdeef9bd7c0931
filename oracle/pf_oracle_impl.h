/* Internal layout shared by the oracle translation units (test infra). */
#ifndef PF_ORACLE_IMPL_H
#define PF_ORACLE_IMPL_H

#include "pf_oracle.h"

struct orc_plan {
    int32_t N, L, P, G, S, H, n_gen, n_var;
    int32_t *bus_h, *bus_k;
    double *coef[8]; /* gl, bl, gl2, bl2, gsh, bsh, gsk, bsk */
    int32_t *pq_bus; double *pq_p0, *pq_q0;
    int32_t *pv_bus; double *pv_p0, *pv_v0; int32_t *pv_qg, *qg_addr_pv;
    int32_t *sl_bus; double *sl_v0, *sl_th0; int32_t *sl_qg, *sl_ps, *qg_addr_sl, *ps_addr_sl;
    int32_t *sh_bus; double *sh_g, *sh_b;
    /* contribution pool (residual.py:57) */
    int64_t off[16];
    int64_t n_pool;
    int32_t *join_ptr, *join_split, *join_idx;
    /* triplet slots + CSC (jacobian.py:42-72) */
    int64_t n_slots;
    int64_t sec[25];           /* 24 sections: 16 line + 8 device, sec[i]..sec[i+1] */
    int32_t *rows, *cols;
    int32_t nnz;
    int32_t *csc_indptr, *csc_indices, *slot_to_csc, *gather_ptr;
};

struct orc_ws {
    const orc_plan* p;
    double *coef[8];           /* mutable copies (scenario outages) */
    double *pq_p0, *pq_q0, *pv_p0;
    double *pool, *vals, *data, *thk, *vh, *vk, *y, *g;
};

/* wf5 line kernels (pf_oracle_wf5.c) */
void orc_line_res_simd(int64_t n, const double* thk, const double* vh, const double* vk,
                       double* const* c, double* ph, double* pk, double* qh, double* qk);
void orc_line_jac_simd_h(int64_t n, const double* thk, const double* vh, const double* vk,
                         const double* gl, const double* bl, const double* gsh,
                         const double* bsh, double* const* out8);
void orc_line_jac_simd_k(int64_t n, const double* thk, const double* vh, const double* vk,
                         const double* gl2, const double* bl2, const double* gsk,
                         const double* bsk, double* const* out8);

#endif
