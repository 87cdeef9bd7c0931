/*
 * pf_oracle.h - CPU restatement of the reference's evaluation path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library,
 * and only as the checker or the CPU baseline - never as the product path.
 *
 * Restates /root/reference/pkg/src/pflow (Python + Numba) in C:
 *   workspace build   residual.py:46-125, jacobian.py:39-80, 179-208
 *   wf1 kernels       kernels.py:79-97, 128-163, 215-282 (libm sin/cos,
 *                     no FMA contraction: bit-exact with pflow wf1)
 *   wf5 kernels       kernels.py:49-63, 100-125, 166-208 (polynomial sincos,
 *                     FMA contraction as under numba fastmath "contract")
 *   wf3               workflow.py:185-197 (static contiguous chunks over
 *                     worker threads; identical arithmetic to wf1)
 *   scenarios         SURVEY.md §8c batched oracle: mutate loads / PV P /
 *                     zero the outaged branch's 8 coefficients, evaluate,
 *                     restore.
 * Parity is pinned against golden vectors produced by the reference itself
 * (tests/golden/, scripts/make_golden.py).
 */
#ifndef PF_ORACLE_H
#define PF_ORACLE_H

#include <stdint.h>
#include "../include/pfgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_plan orc_plan;
typedef struct orc_ws orc_ws;

enum { ORC_NVAR = 0, ORC_NNZ, ORC_NSLOTS, ORC_NPOOL, ORC_NJOIN };

orc_plan* orc_plan_create(const pf_topology* t);
void orc_plan_destroy(orc_plan* p);
int64_t orc_plan_info(const orc_plan* p, int what);
void orc_plan_pattern(const orc_plan* p, int32_t* indptr, int32_t* indices);
void orc_plan_join(const orc_plan* p, int32_t* ptr, int32_t* split, int32_t* idx);
void orc_plan_slots(const orc_plan* p, int32_t* rows, int32_t* cols, int32_t* slot_to_csc,
                    int32_t* gather_ptr);

orc_ws* orc_ws_create(const orc_plan* p);
void orc_ws_destroy(orc_ws* w);

/* wf = 1 (serial scalar, the oracle) or 5 (serial SIMD-style) */
void orc_residual(orc_ws* w, int wf, const double* y, double* g);
void orc_jacobian(orc_ws* w, int wf, const double* y, double* csc_data);
/* pool[n_pool] after a residual evaluation; vals[n_slots] after a Jacobian */
const double* orc_ws_pool(const orc_ws* w);
const double* orc_ws_vals(const orc_ws* w);
void orc_line_injections(orc_ws* w, int wf, const double* y, double* ph, double* pk,
                         double* qh, double* qk);
void orc_libm_sincos(const double* x, double* s, double* c, int64_t n);
void orc_sincos_poly(const double* x, double* s, double* c, int64_t n);

/* wf3: intra-model chunks over nthreads (OpenMP); residual + CSC Jacobian */
void orc_eval_threaded(orc_ws* w, const double* y, double* g, double* csc_data, int nthreads);

/* Scenario batch in PF_LANES-blocked layout (see pfgpu.h).  Outputs g
 * (n_var entries / scenario), jcsc (nnz entries / scenario, CSC order) and
 * norms[K] may be NULL.  Scenarios run in parallel over nthreads, one
 * workspace per thread.  Returns 0. */
int orc_eval_scenarios(const orc_plan* p, int wf, int32_t K, const double* y,
                       const double* pq_p, const double* pq_q, const double* pv_p,
                       const int32_t* outage, double* g, double* jcsc, double* norms,
                       int nthreads);

#ifdef __cplusplus
}
#endif
#endif
