/* CPU twin of the engine's device trig (test helper): the same source,
 * compiled for the host with -ffp-contract=off, must be bit-identical to
 * pf_sincos on the GPU. */
#include <stdint.h>
#include "../../paper_2011_11880_b200/csrc/pf_trig.h"

void twin_sincos(const double* x, double* s, double* c, int64_t n) {
    for (int64_t i = 0; i < n; ++i) pf_sincos_tab(x[i], pf_trig_tab, s + i, c + i);
}
