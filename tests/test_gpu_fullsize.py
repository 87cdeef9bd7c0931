"""Full-size parity of the exact bench workloads, every entry.

bench.py times two batched workloads: BASELINE config 3 (70k buses, K = 256,
seed 1000) and config 4 (200k buses with degree-50 hubs, K = 64).  Here the
product kernel evaluates exactly those inputs and every scenario's residual,
Jacobian (all ~0.5 G values) and infinity norm is compared with the oracle's
wf1 -- the C restatement pinned bit for bit to pflow's own outputs
(tests/test_oracle_golden.py).  The criterion is the north star's per-entry
bound and, beyond it, bit-identity: the device sin/cos are glibc's
(csrc/pf_trig.h) and every other operation rounds where wf1 rounds.

Layout: both sides stay in the blocked scenario layout; the device Jacobian
is permuted to the reference's CSC order on the GPU (pf_jac_to_csc), so the
comparison is one pass over flat arrays.
"""

import os

import numpy as np
import pytest

import oracle
from _util import ABS_TOL, REL_TOL

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _first_bad(got, ref):
    i = int(np.flatnonzero(got.view(np.int64) != ref.view(np.int64))[0])
    return i, got[i], ref[i]


def _compare(got, ref, what):
    """Bit-identity, else the tolerance report of the first mismatch."""
    if np.array_equal(got.view(np.int64), ref.view(np.int64)):
        return
    n_bits = int((got.view(np.int64) != ref.view(np.int64)).sum())
    tol = np.maximum(REL_TOL * np.abs(ref), ABS_TOL)
    n_tol = int((~(np.abs(got - ref) <= tol)).sum())
    i, a, b = _first_bad(got, ref)
    raise AssertionError(f"{what}: {n_bits} of {got.size} entries differ from wf1 "
                         f"({n_tol} beyond the 1e-12 bound); first at {i}: {a!r} vs {b!r}")


@pytest.mark.parametrize("workload", ["config3", "config4"])
def test_bench_workload_every_entry(workload):
    import bench
    from paper_2011_11880_b200.plan import Plan

    K = bench.WORKLOADS[workload][1]
    s = bench.build_case(workload)
    plan = Plan(s)
    o = oracle.Oracle(s)
    cptr, cidx = o.pattern_csc()
    pptr, pidx, _ = plan.pattern_csc()
    assert np.array_equal(cptr, pptr) and np.array_equal(cidx, pidx)
    y, pq_p, pq_q, pv_p, out = bench.blocked_inputs(s, K, bench.SEED)
    t = lambda a: torch.from_numpy(a).cuda()
    g, j, n = plan.empty(plan.n_var, K), plan.empty(plan.nnz, K), plan.empty(K)
    plan.eval_batched(K, t(y), t(pq_p), t(pq_q), t(pv_p), t(out), g, j, n)
    jc = plan.empty(plan.nnz, K)
    plan.jac_to_csc(j, jc, K)
    torch.cuda.synchronize()
    del j
    G = g.cpu().numpy()
    del g
    gr, jr, nr = o.eval_scenarios(K, y, pq_p, pq_q, pv_p, out, nthreads=os.cpu_count() or 1)
    _compare(G, gr, f"{workload} residual")
    del gr
    JC = jc.cpu().numpy()
    del jc
    torch.cuda.empty_cache()
    _compare(JC, jr, f"{workload} Jacobian")
    del JC, jr
    norms = n[:K].cpu().numpy()
    assert np.array_equal(norms, nr)
    # and the norm epilogue is the max |g| of what was written
    Gb = G.reshape(-1, plan.n_var, 32)
    mx = np.abs(Gb).max(axis=1).reshape(-1)[:K]
    assert np.array_equal(norms, mx)
