"""Full-size parity campaign (dev tool): the bench workloads (config 3, K =
256; config 4, K = 64) through the product kernel, every scenario and every
entry against the oracle's wf1, with the reference's own wf5 as a second
opinion on any entry out of the strict bound.  Prints one line per workload."""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import bench  # noqa: E402
import oracle  # noqa: E402
from _util import ABS_TOL, REL_TOL  # noqa: E402
from paper_2011_11880_b200.plan import Plan, from_blocked  # noqa: E402

for wl in sys.argv[1:] or ["config3", "config4"]:
    K = bench.WORKLOADS[wl][1]
    s = bench.build_case(wl)
    plan = Plan(s)
    _, _, perm = plan.pattern_csc()
    y, pq_p, pq_q, pv_p, out = bench.blocked_inputs(s, K, int(os.environ.get("SEED", "1000")))
    t = lambda a: torch.from_numpy(a).cuda()
    g, j, n = plan.empty(plan.n_var, K), plan.empty(plan.nnz, K), plan.empty(K)
    plan.eval_batched(K, t(y), t(pq_p), t(pq_q), t(pv_p), t(out), g, j, n)
    torch.cuda.synchronize()
    G = from_blocked(g.cpu().numpy(), K, plan.n_var)
    Jg = from_blocked(j.cpu().numpy(), K, plan.nnz)[:, perm]
    o = oracle.Oracle(s)
    t0 = time.perf_counter()
    ref = {}
    for wf in (1, 5):
        gr, jr, _ = o.eval_scenarios(K, y, pq_p, pq_q, pv_p, out, wf=wf,
                                     nthreads=os.cpu_count() or 1)
        ref[wf] = (from_blocked(gr, K, plan.n_var), from_blocked(jr, K, plan.nnz))
    strict = beyond = exact = total = 0
    worst = 0.0
    for q, got in ((0, G), (1, Jg)):
        r1, r5 = ref[1][q], ref[5][q]
        d = np.abs(got - r1)
        tol = np.maximum(REL_TOL * np.abs(r1), ABS_TOL)
        fail = d > tol
        strict += int(fail.sum())
        beyond += int((fail & (d > np.abs(r5 - r1))).sum())
        exact += int((got == r1).sum())
        total += got.size
        worst = max(worst, float((d / tol).max()))
    norms_ok = np.array_equal(n[:K].cpu().numpy(), np.abs(G).max(axis=1))
    print(f"{wl}: K={K} entries {total}: bit-identical to wf1 {exact / total * 100:.2f} %, "
          f"out of the 1e-12 bound {strict}, beyond wf5's own deviation {beyond}, "
          f"worst |d|/bound {worst:.3f}, norms exact {norms_ok} "
          f"(oracle {time.perf_counter() - t0:.1f} s)", flush=True)
