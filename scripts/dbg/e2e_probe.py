"""Host-buffer batched pipeline parameters (dev probe): pf_eval_batched_host
on the config-3 bench workload with pinned buffers, per (blocks_per_stage,
n_streams)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2011_11880_b200.plan import Plan  # noqa: E402

s = bench.build_case("config3")
plan = Plan(s)
K = 256
y, pq_p, pq_q, pv_p, out = bench.blocked_inputs(s, K, 1000)
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
hy, hp, hq, hv, ho = pin(y), pin(pq_p), pin(pq_q), pin(pv_p), pin(out)
hg = torch.empty(K * plan.n_var, dtype=torch.float64).pin_memory().numpy()
hj = torch.empty(K * plan.nnz, dtype=torch.float64).pin_memory().numpy()
hn = torch.empty(K, dtype=torch.float64).pin_memory().numpy()
for bps, ns in [(1, 2), (1, 3), (1, 4), (1, 8), (2, 2), (2, 4)] + [tuple(map(int, a.split(","))) for a in sys.argv[1:]]:
    f = lambda: plan.eval_batched_host(K, hy, hp, hq, hv, ho, hg, hj, hn, blocks_per_stage=bps,
                                       n_streams=ns)
    f()
    t0 = time.perf_counter()
    for _ in range(4):
        f()
    dt = (time.perf_counter() - t0) / 4
    print(f"bps {bps} streams {ns}: {dt * 1e3:.2f} ms/step  {K / dt:.0f} evals/s  "
          f"D2H {(hg.nbytes + hj.nbytes) / dt / 1e9:.1f} GB/s", flush=True)
