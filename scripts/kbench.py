"""Kernel-only timing of the batched / single-grid evaluation (dev tool)."""
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2011_11880_b200.plan import Plan  # noqa: E402

WL = os.environ.get("WORKLOAD", "config3")
K = int(os.environ.get("K", str(bench.WORKLOADS[WL][1])))
s = bench.build_case(WL)
plan = Plan(s)
y, pq_p, pq_q, pv_p, out = bench.blocked_inputs(s, K, 1000)
t = lambda a: torch.from_numpy(a).cuda()
dy, dp, dq, dv, do = t(y), t(pq_p), t(pq_q), t(pv_p), t(out)
g, j, n = plan.empty(plan.n_var, K), plan.empty(plan.nnz, K), plan.empty(K)
_, _, by = bench.algorithmic_bytes(s, plan.nnz, K)
mode = os.environ.get("MODE", "fj")
gg = g if "f" in mode else None
jj = j if "j" in mode else None
for _ in range(3):
    plan.eval_batched(K, dy, dp, dq, dv, do, gg, jj, n)
ts = []
for _ in range(int(os.environ.get("REPS", "20"))):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); plan.eval_batched(K, dy, dp, dq, dv, do, gg, jj, n); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
med = statistics.median(ts)
tag = os.environ.get("TAG", "") + f" mode={mode}"
print(f"{tag} batched K={K}: {med:.4f} ms  {by/med/1e6:.0f} GB/s  {by/med/1e6/6552.6*100:.1f}%  evals/s {K/med*1e3:.0f}")
