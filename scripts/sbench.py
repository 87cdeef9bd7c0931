"""Single-grid f+J timing (dev tool): per-call (host submission included)
and device time via a CUDA graph of 100 evaluations on 100 perturbed states
(BASELINE config 1 style), with the L2 flushed only before the graph."""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2011_11880_b200 import synth  # noqa: E402
from paper_2011_11880_b200.plan import Plan  # noqa: E402
from paper_2011_11880_b200.system_model import build_system, random_state  # noqa: E402

for cfg in (int(a) for a in (sys.argv[1:] or ["2"])):
    s = build_system(synth.config_case(cfg, seed=cfg))
    plan = Plan(s)
    y0 = random_state(s, 7)
    ys = torch.as_tensor(synth.perturbed_states(y0, s.n_bus, 100, seed=8), device="cuda")
    g, j, n = plan.empty(plan.n_var), plan.empty(plan.nnz), plan.empty(1)
    norms = torch.empty(100, dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            plan.eval(ys[0], g, j, n)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    import os
    mode = os.environ.get("MODE", "fjn")   # which outputs: f (g), j (J), n (norm)
    with torch.cuda.graph(graph, stream=st):
        for k in range(100):
            plan.eval(ys[k], g if "f" in mode else None, j if "j" in mode else None,
                      norms[k:k + 1] if "n" in mode else None)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        graph.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 10)   # us per evaluation
    print(f"[{mode}] config {cfg}: n_var {plan.n_var} nnz {plan.nnz}  graph {statistics.median(ts):.2f} "
          f"us/eval (100 states, min {min(ts):.2f})")
