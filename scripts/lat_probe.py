"""Per-launch device time of small kernels inside CUDA graphs (dev tool)."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2011_11880_b200 import synth  # noqa: E402
from paper_2011_11880_b200.plan import Plan, sincos  # noqa: E402
from paper_2011_11880_b200.system_model import build_system, random_state  # noqa: E402

s = build_system(synth.config_case(0, seed=0))
plan = Plan(s)
y = torch.as_tensor(random_state(s, 1), device="cuda")
x = torch.linspace(-1, 1, 2500, dtype=torch.float64, device="cuda")
g, j, n = plan.empty(plan.n_var), plan.empty(plan.nnz), plan.empty(1)
outs = [plan.empty(plan.n_line) for _ in range(4)]


def timed(name, fn, reps=100):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn()
        fn()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        for _ in range(reps):
            fn()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        graph.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / reps)
    print(f"{name:40s} {statistics.median(ts):7.2f} us/launch")


timed("torch add (1 elem)", lambda: n.add_(0.0))
timed("pf_sincos 2500", lambda: sincos(x))
timed("pf_device_jacobian_slots", lambda: plan.device_jacobian_slots(y))
timed("pf_line_injections (2500 br)", lambda: plan.line_injections(y))
timed("pf_eval residual only", lambda: plan.eval(y, g=g))
timed("pf_eval jac only", lambda: plan.eval(y, jval=j))
timed("pf_eval f+J+norm", lambda: plan.eval(y, g, j, n))
