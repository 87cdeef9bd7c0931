"""Per-node cost of small graphs (dev probe): launch overhead vs our kernels."""
import statistics, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2011_11880_b200 import synth
from paper_2011_11880_b200.plan import Plan
from paper_2011_11880_b200.system_model import build_system, random_state

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
s = build_system(synth.config_case(cfg, seed=cfg))
plan = Plan(s)
y = torch.as_tensor(random_state(s, 7), device="cuda")
g, j, n = plan.empty(plan.n_var), plan.empty(plan.nnz), plan.empty(1)
x = torch.zeros(16, device="cuda")

def timeit(name, fn, reps=100):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3): fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for _ in range(reps): fn()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); gr.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1000 / reps)
    print(f"cfg{cfg} {name:28s} {statistics.median(ts):7.2f} us/call")

timeit("torch add_ (1 kernel)", lambda: x.add_(1))
timeit("eval g+J+norm", lambda: plan.eval(y, g, j, n))
timeit("eval g only", lambda: plan.eval(y, g=g))
timeit("eval J only", lambda: plan.eval(y, jval=j))
timeit("eval norm only", lambda: plan.eval(y, norm=n))
from paper_2011_11880_b200.plan import sincos as _sc
ss, cc = torch.empty(2500, dtype=torch.float64, device="cuda"), torch.empty(2500, dtype=torch.float64, device="cuda")
timeit("sincos 2500", lambda: _sc(y[:2500]))
