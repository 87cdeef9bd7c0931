import sys, statistics
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2011_11880_b200 import synth
from paper_2011_11880_b200.plan import Plan
from paper_2011_11880_b200.system_model import build_system, random_state
for cfg in (0, 2):
    s = build_system(synth.config_case(cfg, seed=cfg)); plan = Plan(s)
    y = torch.as_tensor(random_state(s, 7), device="cuda")
    g, j, n = plan.empty(plan.n_var), plan.empty(plan.nnz), plan.empty(1)
    for _ in range(5): plan.eval(y, g, j, n)
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3): plan.eval(y, g, j, n)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for _ in range(10): plan.eval(y, g, j, n)
    gr.replay(); torch.cuda.synchronize()
    import ctypes
    from paper_2011_11880_b200._abi import lib
    buf = np.zeros(1024 * 16, dtype=np.uint64)
    lib().pf_debug_trace(buf.ctypes.data_as(ctypes.c_void_p))
    nch = plan.dims()["sg_chunks"] if hasattr(plan, "dims") and isinstance(plan.dims(), dict) and "sg_chunks" in plan.dims() else 1024
    tr = buf.astype(np.int64).reshape(1024, 16)
    used = tr[:, 0] > 0
    tr = tr[used]
    names = ["start", "tab", "ph0", "bar0", "phA", "barA", "phB", "barB", "norm", "out"]
    t0 = tr[:, 0].min()
    print(f"config {cfg}: {len(tr)} CTAs traced; end of last CTA {(tr[:, 9].max() - t0)/1000:.2f} us")
    rel = (tr[:, :10] - tr[:, :1]) / 1000.0
    print("median per-CTA timeline (us from CTA start):", " ".join(f"{nm}={v:.2f}" for nm, v in zip(names, np.median(rel, axis=0))))
    print("max    per-CTA timeline (us from CTA start):", " ".join(f"{nm}={v:.2f}" for nm, v in zip(names, np.max(rel, axis=0))))
    st0 = (tr[:, 0] - t0) / 1000.0
    print("CTA start spread: median", np.median(st0), "max", st0.max())
