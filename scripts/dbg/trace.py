"""Per-phase globaltimer trace of k_eval_single (dev probe; needs the library
built with -DPF_X_TRACE, see profiles/r01_single_grid.md)."""
import ctypes, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2011_11880_b200 import synth
from paper_2011_11880_b200._abi import lib
from paper_2011_11880_b200.plan import Plan
from paper_2011_11880_b200.system_model import build_system, random_state

STAMPS = [(0, "start"), (1, "plan loads issued"), (2, "after wait"), (3, "phase0 done"),
          (6, "barrier0"), (7, "phaseA done"), (8, "barrierA"), (4, "fold done"),
          (5, "devices done"), (9, "phaseB done"), (10, "barrierB"), (11, "norm done")]
for cfg in [int(a) for a in sys.argv[1:]] or [0, 2]:
    s = build_system(synth.config_case(cfg, seed=cfg)); plan = Plan(s)
    ys = [torch.as_tensor(random_state(s, 7 + k), device="cuda") for k in range(10)]
    g, j, n = plan.empty(plan.n_var), plan.empty(plan.nnz), plan.empty(1)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for k in range(3): plan.eval(ys[k], g, j, n)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for k in range(10): plan.eval(ys[k], g, j, n)
    gr.replay(); torch.cuda.synchronize()
    buf = np.zeros(2048 * 16, dtype=np.uint64)
    lib().pf_debug_trace(ctypes.c_void_p(buf.ctypes.data))
    tr = buf.astype(np.int64).reshape(2048, 16)[: plan.single_chunks]
    t0 = tr[:, 0].min()
    rel = (tr - tr[:, :1]) / 1000.0
    print(f"config {cfg}: {len(tr)} CTAs; last CTA end {(tr[:, 11].max() - t0) / 1000:.2f} us; "
          f"CTA start spread {(tr[:, 0].max() - t0) / 1000:.2f} us")
    print("  median:", "  ".join(f"{nm}={np.median(rel[:, k]):.2f}" for k, nm in STAMPS))
    print("  max:   ", "  ".join(f"{nm}={np.max(rel[:, k]):.2f}" for k, nm in STAMPS))
