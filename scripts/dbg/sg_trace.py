"""Per-phase %globaltimer trace of k_eval_single (dev probe).  Needs the
library built with -DPF_X_TRACE:
    python paper_2011_11880_b200/build.py --variant trace PF_X_TRACE
    PFGPU_LIB_PARTIAL=1 PFGPU_LIB=build/var/trace.so python scripts/dbg/sg_trace.py 2
Runs a CUDA graph of 10 back-to-back evaluations and prints the last one's
stamps (µs, relative to the earliest griddepcontrol.wait return = the end of
the previous evaluation)."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2011_11880_b200 import synth  # noqa: E402
from paper_2011_11880_b200._abi import lib  # noqa: E402
from paper_2011_11880_b200.plan import Plan  # noqa: E402
from paper_2011_11880_b200.system_model import build_system, random_state  # noqa: E402

import os
MODE = os.environ.get("MODE", "fjn")   # outputs: f (g), j (J), n (norm)
NAMES = ["start", "pre-wait", "wait done", "y loaded", "phase A", "phase B", "norm", "end"]
for cfg in [int(a) for a in sys.argv[1:]] or [0, 2]:
    s = build_system(synth.config_case(cfg, seed=cfg))
    plan = Plan(s)
    ys = [torch.as_tensor(random_state(s, 7 + k), device="cuda") for k in range(10)]
    g, j, n = plan.empty(plan.n_var), plan.empty(plan.nnz), plan.empty(1)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for k in range(3):
            plan.eval(ys[k], g, j, n)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for k in range(10):
            plan.eval(ys[k], g if "f" in MODE else None, j if "j" in MODE else None,
                      n if "n" in MODE else None)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    buf = np.zeros(4096 * 8, dtype=np.uint64)
    lib().pf_debug_sg_trace(ctypes.c_void_p(buf.ctypes.data))
    tr = buf.astype(np.int64).reshape(4096, 8)[: plan.single_chunks]
    t0 = tr[:, 2].min()
    rel = (tr - t0) / 1000.0
    print(f"[{MODE}] config {cfg}: {len(tr)} CTAs (µs from the first wait return)")
    for k, nm in enumerate(NAMES):
        c = rel[:, k]
        print(f"  {nm:10s} min {c.min():7.2f}  median {np.median(c):7.2f}  max {c.max():7.2f}")
    d = np.diff(tr[:, 2:8], axis=1) / 1000.0
    print("  per-CTA phase durations (median):", "  ".join(
        f"{NAMES[k + 3]}={np.median(d[:, k]):.2f}" for k in range(d.shape[1])))
