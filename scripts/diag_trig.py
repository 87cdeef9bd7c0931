"""Diagnostics: engine trig vs glibc, and parity-failure anatomy on hub grids."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import oracle  # noqa: E402
from paper_2011_11880_b200 import synth  # noqa: E402
from paper_2011_11880_b200.plan import sincos  # noqa: E402


def ulps(a, b):
    ai = a.view(np.int64)
    bi = b.view(np.int64)
    return np.abs(ai - bi)


rng = np.random.default_rng(0)
x = np.concatenate([rng.normal(0, 0.3, 2_000_000), rng.uniform(-np.pi, np.pi, 1_000_000)])
s_ref, c_ref = oracle.libm_sincos(x)
sg, cg = sincos(torch.as_tensor(x, device="cuda"))
sg, cg = sg.cpu().numpy(), cg.cpu().numpy()
for name, a, b in (("sin", sg, s_ref), ("cos", cg, c_ref)):
    u = ulps(a, b)
    print(f"{name}: differ {np.mean(u > 0) * 100:.3f}%  max ulp {u.max()}  hist {np.bincount(u)[:5]}")

# ---- parity-failure anatomy on a hub grid -------------------------------------
from paper_2011_11880_b200.batched import ScenarioBuffers  # noqa: E402
from paper_2011_11880_b200.plan import Plan, from_blocked, to_blocked  # noqa: E402
from paper_2011_11880_b200.system_model import build_system  # noqa: E402

s = build_system(synth.synth_case(20_000, 25_000, seed=9, pq_frac=0.6, pv_frac=0.15,
                                  hub_frac=0.01, hub_degree=50, shunt_frac=0.05))
plan = Plan(s)
K = 40
sb = synth.make_scenarios(s, K, seed=2)
buf = ScenarioBuffers(plan, K)
buf.upload(sb)
buf.evaluate()
torch.cuda.synchronize()
o = oracle.Oracle(s)
_, _, perm = plan.pattern_csc()
g_ref, j_ref, _ = o.eval_scenarios(K, to_blocked(sb.y.T), to_blocked(sb.pq_p.T),
                                   to_blocked(sb.pq_q.T), to_blocked(sb.pv_p.T), sb.outage,
                                   nthreads=8)
G = buf.residual()
J = buf.jacobian_csr()[:, perm]
g_ref = from_blocked(g_ref, K, plan.n_var)
j_ref = from_blocked(j_ref, K, plan.nnz)
cptr, cidx, _ = plan.pattern_csc()
for nm, a, b in (("g", G, g_ref), ("J", J, j_ref)):
    tol = np.maximum(1e-12 * np.abs(b), 1e-14)
    bad = np.argwhere(np.abs(a - b) > tol)
    exact = np.mean(a == b) * 100
    print(f"{nm}: bit-exact {exact:.2f}%  failures {len(bad)}  max|d| {np.abs(a-b).max():.3e}")
    for k, e in bad[:10]:
        extra = ""
        if nm == "J":
            col = np.searchsorted(cptr, e, side="right") - 1
            extra = f" row {cidx[e]} col {col}"
        print(f"   scen {k} entry {e}{extra}: got {a[k, e]!r} ref {b[k, e]!r} d {a[k,e]-b[k,e]:.3e}")
