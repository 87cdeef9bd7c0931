"""Larger randomized parity campaign (dev tool): grids of 1k-6k buses with
hubs of degree up to 120, phase shifters, taps, shunts and out-of-service
rows; single grid and a batch of scenarios against the oracle."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle  # noqa: E402
from _util import parity_failures  # noqa: E402
from paper_2011_11880_b200 import synth  # noqa: E402
from paper_2011_11880_b200.plan import Plan, from_blocked, to_blocked  # noqa: E402
from paper_2011_11880_b200.system_model import build_system, random_state  # noqa: E402

lo, hi = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (0, 20)))
bad = []
dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
for seed in range(lo, hi):
    rng = np.random.default_rng(5000 + seed)
    nb = int(rng.integers(1000, 6000))
    case = synth.synth_case(nb, int(nb * rng.uniform(1.1, 1.6)), seed=seed,
                            pq_frac=float(rng.uniform(0.3, 0.9)), pv_frac=float(rng.uniform(0.05, 0.3)),
                            shunt_frac=float(rng.uniform(0, 0.3)), shift_frac=float(rng.uniform(0, 0.3)),
                            out_of_service_frac=float(rng.uniform(0, 0.1)),
                            hub_frac=float(rng.uniform(0, 0.02)), hub_degree=int(rng.integers(20, 120)))
    s = build_system(case)
    plan = Plan(s)
    o = oracle.Oracle(s)
    _, _, perm = plan.pattern_csc()
    y = random_state(s, seed)
    g, j, n = plan.empty(plan.n_var), plan.empty(plan.nnz), plan.empty(1)
    plan.eval(dev(y), g, j, n)
    torch.cuda.synchronize()
    f = parity_failures(g[: plan.n_var].cpu().numpy(), o.residual(y)) + \
        parity_failures(j[: plan.nnz].cpu().numpy()[perm], o.jacobian(y))
    K = int(rng.integers(1, 100))
    sb = synth.make_scenarios(s, K, seed=seed)
    t = lambda a: dev(to_blocked(np.ascontiguousarray(a.T)))
    gb, jb, nr = plan.empty(plan.n_var, K), plan.empty(plan.nnz, K), plan.empty(K)
    plan.eval_batched(K, t(sb.y), t(sb.pq_p), t(sb.pq_q), t(sb.pv_p), dev(sb.outage), gb, jb, nr)
    torch.cuda.synchronize()
    gr, jr, _ = o.eval_scenarios(K, to_blocked(sb.y.T), to_blocked(sb.pq_p.T), to_blocked(sb.pq_q.T),
                                 to_blocked(sb.pv_p.T), sb.outage, nthreads=8)
    G = from_blocked(gb.cpu().numpy(), K, plan.n_var)
    J = from_blocked(jb.cpu().numpy(), K, plan.nnz)
    f += parity_failures(G, from_blocked(gr, K, plan.n_var))
    f += parity_failures(J[:, perm], from_blocked(jr, K, plan.nnz))
    print(f"seed {seed}: buses {nb} max degree {plan.max_degree} serial chunks {plan.single_serial} "
          f"K {K}: {f} failures", flush=True)
    if f:
        bad.append(seed)
print(f"large fuzz {lo}..{hi - 1}: {hi - lo - len(bad)} passed, {len(bad)} failed {bad}")
