"""Batched Newton on the device vs pflow's loop on the CPU.

Usage: ``batched_newton_bench.py [K] [n_bus] [device|cusolverrf]``.

Workload: a config-0-shaped synthetic grid (default 2,000 buses, 2,500 branches) with
loads scaled to 5 % so that Newton converges from a flat start; K scenarios
from ``synth.make_scenarios`` (load / PV scaling, one outage each).

* GPU: ``batched_newton_solve``. Evaluation runs through pf_eval_batched.
  The linear solves use the batched sparse LU on the device (``device``, the
  default) or one cusolverRf handle per scenario (``cusolverrf``).
* CPU: pflow/newton.py's loop restated on the C oracle (wf1 g and J) with
  SuperLU, one scenario after another, on one core.

Prints one JSON line: both times, per-phase GPU timings, and the agreement
(outcomes, iteration counts, max |y_gpu - y_cpu|).
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import torch

    import oracle
    from test_gpu_parity import _cpu_newton, _light_case
    from paper_2011_11880_b200 import synth
    from paper_2011_11880_b200.batched_newton import batched_newton_solve
    from paper_2011_11880_b200.plan import Plan, from_blocked, to_blocked
    from paper_2011_11880_b200.system_model import build_system, flat_start

    K = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    linear = sys.argv[3] if len(sys.argv) > 3 else "device"
    import os
    scale = float(os.environ.get("LOAD_SCALE", "0.05"))
    s = build_system(_light_case(nb, nb * 5 // 4, seed=0, scale=scale))
    plan = Plan(s)
    o = oracle.Oracle(s)
    sb = synth.make_scenarios(s, K, seed=1)
    y0 = flat_start(s)
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
    t = lambda a: dev(to_blocked(np.ascontiguousarray(a.T)))
    args = (t(sb.pq_p), t(sb.pq_q), t(sb.pv_p), torch.as_tensor(sb.outage, device="cuda"))
    # warm-up (library load, kernels)
    yw = dev(to_blocked(np.tile(y0, (K, 1))))
    batched_newton_solve(plan, K, yw, *args, linear=linear)
    y = dev(to_blocked(np.tile(y0, (K, 1))))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = batched_newton_solve(plan, K, y, *args, linear=linear)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    Y = from_blocked(y.cpu().numpy(), K, plan.n_var)

    import os
    kc = min(K, int(os.environ.get("CPU_K", K)))   # CPU reference on the first kc scenarios
    t0 = time.perf_counter()
    cpu = [_cpu_newton(o, y0, sb.pq_p[:, k].copy(), sb.pq_q[:, k].copy(), sb.pv_p[:, k].copy(),
                       int(sb.outage[k])) for k in range(kc)]
    cpu_s = (time.perf_counter() - t0) * K / kc
    agree = sum(int((st == "converged") == bool(res.converged[k])) for k, (st, _, _) in enumerate(cpu))
    same_it = sum(int(st == "converged" and res.converged[k] and res.iterations[k] == it)
                  for k, (st, it, _) in enumerate(cpu))
    conv = [k for k, (st, _, _) in enumerate(cpu) if st == "converged" and res.converged[k]]
    diffs = {k: float(np.abs(Y[k] - cpu[k][2]).max()) for k in conv}
    dmax = max(diffs.values(), default=None)
    worst = sorted(diffs.items(), key=lambda kv: -kv[1])[:3]
    worst = [(k, v, int(np.abs(Y[k] - cpu[k][2]).argmax()), float(Y[k][int(np.abs(Y[k] - cpu[k][2]).argmax())]),
              float(cpu[k][2][int(np.abs(Y[k] - cpu[k][2]).argmax())]), int(sb.outage[k])) for k, v in worst]
    line = {
        "workload": f"{nb}-bus synthetic grid (loads x{scale}), K={K} scenarios, Newton from flat "
                    "start, tol 1e-8", "linear": linear,
        "n_var": plan.n_var, "nnz": plan.nnz,
        "gpu_s": gpu_s, "gpu_timings_s": res.timings,
        "gpu_scenarios_per_s": K / gpu_s,
        "cpu_s": cpu_s, "cpu_scenarios_per_s": K / cpu_s, "cpu_cores": 1,
        "cpu_scenarios_checked": kc,
        "converged_gpu": int(res.converged.sum()), "singular_gpu": int(res.singular.sum()),
        "converged_cpu": sum(int(st == "converged") for st, _, _ in cpu),
        "converged_gpu_checked": int(res.converged[:kc].sum()),
        "outcome_agreement": agree, "same_iterations": same_it,
        "max_abs_state_diff": dmax, "worst_state_diffs": worst,
        "iterations": int(res.iterations.max()), "n_bus": s.n_bus,
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
