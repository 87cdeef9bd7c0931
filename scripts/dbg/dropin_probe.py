"""Host drop-in timing (dev probe): ResidualWorkspace.run + JacobianWorkspace.run
per Newton-style iteration, unpaired and fused, config 2, median µs."""
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2011_11880_b200 import synth  # noqa: E402
from paper_2011_11880_b200.jacobian import JacobianWorkspace  # noqa: E402
from paper_2011_11880_b200.plan import Plan  # noqa: E402
from paper_2011_11880_b200.residual import ResidualWorkspace  # noqa: E402
from paper_2011_11880_b200.system_model import build_system, random_state  # noqa: E402

for cfg in [int(a) for a in sys.argv[1:]] or [2]:
    s = build_system(synth.config_case(cfg, seed=cfg))
    plan = Plan(s)
    y = np.array(random_state(s, 7))
    for fused in (False, True):
        rws = ResidualWorkspace(s, plan)
        jws = JacobianWorkspace(s, plan, residual_ws=rws) if fused else JacobianWorkspace(s, plan)
        g = np.empty(plan.n_var)
        rws.bind(y, g)
        ts = []
        for k in range(60):
            t0 = time.perf_counter()
            rws.run(y)
            jws.run(y)
            if k >= 10:
                ts.append(time.perf_counter() - t0)
        print(f"config {cfg} {'fused' if fused else 'pair '}: {statistics.median(ts) * 1e6:.0f} us "
              f"(min {min(ts) * 1e6:.0f})")
