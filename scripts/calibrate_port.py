"""Calibrates the oracle port against pflow itself (dev tool; runs only
where /root/reference is importable, never on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
    PYTHONPATH=/root/reference/pkg/src:. python scripts/calibrate_port.py

It times pflow's Numba workflows (wf5, wf1 single-threaded; wf6, wf3
threaded) and the C restatement's wf5 / wf1 on the same config-3 grid and
state in the same process, per f+J.  The port stands in for pflow in
`bench.py --impl reference` and in `cpu_baseline`."""
import os, sys, time, statistics
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2011_11880_b200 import synth
from paper_2011_11880_b200.case import to_rows
from paper_2011_11880_b200.system_model import build_system as our_build
import pflow
from pflow import residual as R, jacobian as J
from pflow.workflow import workflow_config
import oracle
raw = synth.config_case(3, seed=3)
psys = pflow.build_system(to_rows(raw))
osys = our_build(raw)
y = synth.make_scenarios(osys, 1, seed=5).y[:, 0].copy()
out = np.zeros(psys_n := len(y))
rws = R.ResidualWorkspace(psys); jws = J.symbolic_pattern(psys)
res = {}
for wf in (5, 1, 6, 3):
    cfg = workflow_config(wf, 1) if wf in (1, 5) else workflow_config(wf)
    f = lambda: (R.evaluate_residual(psys, y, cfg, out, rws), J.evaluate_jacobian(psys, y, cfg, jws))
    f(); f()
    ts = []
    for _ in range(15):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    res[wf] = statistics.median(ts)
    print(f"pflow wf{wf}: {res[wf]*1e3:.2f} ms per f+J", flush=True)
o = oracle.Oracle(osys)
for wf in (5, 1):
    ts = []
    for _ in range(15):
        t0 = time.perf_counter(); o.residual(y, wf); o.jacobian(y, wf); ts.append(time.perf_counter() - t0)
    print(f"C port wf{wf}: {statistics.median(ts)*1e3:.2f} ms per f+J (incl. numpy out alloc)", flush=True)
# per-scenario batched path of the port, 1 thread
from paper_2011_11880_b200.plan import to_blocked
sb = synth.make_scenarios(osys, 16, seed=5)
args = (16, to_blocked(sb.y.T), to_blocked(sb.pq_p.T), to_blocked(sb.pq_q.T), to_blocked(sb.pv_p.T), sb.outage)
for wf in (5,):
    o.eval_scenarios(*args, want_g=False, want_j=False, wf=wf, nthreads=1)
    t0 = time.perf_counter(); o.eval_scenarios(*args, want_g=False, want_j=False, wf=wf, nthreads=1); dt = time.perf_counter() - t0
    print(f"C port eval_scenarios wf{wf}, 1 thread: {dt/16*1e3:.2f} ms per scenario (with mutation)")
print("cpus", os.cpu_count())
