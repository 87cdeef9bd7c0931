"""Locate and import the live reference package ``pflow`` - TEST / BASELINE
INFRASTRUCTURE ONLY (same rules as the rest of ``oracle/``).

pflow is Python + Numba.  It is looked for, in order, at ``$PFLOW_SRC``,
``baseline/_ref`` (the offline ``pip install --target`` of /root/reference/pkg
that travels to the GPU box) and /root/reference/pkg/src (this
container only).  Numba's on-disk cache goes to a writable temp directory so
nothing is written into the reference tree.
"""

from __future__ import annotations

import importlib
import os
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
_CANDIDATES = [os.environ.get("PFLOW_SRC"), str(ROOT / "baseline" / "_ref"),
               "/root/reference/pkg/src"]
_STATE: dict = {}


def import_pflow():
    """(module, None) or (None, reason)."""
    if "mod" in _STATE:
        return _STATE["mod"], _STATE.get("why")
    os.environ.setdefault("NUMBA_CACHE_DIR", str(Path(tempfile.gettempdir()) / "pflow_numba"))
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    why = "pflow not found at $PFLOW_SRC, baseline/_ref or /root/reference/pkg/src"
    mod = None
    for c in _CANDIDATES:
        if c and (Path(c) / "pflow" / "__init__.py").exists():
            if c not in sys.path:
                sys.path.insert(0, c)
            try:
                mod = importlib.import_module("pflow")
                why = None
                _STATE["path"] = c
            except Exception as e:  # noqa: BLE001 (numba / scipy missing, ...)
                why = f"pflow at {c} failed to import: {e!r}"
            break
    _STATE["mod"], _STATE["why"] = mod, why
    return mod, why


def location() -> str | None:
    return _STATE.get("path")


def pflow_system(pflow, raw_case):
    """pflow's own PowerSystem for one of this package's RawCase objects: the
    case goes through MATPOWER text (case.write_case -> pflow.parse_case), so
    pflow builds it with its own parser and build_system."""
    from paper_2011_11880_b200 import case as C

    return pflow.build_system(pflow.parse_case(C.write_case(raw_case), name=raw_case.name))


def pflow_fixture(pflow, name: str):
    """pflow's bundled MATPOWER fixture (cases/<name>.m) through pflow."""
    path = Path(pflow.__file__).resolve().parent / "cases" / f"{name}.m"
    return pflow.build_system(pflow.parse_case_file(path))


# ---------------------------------------------------------------------------
# live-pflow CPU baselines (bench.py's cpu_baseline_pflow legs)
# ---------------------------------------------------------------------------

def time_single_grid(pflow, psys, y, threads: int, min_seconds: float = 1.0) -> dict:
    """pflow's own f+J (evaluate_residual + evaluate_jacobian on bound
    workspaces) under each of its six workflows with ``threads`` pool
    workers; warm-up discarded, median per f+J (the pflow/bench.py:82-90
    method).  Returns the fastest and every workflow's median."""
    import statistics
    import time

    import numpy as np

    pflow.set_worker_count(max(threads, 6))     # wf4 needs >= 6 (workflow.py:209-212)
    y = np.array(y, dtype=np.float64)
    out = np.zeros(psys.n_var)
    res_ws = pflow.ResidualWorkspace(psys)
    jac_ws = pflow.symbolic_pattern(psys)
    med = {}
    for wf in range(1, 7):
        cfg = pflow.workflow_config(wf, threads)
        pflow.evaluate_residual(psys, y, cfg, out, res_ws)
        pflow.evaluate_jacobian(psys, y, cfg, jac_ws)
        times, t_start = [], time.perf_counter()
        while len(times) < 5 or time.perf_counter() - t_start < min_seconds:
            t0 = time.perf_counter()
            pflow.evaluate_residual(psys, y, cfg, out, res_ws)
            pflow.evaluate_jacobian(psys, y, cfg, jac_ws)
            times.append(time.perf_counter() - t0)
        med[wf] = statistics.median(times)
    best = min(med, key=med.get)
    return {"value": 1.0 / med[best], "unit": "evals/s", "us_per_eval": med[best] * 1e6,
            "wf": best, "cores": threads if best in (2, 3, 4, 6) else 1,
            "kind": "reference",
            "per_workflow_us": {str(k): v * 1e6 for k, v in med.items()},
            "sample": f"live pflow {pflow.__version__} (Numba), evaluate_residual + "
                      "evaluate_jacobian on bound workspaces, each of wf1-6, median per f+J, "
                      "fastest reported"}


def _scenario_worker(args):
    """One process of the batched baseline: its own PowerSystem, mutated in
    place per scenario, wf5 on one thread
    (PAPER.md:416-422).  Returns (scenarios done, seconds)."""
    import time

    import numpy as np

    text, name, K, seed, lo, hi, wf, nthreads = args
    pflow, why = import_pflow()
    if pflow is None:
        raise RuntimeError(why)
    from paper_2011_11880_b200 import synth

    psys = pflow.build_system(pflow.parse_case(text, name=name))
    sb = synth.make_scenarios(psys, K, seed)
    pflow.set_worker_count(max(nthreads, 1))
    cfg = pflow.workflow_config(wf, nthreads)
    out = np.zeros(psys.n_var)
    res_ws = pflow.ResidualWorkspace(psys)
    jac_ws = pflow.symbolic_pattern(psys)
    ln, pq, pv = psys.lines, psys.pq, psys.pv
    coef = [ln.gl, ln.bl, ln.gl2, ln.bl2, ln.g_self_h, ln.b_self_h, ln.g_self_k, ln.b_self_k]
    p0, q0, v0 = pq.p0.copy(), pq.q0.copy(), pv.p0.copy()

    def one(k):
        y = np.ascontiguousarray(sb.y[:, k])
        pq.p0[:] = sb.pq_p[:, k]
        pq.q0[:] = sb.pq_q[:, k]
        pv.p0[:] = sb.pv_p[:, k]
        o = int(sb.outage[k])
        saved = [c[o] for c in coef] if o >= 0 else None
        if o >= 0:
            for c in coef:
                c[o] = 0.0
        pflow.evaluate_residual(psys, y, cfg, out, res_ws)
        pflow.evaluate_jacobian(psys, y, cfg, jac_ws)
        if o >= 0:
            for c, v in zip(coef, saved):
                c[o] = v
        pq.p0[:], pq.q0[:], pv.p0[:] = p0, q0, v0

    one(lo)                                   # warm-up (JIT / cache load)
    t0 = time.perf_counter()
    for k in range(lo, hi):
        one(k)
    return hi - lo, time.perf_counter() - t0


def time_batched(pflow, raw_case, K: int, seed: int, procs: int, n_scen: int,
                 wf: int = 5) -> dict:
    """the paper's recommended batch -- independent
    single-threaded wf5 jobs in parallel processes, one
    per core, over the first ``n_scen`` of the workload's K scenarios (a
    bounded sample) -- and wf3 (threaded inside each model, all cores) run
    sequentially over scenarios in one process; the better is reported."""
    import multiprocessing as mp

    from paper_2011_11880_b200 import case as C

    text = C.write_case(raw_case)
    # populate Numba's on-disk cache once before the workers load it
    _scenario_worker((text, raw_case.name, K, seed, 0, 1, wf, 1))
    n_scen = min(n_scen, K)
    cuts = [n_scen * r // procs for r in range(procs + 1)]
    jobs = [(text, raw_case.name, K, seed, cuts[r], cuts[r + 1], wf, 1) for r in range(procs)
            if cuts[r + 1] > cuts[r]]
    with mp.get_context("spawn").Pool(len(jobs)) as pool:
        res = pool.map(_scenario_worker, jobs)
    done = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    par = {"value": done / wall, "cores": len(jobs), "wf": wf,
           "sample": f"{done} of the {K} scenarios, {len(jobs)} processes x wf{wf} "
                     "single-threaded, each mutating its own PowerSystem per scenario; "
                     "evals / slowest process's time"}
    n_seq = max(2, min(K, n_scen // 4))
    with mp.get_context("spawn").Pool(1) as pool:
        seq_done, seq_s = pool.map(_scenario_worker,
                                   [(text, raw_case.name, K, seed, 0, n_seq, 3, procs)])[0]
    seq = {"value": seq_done / seq_s, "cores": procs, "wf": 3,
           "sample": f"{seq_done} of the {K} scenarios one after another in one process, "
                     f"wf3 on {procs} threads, mutating the PowerSystem per scenario"}
    best = par if par["value"] >= seq["value"] else seq
    return {"value": best["value"], "unit": "evals/s", "cores": best["cores"],
            "kind": "reference", "wf": best["wf"],
            "sample": f"live pflow {pflow.__version__} (Numba), better of two batch modes: "
                      + best["sample"],
            "modes": {"wf5_processes": par, "wf3_sequential": seq}}
