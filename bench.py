"""Benchmark: f+J evaluations/s on the 70k-bus synthetic grid (BASELINE.json).

Workload (per rank, weak scaling): BASELINE config 3 - the config-2-shaped
70,000-bus / 88,000-branch grid shared by K = 256 scenarios (per-device load
scaling U(0.8,1.2), PV scaling U(0.5,1.5), one outaged branch each).  One
step = one fused residual + Jacobian + infinity-norm evaluation of all K
scenarios on the GPU (``pf_eval_batched``), followed on N > 1 by the NCCL
all-gather of the per-scenario norms.  Inputs are resident in HBM; the step
moves ~2.8 GB, more than the 126 MB L2, so no flush is needed.

Extra lines of evidence in the same JSON object:
  roofline      algorithmic bytes / measured kernel time vs MEASURED_PEAKS.json
  e2e           the same metric through the host-buffer C ABI
                (pf_eval_batched_host: H2D inputs, D2H g + J + norms)
  cpu_baseline  the CPU oracle port (C restatement of pflow) on this host
  single_grid   config 2 single grid (one 70k evaluation, L2 flushed between)

``--impl reference`` times the reference algorithm's CPU restatement (the
oracle port; pflow itself is Python and does not travel to the GPU box) with
all host threads on the same workload and prints the same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "f+J evals/s on 70k-bus synthetic grid (fp64); HBM GB/s as % of peak"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def algorithmic_bytes(sys_, nnz: int, K: int) -> tuple[int, int, int]:
    """per-scenario bytes and shared static bytes per launch."""
    n_var = sys_.n_var
    P, G, S, L = len(sys_.pq), len(sys_.pv), len(sys_.slack), len(sys_.lines)
    per_scen = 8 * n_var + 16 * P + 8 * G + 4 + 8 * n_var + 8 * nnz + 8
    coef = 8 * (8 if sys_.lines.has_shift else 6)
    static = L * (8 + coef) + 4 * P + 12 * G + 20 * S
    return per_scen, static, per_scen * K + static


def workload_config(workload: str, sys_, nnz: int) -> dict:
    """The line's `config`: properties of the workload only, computed the same
    way by both arms (so the driver sees one config); how an arm runs it
    goes in the line's `run`."""
    import numpy as np

    K = WORKLOADS[workload][1]
    _, _, by = algorithmic_bytes(sys_, nnz, K)
    deg = np.bincount(np.concatenate([sys_.lines.bus_h, sys_.lines.bus_k]),
                      minlength=sys_.n_bus)
    return {"workload": workload_desc(workload), "n_var": int(sys_.n_var), "nnz": int(nnz),
            "scenarios_total": K, "max_bus_degree": int(deg.max()) if deg.size else 0,
            "l2": (f"inputs+outputs of the {K}-scenario step {by / 1e9:.2f} GB > 126 MB L2 "
                   "(no flush needed)")}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        time.sleep(0.3)

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.2)
        self.p.terminate()
        self.p.wait()
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 8 and r[1].strip().isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 8 and r[2].strip().isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 8 for i in range(4)
                          if r[4 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


WORKLOADS = {
    # name: (BASELINE config, scenarios, default scaling, description)
    # config 3 is "K=256 sharded across 1/2/4/8 B200" (strong: the same 256
    # scenarios split over the ranks); config 4 is "K=64 scenarios per GPU"
    # (weak: every rank evaluates its own 64).
    "config3": (3, 256, "strong", "config3: 70k-bus/88k-branch grid (45k PQ, 6k PV, 1 slack), "
                                  "K=256 scenarios per step"),
    "config4": (4, 64, "weak", "config4 stress: 200k-bus/250k-branch grid + 1% degree-50 hub "
                               "buses, K=64 scenarios per GPU per step"),
}
SEED = 1000   # scenario seed of the bench workloads (tests/test_gpu_fullsize.py checks them)
SCEN = ("per-device load U(0.8,1.2) + PV U(0.5,1.5) scaling, 1 outaged branch each; "
        "fused f+J+inf-norm")


def workload_desc(workload: str) -> str:
    """The workload string both arms print (so the driver sees one config)."""
    return f"{WORKLOADS[workload][3]}, {SCEN}"


def build_case(workload: str = "config3"):
    from paper_2011_11880_b200 import synth
    from paper_2011_11880_b200.system_model import build_system

    cfg = WORKLOADS[workload][0]
    return build_system(synth.config_case(cfg, seed=cfg))


def blocked_inputs(sys_, K, seed, lo: int = 0, hi: int | None = None):
    """Blocked-layout inputs of scenarios [lo, hi) of the K-scenario batch
    drawn with ``seed`` (a rank's shard; the whole batch by default)."""
    from paper_2011_11880_b200 import synth
    from paper_2011_11880_b200.plan import to_blocked

    hi = K if hi is None else hi
    sb = synth.make_scenarios(sys_, K, seed)
    c = lambda a: np.ascontiguousarray(a[:, lo:hi].T)
    return (to_blocked(c(sb.y)), to_blocked(c(sb.pq_p)), to_blocked(c(sb.pq_q)),
            to_blocked(c(sb.pv_p)), np.ascontiguousarray(sb.outage[lo:hi], dtype=np.int32))


def rank_workload(workload: str, scaling: str, rank: int, world: int):
    """(K_total, lo, hi, seed, K_gen) of this rank: strong scaling splits the
    workload's K scenarios with batched.shard; weak scaling gives every rank
    its own K (seed SEED + rank)."""
    from paper_2011_11880_b200.batched import shard

    K = WORKLOADS[workload][1]
    if scaling == "strong":
        lo, hi = shard(K, rank, world)
        return K, lo, hi, SEED, K
    return K * world, 0, K, SEED + rank, K


# ---------------------------------------------------------------------------
# reference arm: the oracle port on host cores
# ---------------------------------------------------------------------------

def cpu_reference(sys_, K, seed, steps, warmup, threads, min_seconds=0.0):
    """Time the C restatement of pflow over K scenarios per step.

    Each scenario: mutate loads / PV P / outage coefficients, run the
    reference's residual (pool + join) and Jacobian (slots + CSC gather)
    algorithm, restore.  Outputs stay in
    each thread's workspace as in pflow (the workspace owns the CSC).
    """
    import oracle  # reference arm / cpu_baseline only

    o = oracle.Oracle(sys_)
    y, pq_p, pq_q, pv_p, outage = blocked_inputs(sys_, K, seed)
    best = None
    for wf in (5, 1):  # pflow's fastest CPU workflows at 70k
        t0 = time.perf_counter()
        o.eval_scenarios(K, y, pq_p, pq_q, pv_p, outage, want_g=False, want_j=False, wf=wf,
                         nthreads=threads)
        dt = time.perf_counter() - t0
        if best is None or dt < best[1]:
            best = (wf, dt)
    wf = best[0]
    for _ in range(max(0, warmup - 1)):
        o.eval_scenarios(K, y, pq_p, pq_q, pv_p, outage, want_g=False, want_j=False, wf=wf,
                         nthreads=threads)
    times = []
    t_start = time.perf_counter()
    while len(times) < steps or (time.perf_counter() - t_start) < min_seconds:
        t0 = time.perf_counter()
        o.eval_scenarios(K, y, pq_p, pq_q, pv_p, outage, want_g=False, want_j=False, wf=wf,
                         nthreads=threads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    return {"value": K * len(times) / total, "ms_per_step": 1e3 * total / len(times),
            "wf": wf, "steps": len(times), "threads": threads, "nnz": int(o.nnz)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sys_ = build_case(args.workload)
    K = WORKLOADS[args.workload][1]
    threads = os.cpu_count() or 1
    r = cpu_reference(sys_, K, SEED, args.steps, args.warmup, threads)
    scaling = args.scaling or WORKLOADS[args.workload][2]
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": "evals/s",
        "n_gpus": args.gpus, "steps": r["steps"], "warmup": args.warmup,
        "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, sys_, r["nnz"]),
        "run": {"parallelism": f"{threads} host threads, one scenario per thread at a time "
                               "(CPU only; the N GPUs are unused)"},
        "cpu_baseline": {"value": r["value"], "unit": "evals/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{r['steps']} steps x {K} scenarios, pflow wf{r['wf']} "
                                   "restated in C (oracle/), workspace outputs"},
        "e2e": {"value": r["value"], "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def traffic_of(workload: str):
    """ncu DRAM bytes per launch of the product kernel, only when
    profiles/traffic.json was captured from this very kernel source."""
    from paper_2011_11880_b200.build import source_hash

    tfile = ROOT / "profiles" / "traffic.json"
    if not tfile.exists():
        return None
    ent = json.loads(tfile.read_text()).get(workload, {})
    return ent.get("bytes") if ent.get("source_hash") == source_hash() else None


def batched_leg(args, workload: str, scaling: str, dev, rank: int, world: int,
                e2e: bool) -> dict | None:
    """One scenario-batched workload on this rank's shard.  Returns rank 0's
    result dict (None elsewhere).  Every rank joins every collective."""
    import torch
    import torch.distributed as dist

    from paper_2011_11880_b200.batched import NormExchange, check_same_pattern, max_shard
    from paper_2011_11880_b200.plan import Plan, launch_count

    K_total, lo, hi, seed, K_gen = rank_workload(workload, scaling, rank, world)
    K = hi - lo
    kmax = max_shard(K_gen, world) if scaling == "strong" else K
    t0 = time.perf_counter()
    sys_ = build_case(workload)
    t1 = time.perf_counter()
    plan = Plan(sys_, device=dev)
    torch.cuda.synchronize(dev)
    if world > 1:   # every rank built the same pattern
        check_same_pattern(*plan.pattern_csr(), device=dev)
    setup_s = {"build_system_s": t1 - t0, "plan_create_s": time.perf_counter() - t1,
               "note": "synthetic case generation + build_system (host), then pf_plan_create: "
                       "upload, device symbolic pattern, staging records"}
    per_scen, static, bytes_launch = algorithmic_bytes(sys_, plan.nnz, K)
    y, pq_p, pq_q, pv_p, outage = blocked_inputs(sys_, K_gen, seed, lo, hi)
    t = lambda a, dt=torch.float64: torch.from_numpy(a).to(dev, dt)
    d_y, d_pqp, d_pqq, d_pvp = t(y), t(pq_p), t(pq_q), t(pv_p)
    d_out = torch.from_numpy(outage).to(dev)
    d_g = plan.empty(plan.n_var, K)
    d_j = plan.empty(plan.nnz, K)
    # double-buffered norms: the all-gather of step i (NCCL, on its own
    # stream) overlaps step i+1's evaluation (batched.NormExchange)
    nx = NormExchange(kmax, dev)
    stream = torch.cuda.current_stream(dev)

    def step(i, ev=None):
        nrm = nx.buffer(i)            # waits (stream-side) for gather i-2
        if ev is not None:
            ev[0].record(stream)
        plan.eval_batched(K, d_y, d_pqp, d_pqq, d_pvp, d_out, d_g, d_j, nrm, stream=stream)
        if ev is not None:
            ev[1].record(stream)
        nx.start(i)

    for i in range(args.warmup):
        step(i)
    nx.drain()
    torch.cuda.synchronize(dev)

    clocks = Clocks(dev.index)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    l0 = launch_count()
    start.record(stream)
    for i in range(args.steps):
        step(i, ev[i])
    nx.drain()                        # the last norms are gathered inside the timed region
    end.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = launch_count() - l0
    clk = clocks.stop()
    ms_total = start.elapsed_time(end)
    kern_ms = [a.elapsed_time(b) for a, b in ev]
    ms_t = torch.tensor([ms_total, statistics.mean(kern_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_total, kern_max = float(ms_t[0]), float(ms_t[1])
    kern_avg = statistics.mean(kern_ms)
    value = K_total * args.steps / (ms_total / 1e3)
    peak, peak_kind = peaks()
    achieved = bytes_launch / (kern_avg / 1e3) / 1e9
    last = args.steps - 1
    assert torch.isfinite(nx.local[last & 1][:K]).all()
    assert torch.equal(nx.result(last)[rank, :K], nx.local[last & 1][:K])   # arrived intact

    out = None
    if rank == 0:
        out = {
            "value": value, "ms_per_step": ms_total / args.steps, "scaling": scaling,
            "workload": workload_desc(workload), "scenarios_total": K_total,
            "scenarios_per_gpu": K, "gpu_launches": launches, "clocks": clk,
            "n_var": plan.n_var, "nnz": plan.nnz, "max_bus_degree": plan.max_degree,
            "config": workload_config(workload, sys_, plan.nnz),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic_of(workload),
                         "frac_of_nominal_8tbs": achieved / 8000.0,
                         "peak_kind": peak_kind, "algorithmic_bytes_per_launch": bytes_launch,
                         "bytes_per_scenario": per_scen, "static_bytes": static,
                         "kernel_ms": kern_avg, "kernel_ms_max_over_ranks": kern_max,
                         "kernel": "k_eval_staged<RES|JAC|NORM>"},
            "l2": f"inputs+outputs per launch {bytes_launch / 1e9:.2f} GB > 126 MB L2 "
                  "(no flush needed)" if bytes_launch > 126e6 else
                  f"inputs+outputs per launch {bytes_launch / 1e6:.0f} MB",
            "setup": setup_s,
        }
    if not e2e:
        return out

    # ---- e2e through the host-buffer C ABI (pinned host memory) ----
    # (an error here is reported in the line; every rank still joins the
    # collectives below)
    del d_y, d_pqp, d_pqq, d_pvp, d_out
    e2e_steps = max(2, min(args.steps, 5))
    e2e_err = None
    bi = bo = 0
    try:
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
        h_y, h_pqp, h_pqq, h_pvp, h_out = pin(y), pin(pq_p), pin(pq_q), pin(pv_p), pin(outage)
        h_g = torch.empty(d_g.numel(), dtype=torch.float64).pin_memory().numpy()
        h_j = torch.empty(d_j.numel(), dtype=torch.float64).pin_memory().numpy()
        h_n = torch.empty(K, dtype=torch.float64).pin_memory().numpy()
        bi = h_y.nbytes + h_pqp.nbytes + h_pqq.nbytes + h_pvp.nbytes + h_out.nbytes
        bo = h_g.nbytes + h_j.nbytes + h_n.nbytes

        def host_step():
            plan.eval_batched_host(K, h_y, h_pqp, h_pqq, h_pvp, h_out, h_g, h_j, h_n,
                                   blocks_per_stage=1, n_streams=8)

        host_step()
    except Exception as e:  # noqa: BLE001
        e2e_err = repr(e)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    if e2e_err is None:
        try:
            for _ in range(e2e_steps):
                host_step()
        except Exception as e:  # noqa: BLE001
            e2e_err = repr(e)
    elapsed = time.perf_counter() - t0 if e2e_err is None else float("inf")
    e2e_s = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = K_total * e2e_steps / float(e2e_s[0])

    # ---- e2e, device-resident workflow (the north star's: g and J stay on
    # the GPU for a device solver; only the per-scenario norms come back) ----
    dr_err = None
    try:
        pt = lambda a: torch.from_numpy(a).pin_memory()
        hp = [pt(a) for a in (y, pq_p, pq_q, pv_p)]
        hp_out = pt(outage)
        dp = [torch.empty_like(a, device=dev) for a in hp]
        dp_out = torch.empty_like(hp_out, device=dev)
        hn = torch.empty(world * kmax, dtype=torch.float64).pin_memory()

        def dr_step():
            for a, b in zip(dp, hp):
                a.copy_(b, non_blocking=True)
            dp_out.copy_(hp_out, non_blocking=True)
            nrm = nx.buffer(0)
            plan.eval_batched(K, dp[0], dp[1], dp[2], dp[3], dp_out, d_g, d_j, nrm,
                              stream=stream)
            nx.start(0)
            hn.copy_(nx.result(0).reshape(-1), non_blocking=True)
            torch.cuda.synchronize(dev)

        dr_step()
    except Exception as e:  # noqa: BLE001
        dr_err = repr(e)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    if dr_err is None:
        try:
            for _ in range(e2e_steps):
                dr_step()
        except Exception as e:  # noqa: BLE001
            dr_err = repr(e)
    elapsed = time.perf_counter() - t0 if dr_err is None else float("inf")
    dr_s = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(dr_s, op=dist.ReduceOp.MAX)
    dr_value = K_total * e2e_steps / float(dr_s[0])
    if rank == 0:
        out["e2e"] = ({"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": bi,
                       "d2h_bytes_per_step": bo,
                       "api": "pf_eval_batched_host (pinned host buffers)", "steps": e2e_steps}
                      if e2e_err is None and e2e_value > 0 else
                      {"value": None, "unit": "evals/s",
                       "error": e2e_err or "failed on a peer rank"})
        out["e2e_device_resident"] = (
            {"value": dr_value, "unit": "evals/s", "h2d_bytes_per_step": bi,
             "d2h_bytes_per_step": 8 * world * kmax,
             "api": "pinned inputs -> device, pf_eval_batched, norms -> host; g and J stay "
                    "in HBM for a device solver", "steps": e2e_steps}
            if dr_err is None and dr_value > 0 else
            {"value": None, "error": dr_err or "failed on a peer rank"})
    return out


def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    scaling = args.scaling or WORKLOADS[args.workload][2]
    head = batched_leg(args, args.workload, scaling, dev, rank, world, e2e=True)
    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": head["config"],
            "run": {
                "scenarios_per_gpu": head["scenarios_per_gpu"],
                "parallelism": f"scenario-sharded x{world} ({scaling} scaling)"
                               + (", NCCL all-gather of norms overlapped with the next step"
                                  if world > 1 else ""),
                "l2": head["l2"],
            },
            "roofline": head["roofline"], "e2e": head["e2e"],
            "e2e_device_resident": head["e2e_device_resident"],
            "gpu_launches": head["gpu_launches"], "setup": head["setup"],
            "clocks": head["clocks"],
        }

    # optional legs: a failure there is reported in the line, never loses it
    if args.workload == "config3" and not args.no_config4:
        try:
            c4 = batched_leg(args, "config4", WORKLOADS["config4"][2], dev, rank, world,
                             e2e=False)
        except Exception as e:  # noqa: BLE001
            c4 = {"error": repr(e)}
        if rank == 0:
            line["config4"] = c4
            if world == 1 and not args.no_cpu and "error" not in c4:
                try:
                    threads = os.cpu_count() or 1
                    s4 = build_case("config4")
                    r = cpu_reference(s4, 64, SEED, 1, 1, threads, min_seconds=args.cpu_seconds)
                    c4["cpu_baseline"] = {
                        "value": r["value"], "unit": "evals/s", "cores": threads, "kind": "port",
                        "sample": f"{r['steps']} x 64 config4 scenarios, pflow wf{r['wf']} "
                                  "restated in C (oracle/), one scenario per thread"}
                except Exception as e:  # noqa: BLE001
                    c4["cpu_baseline"] = {"error": repr(e)}
    if rank == 0 and world == 1 and not args.no_single and args.workload == "config3":
        try:
            line["single_grid"] = single_grid(dev, steps=max(20, args.steps),
                                              cpu=not args.no_cpu)
        except Exception as e:  # noqa: BLE001
            line["single_grid"] = {"error": repr(e)}
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        try:
            sys_ = build_case(args.workload)
            K = WORKLOADS[args.workload][1]
            r = cpu_reference(sys_, K, SEED, 1, 1, threads, min_seconds=args.cpu_seconds)
            line["cpu_baseline"] = {
                "value": r["value"], "unit": "evals/s", "cores": threads, "kind": "port",
                "sample": f"{r['steps']} x {K} {args.workload} scenarios, pflow wf{r['wf']} "
                          "restated in C (oracle/), one scenario per thread, workspace outputs"}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"error": repr(e)}
        # the live reference beside the port (when pflow travelled here)
        try:
            from oracle import live  # cpu_baseline legs only

            from paper_2011_11880_b200 import synth

            pflow, why = live.import_pflow()
            cfg = WORKLOADS[args.workload][0]
            line["cpu_baseline_pflow"] = (
                live.time_batched(pflow, synth.config_case(cfg, seed=cfg),
                                  WORKLOADS[args.workload][1], SEED, threads, 4 * threads)
                if pflow is not None else {"unavailable": why})
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline_pflow"] = {"error": repr(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def single_grid(dev, steps: int, cpu: bool = True) -> dict:
    """Single grids, one f+J+norm per evaluation (BASELINE configs 0-2).

    cold: L2 flushed (256 MB write) before every evaluation, CUDA events
    around the one launch.  graph100: BASELINE config-1 style - 100
    evaluations on 100 perturbed states replayed as one CUDA graph (topology
    warm in L2, no host launch overhead), L2 flushed before each replay.
    batch100: the same 100 independent states in one scenario-batched launch
    (the evaluations do not depend on each other, so they need not be
    sequential); L2 flushed before each launch.
    The top-level keys are config 2 (the metric's 70k-bus grid); configs 0
    and 1 are listed under "smaller".
    """
    out = _single_grid_config(dev, 2, steps, cpu)
    out["smaller"] = [_single_grid_config(dev, c, steps, cpu) for c in (0, 1)]
    return out


def single_cpu_baseline(sys_, y, min_seconds: float = 0.5) -> dict:
    """The reference's fastest CPU workflow for one grid:
    pflow's f+J restated in C (oracle/), wf1 and wf5 on one thread and wf3 on
    every host thread; the fastest one's median over >= min_seconds."""
    import oracle  # cpu_baseline leg only

    o = oracle.Oracle(sys_)
    threads = os.cpu_count() or 1
    runs = {1: lambda: (o.residual(y, 1), o.jacobian(y, 1)),
            5: lambda: (o.residual(y, 5), o.jacobian(y, 5)),
            3: lambda: o.eval_threaded(y, threads)}
    best = None
    for wf, fn in runs.items():
        fn()
        times, t_start = [], time.perf_counter()
        while len(times) < 3 or time.perf_counter() - t_start < min_seconds:
            t0 = time.perf_counter()
            fn()
            times.append(time.perf_counter() - t0)
        med = statistics.median(times)
        if best is None or med < best[1]:
            best = (wf, med)
    wf, med = best
    return {"value": 1.0 / med, "unit": "evals/s", "us_per_eval": med * 1e6,
            "cores": threads if wf == 3 else 1, "kind": "port", "wf": wf,
            "sample": "fastest of pflow wf1 / wf5 (one thread) and wf3 (all host threads), "
                      "restated in C (oracle/), median per f+J"}


def _single_grid_config(dev, cfg: int, steps: int, cpu: bool = True) -> dict:
    import torch

    from paper_2011_11880_b200 import synth
    from paper_2011_11880_b200.plan import Plan
    from paper_2011_11880_b200.system_model import build_system, random_state

    raw = synth.config_case(cfg, seed=cfg)
    s = build_system(raw)
    plan = Plan(s, device=dev)
    _, static, _ = algorithmic_bytes(s, plan.nnz, 1)
    # single grid: base loads read from the plan's device parameters
    bytes_eval = (8 * s.n_var + 8 * s.n_var + 8 * plan.nnz + 8 + static
                  + 16 * len(s.pq) + 8 * len(s.pv))
    y0 = random_state(s, 7)
    ys = torch.as_tensor(synth.perturbed_states(y0, s.n_bus, 100, seed=8), device=dev)
    g, j, n = plan.empty(plan.n_var), plan.empty(plan.nnz), plan.empty(1)
    norms = torch.empty(100, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    st = torch.cuda.Stream(dev)
    with torch.cuda.stream(st):
        for _ in range(5):
            plan.eval(ys[0], g, j, n, stream=st)
        cold = []
        for k in range(steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            plan.eval(ys[k % 100], g, j, n, stream=st)
            b.record(st)
            st.synchronize()
            cold.append(a.elapsed_time(b))
    torch.cuda.synchronize(dev)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        for k in range(100):
            plan.eval(ys[k], g, j, norms[k:k + 1], stream=st)
    rep = []
    with torch.cuda.stream(st):
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            graph.replay()
            b.record(st)
            st.synchronize()
            rep.append(a.elapsed_time(b) / 100)
    # batch100: the same 100 perturbed states are independent evaluations,
    # so the scenario-batched kernel evaluates them in one launch (K = 100,
    # base loads, no outages); L2 flushed before each launch
    from paper_2011_11880_b200.plan import to_blocked
    yb = torch.as_tensor(to_blocked(ys.cpu().numpy()), device=dev)
    gb, jb, nb_ = plan.empty(plan.n_var, 100), plan.empty(plan.nnz, 100), plan.empty(100)
    bat = []
    with torch.cuda.stream(st):
        for k in range(3 + max(steps, 5)):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            plan.eval_batched(100, yb, g=gb, jval=jb, norms=nb_, stream=st)
            b.record(st)
            st.synchronize()
            if k >= 3:
                bat.append(a.elapsed_time(b) / 100)
    torch.cuda.synchronize(dev)
    # drop-in: the reference-facing host API a pflow caller uses (numpy y in,
    # numpy g and the scipy CSC matrix out, pflow/newton.py:70 and :97):
    # ResidualWorkspace.run + JacobianWorkspace.run, each a pf_eval_host call
    from paper_2011_11880_b200.jacobian import JacobianWorkspace
    from paper_2011_11880_b200.residual import ResidualWorkspace

    rws, jws = ResidualWorkspace(s, plan), JacobianWorkspace(s, plan)
    y_h = np.array(y0)
    g_h = np.empty(plan.n_var)
    rws.bind(y_h, g_h)
    drop = []
    for k in range(3 + max(steps, 10)):
        t0 = time.perf_counter()
        rws.run(y_h)
        jws.run(y_h)
        if k >= 3:
            drop.append(time.perf_counter() - t0)
    med_d = statistics.median(drop)
    # the fused pair (JacobianWorkspace(..., residual_ws=rws)): one upload and
    # one launch per Newton iteration, as pflow's newton_solve calls them
    rws_f = ResidualWorkspace(s, plan)
    jws_f = JacobianWorkspace(s, plan, residual_ws=rws_f)
    rws_f.bind(y_h, g_h)
    drop_f = []
    for k in range(3 + max(steps, 10)):
        t0 = time.perf_counter()
        rws_f.run(y_h)
        jws_f.run(y_h)
        if k >= 3:
            drop_f.append(time.perf_counter() - t0)
    med_f = statistics.median(drop_f)
    # per state: y, g, J, norm; the plan's static data once per launch
    bytes_b = 100 * (16 * s.n_var + 8 * plan.nnz + 8) + static + 16 * len(s.pq) + 8 * len(s.pv)
    med_b = statistics.median(bat)
    med_c = statistics.median(cold)
    med_g = statistics.median(rep)
    peak, _ = peaks()
    return {"workload": f"config{cfg}: {s.n_bus} buses, {len(s.lines.bus_h)} branches, "
                        "one f+J+norm per evaluation",
            "cold_us_per_eval": med_c * 1e3, "cold_evals_per_s": 1e3 / med_c,
            "graph100_us_per_eval": med_g * 1e3, "graph100_evals_per_s": 1e3 / med_g,
            "algorithmic_bytes": bytes_eval,
            "cold_frac": bytes_eval / (med_c / 1e3) / 1e9 / peak,
            "graph100_frac": bytes_eval / (med_g / 1e3) / 1e9 / peak,
            "dropin_us_per_eval": med_d * 1e6, "dropin_evals_per_s": 1.0 / med_d,
            "dropin_api": "ResidualWorkspace.run + JacobianWorkspace.run (numpy y, numpy g, "
                          "scipy CSC J; host copies included)",
            "dropin_fused_us_per_eval": med_f * 1e6, "dropin_fused_evals_per_s": 1.0 / med_f,
            "dropin_fused_api": "the same pair fused (JacobianWorkspace(..., residual_ws=rws)): "
                                "one upload of y and one launch for g and J",
            "batch100_us_per_eval": med_b * 1e3, "batch100_evals_per_s": 1e3 / med_b,
            "batch100_frac": bytes_b / (med_b * 100 / 1e3) / 1e9 / peak,
            "batch100_kernel": "k_eval_staged<RES|JAC|NORM> (K = 100 states, one launch)",
            "n_var": plan.n_var, "nnz": plan.nnz, "kernel": "k_eval_single<RES|JAC|NORM>",
            "ctas": plan.single_chunks,
            "cpu_baseline": single_cpu_baseline(s, y0) if cpu else None,
            "cpu_baseline_pflow": single_pflow_baseline(raw, y0) if cpu else None}


def single_pflow_baseline(raw, y0) -> dict | None:
    """The live reference (pflow, Numba) timed beside the C port, when it is
    importable here (baseline/_ref travels to the GPU box)."""
    try:
        from oracle import live  # cpu_baseline legs only

        pflow, why = live.import_pflow()
        if pflow is None:
            return {"unavailable": why}
        return live.time_single_grid(pflow, live.pflow_system(pflow, raw), y0,
                                     os.cpu_count() or 1, min_seconds=0.3)
    except Exception as e:  # noqa: BLE001
        return {"error": repr(e)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-single", action="store_true", help="skip the single-grid leg")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--workload", default="config3", choices=sorted(WORKLOADS))
    ap.add_argument("--scaling", default=None, choices=["strong", "weak"],
                    help="strong: split the workload's K over the ranks (config 3 default); "
                         "weak: K per rank (config 4 default)")
    ap.add_argument("--no-config4", action="store_true", help="skip the config-4 leg")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
