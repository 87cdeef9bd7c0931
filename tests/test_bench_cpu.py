"""bench.py contract pieces that run without a GPU: the reference arm (the
CPU oracle port on host threads) prints one well-formed JSON line."""

import json
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["unit"] == "evals/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["metric"].startswith("f+J evals/s")
    # the config holds workload properties only, computed as the GPU arm does
    # (bench.workload_config); how this arm ran goes in "run"
    sys.path.insert(0, str(ROOT))
    import bench

    sys_ = bench.build_case("config3")
    assert d["config"] == bench.workload_config("config3", sys_, d["config"]["nnz"])
    assert d["config"]["n_var"] == sys_.n_var and d["config"]["scenarios_total"] == 256
    assert "parallelism" in d["run"]


def test_reference_arm_other_ranks_exit_quietly():
    env = {"RANK": "1", "WORLD_SIZE": "2", "PATH": "/usr/bin:/bin"}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode == 0
    assert out.stdout.strip() == ""


def test_rank_workloads_cover_the_batch():
    """Strong scaling (config 3) splits the same K = 256 scenarios over the
    ranks, every rank busy; weak scaling (config 4) gives each rank K = 64 of
    its own.  Both arms print one workload string."""
    sys.path.insert(0, str(ROOT))
    import bench

    for world in (1, 2, 4, 8):
        got = []
        for r in range(world):
            K_total, lo, hi, seed, K_gen = bench.rank_workload("config3", "strong", r, world)
            assert (K_total, seed, K_gen) == (256, bench.SEED, 256) and hi > lo
            got.extend(range(lo, hi))
        assert got == list(range(256))
        seeds = set()
        for r in range(world):
            K_total, lo, hi, seed, K_gen = bench.rank_workload("config4", "weak", r, world)
            assert (K_total, lo, hi, K_gen) == (64 * world, 0, 64, 64)
            seeds.add(seed)
        assert len(seeds) == world
    assert bench.WORKLOADS["config3"][2] == "strong" and bench.WORKLOADS["config4"][2] == "weak"


def test_strong_shard_inputs_are_slices_of_the_n1_workload():
    """Rank r's inputs under strong scaling are exactly columns [lo, hi) of
    the N = 1 batch (same seed), so the sharded run evaluates the same
    scenarios as the single-GPU run."""
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2011_11880_b200 import synth
    from paper_2011_11880_b200.plan import from_blocked
    from paper_2011_11880_b200.system_model import build_system

    s = build_system(synth.synth_case(200, 260, seed=1, pq_frac=0.6, pv_frac=0.2))
    full = bench.blocked_inputs(s, 70, 5)
    parts = [bench.blocked_inputs(s, 70, 5, *bench_shard) for bench_shard in
             [(0, 23), (23, 47), (47, 70)]]
    n = [s.n_var, len(s.pq), len(s.pq), len(s.pv)]
    for q in range(4):
        F = from_blocked(full[q], 70, n[q])
        P = np.concatenate([from_blocked(p[q], p[4].size, n[q]) for p in parts])
        assert np.array_equal(F, P)
    assert np.array_equal(full[4], np.concatenate([p[4] for p in parts]))
