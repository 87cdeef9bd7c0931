"""Scenario sharding + the overlapped norm all-gather across processes over
gloo (CPU), world sizes 2 and 4.

The GPU run (bench.py, NCCL, one process per GPU) uses the same code:
``batched.shard`` splits the scenarios, every rank evaluates its own shard,
and ``batched.NormExchange`` all-gathers the per-scenario infinity norms
double-buffered over several steps.  Here each rank's "evaluation" is the CPU
oracle on its shard, so the multi-rank host logic is exercised end to end and
compared with one process evaluating every scenario."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2011_11880_b200.batched import (NormExchange, check_same_pattern, max_shard,
                                           pattern_digest, shard)

HERE = Path(__file__).resolve().parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _system():
    from paper_2011_11880_b200 import synth
    from paper_2011_11880_b200.system_model import build_system

    return build_system(synth.synth_case(300, 380, seed=3, pq_frac=0.6, pv_frac=0.15,
                                         shunt_frac=0.1, shift_frac=0.1))


def _inputs(s, K, step, lo, hi):
    """Scenario batch of one step (a different draw per step), rank's slice."""
    from paper_2011_11880_b200 import synth
    from paper_2011_11880_b200.plan import to_blocked

    sb = synth.make_scenarios(s, K, seed=100 + step)
    c = lambda a: to_blocked(np.ascontiguousarray(a[:, lo:hi].T))
    return (c(sb.y), c(sb.pq_p), c(sb.pq_q), c(sb.pv_p),
            np.ascontiguousarray(sb.outage[lo:hi]))


def _worker(rank, world, port, K, steps, q):
    sys.path.insert(0, str(HERE))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle

        s = _system()
        o = oracle.Oracle(s)
        check_same_pattern(*o.pattern_csc())   # every rank built the same pattern
        lo, hi = shard(K, rank, world)
        nx = NormExchange(max_shard(K, world), "cpu")
        got = []
        for i in range(steps):
            buf = nx.buffer(i)
            y, pq_p, pq_q, pv_p, out = _inputs(s, K, i, lo, hi)
            _, _, norms = o.eval_scenarios(hi - lo, y, pq_p, pq_q, pv_p, out,
                                           want_g=False, want_j=False)
            buf[: hi - lo] = torch.from_numpy(norms)
            nx.start(i)            # overlaps the next step's evaluation
            if i >= 1:
                got.append(nx.norms(i - 1, K).numpy().copy())
        nx.drain()
        got.append(nx.norms(steps - 1, K).numpy().copy())
        q.put((rank, hi - lo, np.stack(got)))
    finally:
        dist.destroy_process_group()


def test_shard_even_split_no_idle_rank():
    for K in (1, 31, 32, 64, 70, 100, 256):
        for world in (1, 2, 3, 4, 8):
            got, sizes = [], []
            for r in range(world):
                lo, hi = shard(K, r, world)
                got.extend(range(lo, hi))
                sizes.append(hi - lo)
            assert got == list(range(K))
            assert max(sizes) - min(sizes) <= 1
            assert max(sizes) == max_shard(K, world)
            if K >= world:
                assert min(sizes) >= 1, (K, world)
    # round 1's block-aligned split left 6 of 8 ranks idle here
    assert all(shard(64, r, 8)[1] - shard(64, r, 8)[0] == 8 for r in range(8))
    with pytest.raises(ValueError):
        shard(64, 4, 4)


@pytest.mark.parametrize("world,K", [(2, 64), (4, 64), (4, 70)])
def test_sharded_norm_exchange(world, K):
    import oracle
    from paper_2011_11880_b200.plan import to_blocked

    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank did real work and every rank saw the same gathered norms
    assert sorted(r[1] for r in res) == sorted(shard(K, r, world)[1] - shard(K, r, world)[0]
                                               for r in range(world))
    assert all(r[1] > 0 for r in res)
    for r in res[1:]:
        assert np.array_equal(r[2], res[0][2])
    # ... equal to one process evaluating all K scenarios of each step
    s = _system()
    o = oracle.Oracle(s)
    for i in range(steps):
        y, pq_p, pq_q, pv_p, out = _inputs(s, K, i, 0, K)
        _, _, ref = o.eval_scenarios(K, y, pq_p, pq_q, pv_p, out, want_g=False, want_j=False)
        assert np.array_equal(res[0][2][i], ref), i


def _mismatch_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ptr = np.array([0, 1, 2], np.int32)
        idx = np.array([0, rank], np.int32)     # rank 1 differs
        try:
            check_same_pattern(ptr, idx)
            q.put((rank, "ok"))
        except RuntimeError as e:
            q.put((rank, str(e)))
    finally:
        dist.destroy_process_group()


def test_pattern_check_detects_a_rank_with_another_pattern():
    assert pattern_digest([0, 1], [0]) == pattern_digest(np.array([0, 1]), np.array([0]))
    assert pattern_digest([0, 1], [0]) != pattern_digest([0, 1], [1])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_mismatch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert all("different Jacobian patterns" in v for v in res.values()), res
