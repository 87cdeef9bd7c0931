"""Scenario sharding + norm all-gather with world_size 2 over gloo (CPU).

The GPU run uses the same code with the NCCL backend (one process per GPU);
here the per-rank "evaluation" is the CPU oracle on that rank's scenario
shard, so the host-side multi-rank logic is exercised end to end."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2011_11880_b200.batched import gather_norms, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, K, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from _util import load, system_of
        from paper_2011_11880_b200.plan import to_blocked

        d = load("batch_edge300")
        s = system_of(d)
        lo, hi = shard(K, rank, world)
        o = oracle.Oracle(s)
        Kl = hi - lo
        _, _, norms = o.eval_scenarios(Kl, to_blocked(d["y"][lo:hi]), to_blocked(d["pq_p"][lo:hi]),
                                       to_blocked(d["pq_q"][lo:hi]), to_blocked(d["pv_p"][lo:hi]),
                                       d["outage"][lo:hi], want_g=False, want_j=False)
        kmax = max(shard(K, r, world)[1] - shard(K, r, world)[0] for r in range(world))
        buf = torch.zeros(kmax, dtype=torch.float64)
        buf[:Kl] = torch.from_numpy(norms)
        allv = gather_norms(buf, kmax)
        if rank == 0:
            parts = []
            for r in range(world):
                a, b = shard(K, r, world)
                parts.append(allv[r * kmax: r * kmax + (b - a)].numpy())
            q.put(np.concatenate(parts))
    finally:
        dist.destroy_process_group()


def test_shard_covers_all():
    for K in (1, 31, 32, 64, 100, 256):
        for world in (1, 2, 4, 8):
            got = []
            for r in range(world):
                lo, hi = shard(K, r, world)
                assert lo % 32 == 0
                got.extend(range(lo, hi))
            assert got == list(range(K))


def test_gather_norms_world2():
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from _util import load

    d = load("batch_edge300")
    K = int(d["K"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, K, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(res, d["norms"])
