"""Scenario-batched evaluation and its multi-GPU sharding.

K contingency / renewable scenarios share one topology (one ``Plan``);
each scenario has its own state y, PQ loads, PV schedules and an outaged
branch.  Arrays use the PF_LANES-blocked layout of include/pfgpu.h so that a
warp's 32 lanes are 32 scenarios of the same bus: every state load and every
residual/Jacobian store is one coalesced 256-byte transaction.

The reference has no batched mode; its equivalent mutates the
PowerSystem arrays per scenario and re-runs workflow 1.  Scenarios are
independent, so multi-GPU runs shard them in contiguous, even ranges across
ranks (one process per GPU, ``shard``); the only exchange is the all-gather
of per-scenario infinity norms (``NormExchange``, NCCL over NVLink,
overlapped with the next evaluation).
"""

from __future__ import annotations

import numpy as np

from .plan import PF_LANES, Plan, from_blocked, n_blocks, to_blocked


class ScenarioBuffers:
    """Device buffers for K scenarios in the blocked layout."""

    def __init__(self, plan: Plan, K: int, *, loads: bool = True, outages: bool = True,
                 residual: bool = True, jacobian: bool = True):
        import torch

        self.plan, self.K = plan, int(K)
        e = plan.empty
        self.y = e(plan.n_var, K)
        self.pq_p = e(plan.n_pq, K) if loads else None
        self.pq_q = e(plan.n_pq, K) if loads else None
        self.pv_p = e(plan.n_pv, K) if loads else None
        self.outage = (torch.full((max(K, 1),), -1, dtype=torch.int32, device=plan.device)
                       if outages else None)
        self.g = e(plan.n_var, K) if residual else None
        self.jval = e(plan.nnz, K) if jacobian else None
        self.norms = e(K)

    def upload(self, batch) -> None:
        """Copy a ``synth.ScenarioBatch`` ([entry, K] arrays) into the buffers."""
        import torch

        def put(dst, a):
            if dst is None or a is None:
                return
            flat = to_blocked(np.ascontiguousarray(np.asarray(a).T))
            dst[: flat.size].copy_(torch.from_numpy(flat))

        put(self.y, batch.y)
        put(self.pq_p, batch.pq_p)
        put(self.pq_q, batch.pq_q)
        put(self.pv_p, batch.pv_p)
        if self.outage is not None:
            out = np.asarray(batch.outage, np.int32)
            if out.size != self.K:
                raise ValueError(f"outage has {out.size} entries, expected {self.K}")
            if out.size and (out.min() < -1 or out.max() >= self.plan.n_line):
                raise ValueError(f"outage indices must lie in [-1, {self.plan.n_line})")
            self.outage[: self.K].copy_(torch.from_numpy(out))

    def evaluate(self, stream=None) -> None:
        self.plan.eval_batched(self.K, self.y, self.pq_p, self.pq_q, self.pv_p, self.outage,
                               self.g, self.jval, self.norms, stream=stream)

    def residual(self, s: int | None = None) -> np.ndarray:
        """g as [K, n_var] (or one scenario) on the host."""
        g = from_blocked(self.g[: n_blocks(self.K) * PF_LANES * self.plan.n_var].cpu().numpy(),
                         self.K, self.plan.n_var)
        return g if s is None else g[s]

    def jacobian_csr(self, s: int | None = None) -> np.ndarray:
        j = from_blocked(self.jval[: n_blocks(self.K) * PF_LANES * self.plan.nnz].cpu().numpy(),
                         self.K, self.plan.nnz)
        return j if s is None else j[s]


def shard(K_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous scenario range [lo, hi) of ``rank``: an even split, so no
    rank idles while K_total >= world (sizes differ by at most one).  Each
    rank pads its own buffers to whole PF_LANES blocks (``Plan.empty``), so
    a shard need not start on a block boundary of the global batch."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world of {world}")
    return (K_total * rank) // world, (K_total * (rank + 1)) // world


def max_shard(K_total: int, world: int) -> int:
    """Largest shard: the per-rank length of the padded norm all-gather."""
    return -(-K_total // world) if world else 0


class NormExchange:
    """All-gather of per-scenario infinity norms, double-buffered so it
    overlaps the next evaluation (SURVEY.md §7 hard part 6).

    Step i writes its norms into ``buffer(i)`` (buffer i & 1), then
    ``start(i)`` issues an asynchronous all-gather of it.  On NCCL the
    collective runs on the process group's own stream after the current
    stream's work (the evaluation), so the evaluation of step i + 1 proceeds
    while it runs; ``buffer(i + 2)`` makes the current stream wait (on the
    device, no host sync) for gather i before that buffer is written again.
    ``result(i)`` returns the gathered [world, kmax] norms of step i after
    waiting for it.  The only inter-rank traffic of batched mode: kmax fp64
    per rank per step; g and J never leave their GPU.
    """

    def __init__(self, kmax: int, device, group=None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.kmax = int(kmax)
        self.gloo = self.world > 1 and dist.get_backend(group) == "gloo"
        self.local = [torch.zeros(max(self.kmax, 1), dtype=torch.float64, device=device)
                      for _ in range(2)]
        self.gathered = [torch.zeros(self.world * max(self.kmax, 1), dtype=torch.float64,
                                     device=device) for _ in range(2)]
        self.work = [None, None]

    def _wait(self, b: int) -> None:
        if self.work[b] is not None:
            self.work[b].wait()
            self.work[b] = None

    def buffer(self, i: int):
        b = i & 1
        self._wait(b)
        return self.local[b]

    def start(self, i: int) -> None:
        import torch.distributed as dist

        b = i & 1
        if self.world == 1:
            return                     # result() reads the local buffer
        if self.gloo:
            parts = list(self.gathered[b].chunk(self.world))
            self.work[b] = dist.all_gather(parts, self.local[b], group=self.group,
                                           async_op=True)
        else:
            self.work[b] = dist.all_gather_into_tensor(self.gathered[b], self.local[b],
                                                       group=self.group, async_op=True)

    def drain(self) -> None:
        self._wait(0)
        self._wait(1)

    def result(self, i: int):
        b = i & 1
        self._wait(b)
        src = self.local[b] if self.world == 1 else self.gathered[b]
        return src.view(self.world, max(self.kmax, 1))[:, : self.kmax]

    def norms(self, i: int, K_total: int):
        """The K_total norms of step i in global scenario order (strong
        scaling's even split: rank r holds shard(K_total, r, world))."""
        import torch

        g = self.result(i)
        return torch.cat([g[r, : hi - lo] for r, (lo, hi) in
                          enumerate(shard(K_total, r, self.world) for r in range(self.world))])


def pattern_digest(indptr, indices) -> int:
    """63-bit digest of a Jacobian pattern (every rank builds
    the same plan from the same seed, checkable by hash)."""
    import hashlib

    import numpy as np

    h = hashlib.sha256()
    h.update(np.ascontiguousarray(indptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(indices, dtype=np.int64).tobytes())
    return int.from_bytes(h.digest()[:8], "little") >> 1


def check_same_pattern(indptr, indices, device="cpu", group=None) -> int:
    """All ranks must hold the same pattern: min and max of the digest over
    the group are compared; raises RuntimeError on a mismatch.  Returns the
    digest.  (A NCCL group needs ``device`` to be the rank's GPU.)"""
    import torch
    import torch.distributed as dist

    dg = pattern_digest(indptr, indices)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return dg
    lo = torch.tensor([dg], dtype=torch.int64, device=device)
    hi = lo.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    if int(lo) != int(hi):
        raise RuntimeError("ranks built different Jacobian patterns")
    return dg


def gather_norms(norms_local, K_local_max: int, group=None):
    """All-gather per-scenario infinity norms from every rank (blocking).

    ``norms_local``: float64 tensor of this rank's norms (padded to
    ``K_local_max``).  Returns a [world * K_local_max] tensor on every rank.
    Uses ``torch.distributed.all_gather_into_tensor`` (NCCL over NVLink on
    GPUs; gloo in CPU tests).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    src = norms_local[:K_local_max].contiguous()
    out = torch.empty(world * K_local_max, dtype=src.dtype, device=src.device)
    if dist.get_backend(group) == "gloo":
        parts = list(out.chunk(world))
        dist.all_gather(parts, src, group=group)
    else:
        dist.all_gather_into_tensor(out, src, group=group)
    return out
