"""Scenario-batched evaluation and its multi-GPU sharding.

K contingency / renewable scenarios share one topology (one ``Plan``);
each scenario has its own state y, PQ loads, PV schedules and an outaged
branch.  Arrays use the PF_LANES-blocked layout of include/pfgpu.h so that a
warp's 32 lanes are 32 scenarios of the same bus: every state load and every
residual/Jacobian store is one coalesced 256-byte transaction.

The reference has no batched mode; its equivalent mutates the
PowerSystem arrays per scenario and re-runs workflow 1.  Scenarios are
independent, so multi-GPU runs shard them by contiguous blocks across ranks
(one process per GPU); the only exchange is the all-gather of per-scenario
infinity norms (``gather_norms``, NCCL over NVLink).
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
            self.outage[: self.K].copy_(torch.from_numpy(np.asarray(batch.outage, np.int32)))

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
    """Contiguous scenario range [lo, hi) of ``rank``, aligned to PF_LANES
    blocks so every rank's buffers start on a block boundary."""
    nb = n_blocks(K_total)
    lo_b = (nb * rank) // world
    hi_b = (nb * (rank + 1)) // world
    return min(lo_b * PF_LANES, K_total), min(hi_b * PF_LANES, K_total)


def gather_norms(norms_local, K_local_max: int, group=None):
    """All-gather per-scenario infinity norms from every rank.

    ``norms_local``: CUDA float64 tensor of this rank's norms (padded to
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
