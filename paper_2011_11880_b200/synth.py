"""Seeded synthetic grids, states and scenarios for BASELINE.json configs 0-4.

The paper's ACTIVSg70k case is not available here, so these grids stand in
for it with the shapes BASELINE.json names:

* topology: a random spanning tree (bus i > 0 attaches to a uniform earlier
  bus) plus uniformly random extra edges without self-loops (parallel edges
  allowed); branch order is shuffled;
* r ~ U(0.001, 0.05), x ~ U(0.01, 0.3), b ~ U(0, 0.1); tap 1 on 85% of
  branches, U(0.95, 1.05) on the rest; phase shift 0 unless ``shift_frac``;
* slack at bus 0 (V = 1, theta = 0); PV gens at a fraction (or count) of
  the other buses with P ~ U(0.2, 2), Vset ~ U(0.98, 1.05); PQ loads on a
  fraction (or count) of buses with P ~ U(0, 1), Q ~ U(0, 0.5);
* ``base_mva = 1`` so per-unit conversion is exact;
* optional shunts / phase shifters / hubs / out-of-service rows exercise
  the remaining code paths in parity tests.

Scenarios (config 3): per-device load scale U(0.8, 1.2) applied to P and Q,
per-device PV scale U(0.5, 1.5), one outaged branch per scenario.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .case import RawCase, make_case

CONFIGS = {
    0: dict(n_bus=2_000, n_branch=2_500, pq_frac=0.60, pv_frac=0.15),
    1: dict(n_bus=10_000, n_branch=12_500, pq_frac=0.60, pv_frac=0.15),
    2: dict(n_bus=70_000, n_branch=88_000, n_pq=45_000, n_pv=6_000),
    3: dict(n_bus=70_000, n_branch=88_000, n_pq=45_000, n_pv=6_000),
    4: dict(n_bus=200_000, n_branch=250_000, pq_frac=0.60, pv_frac=0.15,
            hub_frac=0.01, hub_degree=50),
}


def synth_case(n_bus: int, n_branch: int, seed: int = 0, *,
               pq_frac: float | None = None, pv_frac: float | None = None,
               n_pq: int | None = None, n_pv: int | None = None,
               shunt_frac: float = 0.0, shift_frac: float = 0.0,
               hub_frac: float = 0.0, hub_degree: int = 50,
               out_of_service_frac: float = 0.0, name: str = "") -> RawCase:
    """Random connected grid as a columnar RawCase (base_mva = 1)."""
    if n_bus < 1:
        raise ValueError("n_bus must be >= 1")
    if n_branch < n_bus - 1:
        raise ValueError("n_branch must be >= n_bus - 1 (spanning tree)")
    rng = np.random.default_rng(seed)
    nb = n_bus
    # spanning tree: bus i attaches to a uniform earlier bus
    child = np.arange(1, nb)
    parent = np.floor(rng.random(nb - 1) * child).astype(np.int64)
    n_extra = n_branch - (nb - 1)
    eh = rng.integers(0, nb, n_extra) if nb > 1 else np.zeros(0, np.int64)
    ek = rng.integers(0, nb, n_extra) if nb > 1 else np.zeros(0, np.int64)
    bad = eh == ek
    while bad.any():
        ek[bad] = rng.integers(0, nb, int(bad.sum()))
        bad = eh == ek
    fb = np.concatenate([parent, eh])
    tb = np.concatenate([child, ek])
    if hub_frac > 0.0 and nb > hub_degree + 1:
        n_hub = max(1, int(round(hub_frac * nb)))
        hubs = rng.choice(nb, n_hub, replace=False)
        deg = np.bincount(np.concatenate([fb, tb]), minlength=nb)
        hh, hk = [], []
        for h in hubs:
            need = max(0, hub_degree - int(deg[h]))
            if need:
                other = rng.integers(0, nb - 1, need)
                other = other + (other >= h)  # never h itself
                hh.append(np.full(need, h, np.int64))
                hk.append(other)
        if hh:
            fb = np.concatenate([fb, *hh])
            tb = np.concatenate([tb, *hk])
    # random orientation, then shuffle branch order
    flip = rng.random(fb.size) < 0.5
    fb, tb = np.where(flip, tb, fb), np.where(flip, fb, tb)
    perm = rng.permutation(fb.size)
    fb, tb = fb[perm], tb[perm]
    m = fb.size

    r = rng.uniform(0.001, 0.05, m)
    x = rng.uniform(0.01, 0.3, m)
    bc = rng.uniform(0.0, 0.1, m)
    ratio = np.where(rng.random(m) < 0.85, 1.0, rng.uniform(0.95, 1.05, m))
    angle = np.zeros(m)
    if shift_frac > 0.0:
        s = rng.random(m) < shift_frac
        angle[s] = rng.uniform(-10.0, 10.0, int(s.sum()))
    br_status = np.ones(m, np.int64)
    if out_of_service_frac > 0.0:
        br_status[rng.random(m) < out_of_service_frac] = 0

    bus_type = np.ones(nb, np.int64)
    bus_type[0] = 3
    others = np.arange(1, nb)
    if n_pv is None:
        n_pv = int(round((pv_frac or 0.0) * (nb - 1)))
    pv_buses = np.sort(rng.choice(others, min(n_pv, others.size), replace=False)) \
        if others.size else np.zeros(0, np.int64)
    bus_type[pv_buses] = 2
    if n_pq is None:
        n_pq = int(round((pq_frac or 0.0) * nb))
    load_buses = rng.choice(nb, min(n_pq, nb), replace=False)
    pd = np.zeros(nb)
    qd = np.zeros(nb)
    pd[load_buses] = rng.uniform(0.0, 1.0, load_buses.size)
    qd[load_buses] = rng.uniform(0.0, 0.5, load_buses.size)
    gs = np.zeros(nb)
    bs = np.zeros(nb)
    if shunt_frac > 0.0:
        sh = rng.random(nb) < shunt_frac
        gs[sh] = rng.uniform(0.0, 0.05, int(sh.sum()))
        bs[sh] = rng.uniform(-0.2, 0.3, int(sh.sum()))

    # gens: slack first, then one per PV bus
    gen_bus = np.concatenate([[0], pv_buses]).astype(np.int64)
    ng = gen_bus.size
    pg = np.concatenate([[0.0], rng.uniform(0.2, 2.0, pv_buses.size)])
    vg = np.concatenate([[1.0], rng.uniform(0.98, 1.05, pv_buses.size)])
    gen_status = np.ones(ng, np.int64)
    if out_of_service_frac > 0.0 and ng > 1:
        gen_status[1:][rng.random(ng - 1) < out_of_service_frac] = 0

    bus_id = np.arange(1, nb + 1, dtype=np.int64)
    bus = dict(bus_id=bus_id, bus_type=bus_type, pd=pd, qd=qd, gs=gs, bs=bs,
               vm=np.ones(nb), va=np.zeros(nb), base_kv=np.full(nb, 230.0))
    gen = dict(gen_bus=gen_bus + 1, pg=pg, qg=np.zeros(ng), qmax=np.full(ng, 9999.0),
               qmin=np.full(ng, -9999.0), vg=vg, gen_status=gen_status)
    branch = dict(from_bus=fb + 1, to_bus=tb + 1, r=r, x=x, b=bc, ratio=ratio,
                  angle=angle, br_status=br_status)
    return make_case(1.0, bus, gen, branch, name=name or f"synth{nb}")


def config_case(cfg: int, seed: int = 0) -> RawCase:
    """The grid of BASELINE.json config ``cfg`` (0..4)."""
    return synth_case(seed=seed, name=f"config{cfg}", **CONFIGS[cfg])


def perturbed_states(y0: np.ndarray, n_bus: int, count: int, seed: int) -> np.ndarray:
    """Config 1: ``count`` states y0 + (dtheta ~ N(0,0.01), dV ~ N(0,0.01)).

    Returns shape [count, n_var]."""
    rng = np.random.default_rng(seed)
    ys = np.repeat(y0[None, :], count, axis=0)
    ys[:, :n_bus] += rng.normal(0.0, 0.01, (count, n_bus))
    ys[:, n_bus:2 * n_bus] += rng.normal(0.0, 0.01, (count, n_bus))
    return ys


@dataclass
class ScenarioBatch:
    """K scenarios over one topology, scenario-minor (``[entry, K]``) arrays.

    ``y``: [n_var, K] states; ``pq_p``/``pq_q``: [n_pq, K] loads;
    ``pv_p``: [n_pv, K] PV schedules; ``outage``: [K] int32 branch index
    (-1 = none).  Element (e, s) lives at ``e * K + s``.
    """

    y: np.ndarray
    pq_p: np.ndarray
    pq_q: np.ndarray
    pv_p: np.ndarray
    outage: np.ndarray

    @property
    def K(self) -> int:
        return int(self.outage.shape[0])

    def scenario(self, s: int):
        """(y, pq_p, pq_q, pv_p, outage) of scenario s as contiguous arrays."""
        return (np.ascontiguousarray(self.y[:, s]), np.ascontiguousarray(self.pq_p[:, s]),
                np.ascontiguousarray(self.pq_q[:, s]), np.ascontiguousarray(self.pv_p[:, s]),
                int(self.outage[s]))


def make_scenarios(sys, K: int, seed: int, *, outages: bool = True) -> ScenarioBatch:
    """Config-3 scenarios: per-device scale factors and one outage each.

    Each scenario also gets its own random state.
    """
    rng = np.random.default_rng(seed)
    nb = sys.n_bus
    n_var = sys.n_var
    y = np.empty((n_var, K))
    y[:nb] = rng.normal(0.0, 0.2, (nb, K))
    y[nb:2 * nb] = rng.uniform(0.95, 1.05, (nb, K))
    y[2 * nb:] = rng.uniform(-0.5, 0.5, (n_var - 2 * nb, K))
    ls = rng.uniform(0.8, 1.2, (len(sys.pq), K))
    pq_p = sys.pq.p0[:, None] * ls
    pq_q = sys.pq.q0[:, None] * ls
    pv_p = sys.pv.p0[:, None] * rng.uniform(0.5, 1.5, (len(sys.pv), K))
    L = len(sys.lines)
    if outages and L:
        outage = rng.integers(0, L, K).astype(np.int32)
    else:
        outage = np.full(K, -1, np.int32)
    return ScenarioBatch(y=y, pq_p=np.ascontiguousarray(pq_p), pq_q=np.ascontiguousarray(pq_q),
                         pv_p=np.ascontiguousarray(pv_p), outage=outage)
