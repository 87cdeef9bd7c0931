"""Per-unit structure-of-arrays network model with global addressing.

Host-side restatement of pflow/system_model.py (the reference's L1 layer):
the same device groups, the same ``AddressMap`` identity-block layout
(pflow/system_model.py:3-11, 321-332) and the same ``LineGroup`` coefficient
formulas (pflow/system_model.py:101-125, 279-318), evaluated with the same
IEEE operations in the same order so that every coefficient is bit-identical
to the reference's.  This is plan-time setup, not the hot path: the arrays
built here are uploaded once into a device plan (``plan.Plan``).

Variable vector ``y``:  theta (n_bus) | V (n_bus) | Q_g (PV gens, then slack
gens) | P_s (slack);  equation vector ``g``: g_p | g_q | g_V | g_theta.

Sign convention (pflow/system_model.py:23-25): a residual row is
(generation) - (load) - (flows leaving the bus).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .case import RawCase, from_rows, validate_case

StateVector = np.ndarray
ResidualVector = np.ndarray

_IDX = np.int32


@dataclass(frozen=True)
class BusGroup:
    ids: np.ndarray
    bus_type: np.ndarray

    def __len__(self) -> int:
        return self.ids.shape[0]


@dataclass(frozen=True)
class PqGroup:
    """Fixed-power injections: bus loads, then gens at PQ buses (negated)."""

    bus: np.ndarray
    p0: np.ndarray
    q0: np.ndarray

    def __len__(self) -> int:
        return self.bus.shape[0]


@dataclass(frozen=True)
class PvGroup:
    bus: np.ndarray
    p0: np.ndarray
    v0: np.ndarray
    qg: np.ndarray

    def __len__(self) -> int:
        return self.bus.shape[0]


@dataclass(frozen=True)
class SlackGroup:
    bus: np.ndarray
    v0: np.ndarray
    theta0: np.ndarray
    qg: np.ndarray
    ps: np.ndarray

    def __len__(self) -> int:
        return self.bus.shape[0]


@dataclass(frozen=True)
class ShuntGroup:
    bus: np.ndarray
    g: np.ndarray
    b: np.ndarray

    def __len__(self) -> int:
        return self.bus.shape[0]


@dataclass(frozen=True)
class LineGroup:
    """Pi-model branches (pflow/system_model.py:101-144).

    gl, bl   = (g cos phi - b sin phi)/m, (b cos phi + g sin phi)/m
    gl2, bl2 = (g cos phi + b sin phi)/m, (b cos phi - g sin phi)/m
    g_self_h, b_self_h = g/m^2, (b + b_c/2)/m^2 ;  g_self_k, b_self_k = g, b + b_c/2
    ``gl2``/``bl2`` alias ``gl``/``bl`` when no branch has a phase shift.
    """

    bus_h: np.ndarray
    bus_k: np.ndarray
    gl: np.ndarray
    bl: np.ndarray
    gl2: np.ndarray
    bl2: np.ndarray
    g_self_h: np.ndarray
    b_self_h: np.ndarray
    g_self_k: np.ndarray
    b_self_k: np.ndarray
    ph: np.ndarray = field(repr=False, default=None)
    pk: np.ndarray = field(repr=False, default=None)
    qh: np.ndarray = field(repr=False, default=None)
    qk: np.ndarray = field(repr=False, default=None)

    def __len__(self) -> int:
        return self.bus_h.shape[0]

    @property
    def has_shift(self) -> bool:
        return self.gl2 is not self.gl


@dataclass(frozen=True)
class AddressMap:
    theta_of_bus: np.ndarray
    v_of_bus: np.ndarray
    qg_of_gen: np.ndarray
    ps_of_slack: np.ndarray
    gp_of_bus: np.ndarray
    gq_of_bus: np.ndarray
    gv_of_gen: np.ndarray
    gtheta_of_slack: np.ndarray


@dataclass(frozen=True)
class PowerSystem:
    name: str
    base_mva: float
    n_bus: int
    buses: BusGroup
    pq: PqGroup
    pv: PvGroup
    slack: SlackGroup
    lines: LineGroup
    shunts: ShuntGroup
    addr: AddressMap

    @property
    def n_var(self) -> int:
        return count_variables(self)

    @property
    def n_eq(self) -> int:
        return count_variables(self)


def count_variables(sys) -> int:
    """2*n_bus + n_pv + 2*n_slack (pflow/system_model.py:183-185)."""
    return 2 * sys.n_bus + len(sys.pv) + 2 * len(sys.slack)


def _c_reciprocal(re: np.ndarray, im: np.ndarray):
    """``1.0/complex(re, im)`` elementwise, bit-identical to CPython 3.12.

    CPython's complex division (Objects/complexobject.c ``_Py_c_quot``) is
    Smith's algorithm; the reference computes ``ys = 1.0/complex(r, x)``
    (pflow/system_model.py:294).  Restated with the same operation order.
    """
    are, aim = 1.0, 0.0
    abs_re = np.abs(re)
    abs_im = np.abs(im)
    by_re = abs_re >= abs_im
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio_a = im / re
        denom_a = re + im * ratio_a
        real_a = (are + aim * ratio_a) / denom_a
        imag_a = (aim - are * ratio_a) / denom_a
        ratio_b = re / im
        denom_b = re * ratio_b + im
        real_b = (are * ratio_b + aim) / denom_b
        imag_b = (aim * ratio_b - are) / denom_b
    return np.where(by_re, real_a, real_b), np.where(by_re, imag_a, imag_b)


def build_system(raw) -> PowerSystem:
    """Per-unit PowerSystem from a RawCase (pflow/system_model.py:188-276).

    Accepts this package's columnar :class:`RawCase` or the reference's
    row-record ``RawCase``.  Raises ``ValueError`` listing the violations
    when ``validate_case`` is not empty, as the reference does.
    """
    if not isinstance(raw, RawCase):
        raw = from_rows(raw)
    violations = validate_case(raw)
    if violations:
        detail = "; ".join(f"{v.code}[{v.row}]" for v in violations)
        raise ValueError(f"case fails validation: {detail}")

    base = raw.base_mva
    n_bus = raw.n_bus
    order = np.argsort(raw.bus_id, kind="stable")
    sorted_ids = raw.bus_id[order]

    def pos_of(ids):
        p = order[np.searchsorted(sorted_ids, ids)]
        return p.astype(np.int64)

    bus_type = raw.bus_type.astype(np.int8)
    buses = BusGroup(ids=raw.bus_id.astype(np.int64), bus_type=bus_type)

    # fixed injections: nonzero bus loads (bus order), then in-service gens
    # at PQ buses folded in as negative demand (gen order)
    load_rows = np.flatnonzero((raw.pd != 0.0) | (raw.qd != 0.0))
    gen_on = np.flatnonzero(raw.gen_status != 0)
    gen_pos = pos_of(raw.gen_bus[gen_on]) if gen_on.size else np.zeros(0, np.int64)
    gen_kind = bus_type[gen_pos] if gen_on.size else np.zeros(0, np.int8)
    slack_bus_rows = np.flatnonzero(bus_type == 3)
    is_slack_gen = np.zeros(gen_on.size, dtype=bool)
    slack_cand = np.flatnonzero(gen_kind == 3)
    if slack_cand.size:
        is_slack_gen[slack_cand[0]] = True
    is_pv = ((gen_kind == 2) | (gen_kind == 3)) & ~is_slack_gen
    is_pqgen = ~(is_pv | is_slack_gen)

    pq_bus = np.concatenate([load_rows, gen_pos[is_pqgen]]).astype(_IDX)
    pq_p0 = np.concatenate([raw.pd[load_rows] / base, (-raw.pg[gen_on][is_pqgen]) / base])
    pq_q0 = np.concatenate([raw.qd[load_rows] / base, (-raw.qg[gen_on][is_pqgen]) / base])
    pq = PqGroup(bus=pq_bus, p0=pq_p0.astype(np.float64), q0=pq_q0.astype(np.float64))

    n_pv = int(is_pv.sum())
    pv = PvGroup(
        bus=gen_pos[is_pv].astype(_IDX),
        p0=(raw.pg[gen_on][is_pv] / base).astype(np.float64),
        v0=raw.vg[gen_on][is_pv].astype(np.float64),
        qg=np.arange(n_pv, dtype=_IDX),
    )
    n_slack = int(is_slack_gen.sum())
    if n_slack:
        sb = int(gen_pos[is_slack_gen][0])
        # theta0 from the first bus row carrying the slack gen's bus id
        va = raw.va[np.flatnonzero(raw.bus_id == raw.bus_id[sb])[0]]
        theta0 = np.array([math.radians(float(va))])
        slack = SlackGroup(
            bus=np.array([sb], dtype=_IDX),
            v0=raw.vg[gen_on][is_slack_gen].astype(np.float64),
            theta0=theta0,
            qg=np.arange(n_pv, n_pv + n_slack, dtype=_IDX),
            ps=np.arange(n_slack, dtype=_IDX),
        )
    else:
        slack = SlackGroup(bus=np.zeros(0, _IDX), v0=np.zeros(0), theta0=np.zeros(0),
                           qg=np.zeros(0, _IDX), ps=np.zeros(0, _IDX))
    del slack_bus_rows

    sh_rows = np.flatnonzero((raw.gs != 0.0) | (raw.bs != 0.0))
    shunts = ShuntGroup(bus=sh_rows.astype(_IDX), g=raw.gs[sh_rows] / base,
                        b=raw.bs[sh_rows] / base)

    lines = _build_lines(raw, pos_of)
    addr = _build_addresses(n_bus, n_pv, n_slack)
    return PowerSystem(name=raw.name or "case", base_mva=base, n_bus=n_bus, buses=buses,
                       pq=pq, pv=pv, slack=slack, lines=lines, shunts=shunts, addr=addr)


def _build_lines(raw: RawCase, pos_of) -> LineGroup:
    """pflow/system_model.py:279-318, vectorised with identical operations."""
    on = np.flatnonzero(raw.br_status != 0)
    n = on.size
    bus_h = pos_of(raw.from_bus[on]).astype(_IDX) if n else np.zeros(0, _IDX)
    bus_k = pos_of(raw.to_bus[on]).astype(_IDX) if n else np.zeros(0, _IDX)
    r, x, bc = raw.r[on], raw.x[on], raw.b[on]
    m = raw.ratio[on]
    angle = raw.angle[on]
    g, b = _c_reciprocal(r, x)
    # math.radians / math.cos / math.sin per element: numpy's SIMD trig is
    # not guaranteed to round like libm, and phi is setup-only anyway
    shifted = np.flatnonzero(angle != 0.0)
    cphi = np.ones(n)
    sphi = np.zeros(n)
    has_shift = False
    for i in shifted:
        phi = math.radians(float(angle[i]))
        if phi != 0.0:
            has_shift = True
        cphi[i] = math.cos(phi)
        sphi[i] = math.sin(phi)
    gl = (g * cphi - b * sphi) / m
    bl = (b * cphi + g * sphi) / m
    gl2 = (g * cphi + b * sphi) / m
    bl2 = (b * cphi - g * sphi) / m
    bc2 = 0.5 * bc
    g_self_h = g / (m * m)
    b_self_h = (b + bc2) / (m * m)
    g_self_k = g.copy()
    b_self_k = b + bc2
    if not has_shift:
        gl2, bl2 = gl, bl
    return LineGroup(bus_h=bus_h, bus_k=bus_k, gl=gl, bl=bl, gl2=gl2, bl2=bl2,
                     g_self_h=g_self_h, b_self_h=b_self_h,
                     g_self_k=g_self_k, b_self_k=b_self_k,
                     ph=np.zeros(n), pk=np.zeros(n), qh=np.zeros(n), qk=np.zeros(n))


def _build_addresses(n_bus: int, n_pv: int, n_slack: int) -> AddressMap:
    """Identity blocks (pflow/system_model.py:321-332)."""
    n_gen = n_pv + n_slack
    return AddressMap(
        theta_of_bus=np.arange(n_bus, dtype=_IDX),
        v_of_bus=np.arange(n_bus, 2 * n_bus, dtype=_IDX),
        qg_of_gen=np.arange(2 * n_bus, 2 * n_bus + n_gen, dtype=_IDX),
        ps_of_slack=np.arange(2 * n_bus + n_gen, 2 * n_bus + n_gen + n_slack, dtype=_IDX),
        gp_of_bus=np.arange(n_bus, dtype=_IDX),
        gq_of_bus=np.arange(n_bus, 2 * n_bus, dtype=_IDX),
        gv_of_gen=np.arange(2 * n_bus, 2 * n_bus + n_gen, dtype=_IDX),
        gtheta_of_slack=np.arange(2 * n_bus + n_gen, 2 * n_bus + n_gen + n_slack, dtype=_IDX),
    )


def flat_start(sys) -> StateVector:
    """Reference angle everywhere, setpoint voltages (pflow/system_model.py:335-351)."""
    y = np.zeros(sys.n_var)
    addr = sys.addr
    theta0 = sys.slack.theta0[0] if len(sys.slack) else 0.0
    y[addr.theta_of_bus] = theta0
    y[addr.v_of_bus] = 1.0
    # the first generator on a bus sets its voltage; slack overrides PV
    for grp in (sys.pv, sys.slack):
        if len(grp):
            b, first = np.unique(np.asarray(grp.bus), return_index=True)
            y[addr.v_of_bus[b]] = grp.v0[first]
    return y


def random_state(sys, seed: int) -> StateVector:
    """Random evaluation state (pflow/cli.py:151-159 style).

    V ~ U(0.95, 1.05), theta ~ N(0, 0.2), Q_g and P_s ~ U(-0.5, 0.5).
    """
    rng = np.random.default_rng(seed)
    nb = sys.n_bus
    y = np.empty(sys.n_var)
    y[:nb] = rng.normal(0.0, 0.2, nb)
    y[nb:2 * nb] = rng.uniform(0.95, 1.05, nb)
    y[2 * nb:] = rng.uniform(-0.5, 0.5, sys.n_var - 2 * nb)
    return y
