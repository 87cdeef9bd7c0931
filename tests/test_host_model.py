"""Host model layer: build_system bit-exact with the reference, generator."""

import math

import numpy as np
import pytest

from _util import SINGLE, load, system_of
from paper_2011_11880_b200 import case as C
from paper_2011_11880_b200 import synth
from paper_2011_11880_b200.system_model import _c_reciprocal, build_system, flat_start


@pytest.mark.parametrize("name", SINGLE + ["batch_edge300"])
def test_build_system_bit_exact(name):
    d = load(name)
    if "sys_n_bus" not in d.files:
        pytest.skip("fixture without system arrays")
    s = system_of(d)
    for key in d.files:
        if not key.startswith("sys_") or key in ("sys_n_bus", "sys_lines_shift"):
            continue
        _, grp, field = key.split("_", 2)
        got = getattr(getattr(s, grp), field)
        ref = d[key]
        assert got.shape == ref.shape, key
        assert got.dtype == ref.dtype, key
        assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), key  # bitwise
    assert s.n_bus == int(d["sys_n_bus"])
    assert s.lines.has_shift == bool(d["sys_lines_shift"])


@pytest.mark.parametrize("name", SINGLE)
def test_flat_start_matches_reference(name):
    d = load(name)
    assert np.array_equal(flat_start(system_of(d)), d["ys"][0])


def test_complex_reciprocal_matches_cpython():
    rng = np.random.default_rng(0)
    re = np.concatenate([rng.uniform(-1, 1, 5000), rng.uniform(0.001, 0.05, 5000), [0.0, 1.0]])
    im = np.concatenate([rng.uniform(-1, 1, 5000), rng.uniform(0.01, 0.3, 5000), [0.1, 0.0]])
    g, b = _c_reciprocal(re, im)
    for i in range(re.size):
        z = 1.0 / complex(re[i], im[i])
        assert g[i] == z.real and b[i] == z.imag, i


def test_spec_line_coefficients():
    """pflow SPEC.md:111-113: r=0.01, x=0.1 -> gl 0.990099..., bl -9.900990..."""
    g, b = _c_reciprocal(np.array([0.01, 0.0]), np.array([0.1, 0.1]))
    assert math.isclose(g[0], 0.9900990099009901, rel_tol=1e-15)
    assert math.isclose(b[0], -9.900990099009901, rel_tol=1e-15)
    assert g[1] == 0.0 and b[1] == -10.0


def test_validate_codes():
    d = load("case14")
    raw = C.RawCase.from_arrays({k[5:]: d[k] for k in d.files if k.startswith("case_")})
    assert C.validate_case(raw) == []
    bt = raw.bus_type.copy()
    bt[1] = 3
    bad = C.RawCase(**{**raw.__dict__, "bus_type": bt})
    codes = [v.code for v in C.validate_case(bad)]
    assert "MULTIPLE_SLACK" in codes
    r = raw.r.copy()
    x = raw.x.copy()
    r[0] = x[0] = 0.0
    bad = C.RawCase(**{**raw.__dict__, "r": r, "x": x})
    assert [v.code for v in C.validate_case(bad)] == ["ZERO_IMPEDANCE"]
    with pytest.raises(ValueError, match="ZERO_IMPEDANCE"):
        build_system(bad)


def test_synth_shapes_and_determinism():
    c0 = synth.config_case(0, seed=0)
    assert c0.n_bus == 2000 and c0.n_branch == 2500
    s = build_system(c0)
    assert len(s.pv) == round(0.15 * 1999) and len(s.slack) == 1
    c0b = synth.config_case(0, seed=0)
    assert np.array_equal(c0.from_bus, c0b.from_bus) and np.array_equal(c0.r, c0b.r)
    assert not np.any(c0.from_bus == c0.to_bus)
    # connected: spanning tree included
    import scipy.sparse as sp
    import scipy.sparse.csgraph as cg

    a = sp.coo_matrix((np.ones(c0.n_branch), (c0.from_bus - 1, c0.to_bus - 1)),
                      shape=(2000, 2000))
    assert cg.connected_components(a, directed=False)[0] == 1


def test_synth_config2_counts():
    c2 = synth.config_case(2, seed=0)
    s = build_system(c2)
    assert s.n_bus == 70_000 and len(s.lines) == 88_000
    assert len(s.pq) == 45_000 and len(s.pv) == 6_000 and len(s.slack) == 1
    assert s.n_var == 2 * 70_000 + 6_000 + 2


def test_scenarios_shapes():
    s = build_system(synth.config_case(0, seed=0))
    sb = synth.make_scenarios(s, 40, seed=3)
    assert sb.y.shape == (s.n_var, 40)
    assert sb.pq_p.shape == (len(s.pq), 40)
    assert sb.outage.min() >= 0 and sb.outage.max() < len(s.lines)
    ratio = sb.pq_p / s.pq.p0[:, None]
    ok = np.isfinite(ratio)
    assert ratio[ok].min() >= 0.8 - 1e-12 and ratio[ok].max() <= 1.2 + 1e-12


def test_blocked_layout_roundtrip():
    from paper_2011_11880_b200.plan import from_blocked, to_blocked

    a = np.arange(70 * 5, dtype=np.float64).reshape(70, 5)
    flat = to_blocked(a)
    assert flat.size == 3 * 32 * 5
    assert np.array_equal(from_blocked(flat, 70, 5), a)
    # element (e, s) at ((s // 32) * n + e) * 32 + s % 32
    assert flat[((65 // 32) * 5 + 3) * 32 + 65 % 32] == a[65, 3]


def test_newton_options_accept_a_workflow_and_validate():
    """pflow's NewtonOptions(workflow=...) is accepted (and ignored: one GPU
    execution strategy); tol / max_iter are validated as pflow does."""
    from paper_2011_11880_b200.newton import NewtonOptions

    marker = object()
    assert NewtonOptions(workflow=marker).workflow is marker
    with pytest.raises(ValueError):
        NewtonOptions(max_iter=0)
    with pytest.raises(ValueError):
        NewtonOptions(tol=0)


def test_batched_lu_schedule_reference_solve_matches_scipy():
    """Host side of the batched sparse LU (batched_lu.py): the schedule built
    from the outage-proof pivots solves J x = b like SciPy, for the base
    scenario and for a scenario with a branch outaged."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla

    import oracle
    from paper_2011_11880_b200 import batched_lu as BL
    from paper_2011_11880_b200 import synth
    from paper_2011_11880_b200.batched_newton import base_lu, robust_row_match
    from paper_2011_11880_b200.plan import from_blocked, to_blocked
    from paper_2011_11880_b200.system_model import build_system, flat_start

    raw = synth.synth_case(200, 260, seed=4, pq_frac=0.6, pv_frac=0.15, shunt_frac=0.1)
    for col in ("pd", "qd", "pg"):
        getattr(raw, col)[:] *= 0.05
    s = build_system(raw)
    o = oracle.Oracle(s)
    n = s.n_var
    ptr, idx = o.pattern_csc()
    y0 = flat_start(s)

    def jac(outage):
        g, j, _ = o.eval_scenarios(1, to_blocked(y0[None]), outage=np.array([outage], np.int32))
        return (sp.csc_matrix((from_blocked(j, 1, o.nnz)[0], idx, ptr), shape=(n, n)).tocsr(),
                from_blocked(g, 1, n)[0])

    J0, g0 = jac(-1)
    J0.sort_indices()
    assert robust_row_match(J0, s.n_bus) is not None
    L, U, P, Q = base_lu(J0.tocsc(), n_bus=s.n_bus)
    sched = BL.analyze(J0.indptr, J0.indices, L, U, P, Q)
    assert 0 <= sched.D <= n and len(sched.row_list) == n
    for outage in (-1, 7):
        J, g = jac(outage)
        J.sort_indices()
        x = BL.reference_factor_solve(sched, J.data, -g)
        ref = spla.spsolve(J.tocsc(), -g)
        assert np.abs(x - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("name", SINGLE + ["batch_edge300"])
def test_q_limit_gen_rows_follow_build_system(name):
    """newton._pv_gen_rows (the limit-switching loop's map from PV index to
    gen row) follows build_system's PV numbering: same buses, setpoints and
    scheduled powers, in order."""
    from _util import case_of
    from paper_2011_11880_b200.newton import _pv_gen_rows

    raw = case_of(load(name))
    s = build_system(raw)
    rows = _pv_gen_rows(raw)
    assert len(rows) == len(s.pv.bus)
    order = np.argsort(raw.bus_id, kind="stable")
    pos = order[np.searchsorted(raw.bus_id[order], raw.gen_bus[rows])]
    assert np.array_equal(pos, s.pv.bus)
    assert np.array_equal(raw.vg[rows], s.pv.v0)
    assert np.array_equal(raw.pg[rows] / raw.base_mva, s.pv.p0)
