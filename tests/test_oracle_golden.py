"""Pin the CPU oracle (oracle/liboracle.so) to the reference's own outputs.

The golden vectors in tests/golden were produced by running pflow itself
(scripts/make_golden.py).  The oracle's workflow-1 restatement must match
them bit for bit; its workflow-5 restatement within the reference's own
cross-workflow tolerance (pflow/cli.py:183-196).
"""

import numpy as np
import pytest

import oracle
from _util import SINGLE, assert_parity, load, system_of
from paper_2011_11880_b200.plan import from_blocked, to_blocked


@pytest.fixture(scope="module", params=SINGLE)
def fx(request):
    d = load(request.param)
    s = system_of(d)
    return d, s, oracle.Oracle(s)


def test_pattern_bit_exact(fx):
    d, s, o = fx
    indptr, indices = o.pattern_csc()
    assert np.array_equal(indptr, d["csc_indptr"])
    assert np.array_equal(indices, d["csc_indices"])


def test_wf1_bit_exact(fx):
    d, s, o = fx
    for i, y in enumerate(d["ys"]):
        assert np.array_equal(o.residual(y, 1), d["g_wf1"][i]), f"g state {i}"
        assert np.array_equal(o.jacobian(y, 1), d["j_wf1"][i]), f"J state {i}"


def test_wf5_matches_reference_wf5_normwise(fx):
    d, s, o = fx
    for i, y in enumerate(d["ys"]):
        g5 = o.residual(y, 5)
        j5 = o.jacobian(y, 5)
        scale_g = max(1.0, np.abs(d["g_wf1"][i]).max())
        scale_j = max(1.0, np.abs(d["j_wf1"][i]).max()) if d["j_wf1"][i].size else 1.0
        assert np.abs(g5 - d["g_wf5"][i]).max(initial=0) / scale_g <= 1e-12
        assert np.abs(j5 - d["j_wf5"][i]).max(initial=0) / scale_j <= 1e-12


def test_internals_bit_exact(fx):
    d, s, o = fx
    y = d["ys"][-1]
    o.residual(y, 1)
    assert np.array_equal(o.pool(), d["pool"])
    o.jacobian(y, 1)
    assert np.array_equal(o.vals(), d["slot_vals"])
    ptr, split, idx = o.join()
    assert np.array_equal(ptr, d["join_ptr"])
    assert np.array_equal(split, d["join_split"])
    assert np.array_equal(idx, d["join_idx"])
    rows, cols, s2c, gp = o.slots()
    assert np.array_equal(rows, d["slot_rows"])
    assert np.array_equal(cols, d["slot_cols"])
    assert np.array_equal(s2c, d["slot_to_csc"])
    assert np.array_equal(gp, d["gather_ptr"])
    li = o.line_injections(y, 1)
    assert all(np.array_equal(a, b) for a, b in zip(li, d["line_inj"]))


def test_threaded_wf3_equals_wf1(fx):
    d, s, o = fx
    y = d["ys"][-1]
    g, j = o.eval_threaded(y, 4)
    assert np.array_equal(g, d["g_wf1"][-1])
    assert np.array_equal(j, d["j_wf1"][-1])


def test_fd_oracle_agrees(fx):
    d, s, o = fx
    if "fd_jac" not in d.files:
        pytest.skip("no FD reference stored for this size")
    import scipy.sparse as sp

    n = s.n_var
    jac = sp.csc_matrix((o.jacobian(d["ys"][-1]), d["csc_indices"], d["csc_indptr"]),
                        shape=(n, n)).toarray()
    fd = d["fd_jac"]
    err = np.abs(jac - fd) / np.maximum(1.0, np.abs(fd))
    assert err.max() < 1e-6  # pflow/cli.py:174


def test_batch_golden_bit_exact():
    d = load("batch_edge300")
    s = system_of(d)
    o = oracle.Oracle(s)
    K = int(d["K"])
    g, j, norms = o.eval_scenarios(K, to_blocked(d["y"]), to_blocked(d["pq_p"]),
                                   to_blocked(d["pq_q"]), to_blocked(d["pv_p"]), d["outage"])
    assert np.array_equal(from_blocked(g, K, o.n_var), d["g_wf1"])
    assert np.array_equal(from_blocked(j, K, o.nnz), d["j_wf1"])
    assert np.array_equal(norms, d["norms"])
    # threaded scenario evaluation is identical
    g2, j2, n2 = o.eval_scenarios(K, to_blocked(d["y"]), to_blocked(d["pq_p"]),
                                  to_blocked(d["pq_q"]), to_blocked(d["pv_p"]), d["outage"],
                                  nthreads=3)
    assert np.array_equal(g2, g) and np.array_equal(j2, j) and np.array_equal(n2, norms)


def test_spec_known_answers():
    """pflow SPEC.md:121, 191, 233 known answers through the oracle."""
    d = load("case2")
    s = system_of(d)
    o = oracle.Oracle(s)
    assert o.n_slots == 20
    g = o.residual(d["ys"][0])
    pq_bus = int(s.pq.bus[0])
    assert g[pq_bus] == -0.5
    assert system_of(load("case14")).n_var == 34


def test_sincos_poly_accuracy():
    x = np.linspace(-np.pi, np.pi, 20001)
    s, c = oracle.sincos_poly(x)
    assert np.abs(s - np.sin(x)).max() < 4e-16
    assert np.abs(c - np.cos(x)).max() < 4e-16


def test_assert_parity_helper():
    assert_parity(np.array([1.0, 0.0]), np.array([1.0 + 1e-13, 5e-15]), bitwise=False)
    with pytest.raises(AssertionError):
        assert_parity(np.array([1.0]), np.array([1.0 + 1e-11]), bitwise=False)
    # the default also demands bit-identity (signed zeros included)
    assert_parity(np.array([1.0, -0.0]), np.array([1.0, -0.0]))
    with pytest.raises(AssertionError, match="bit-identical"):
        assert_parity(np.array([1.0]), np.array([1.0 + 1e-13]))
    with pytest.raises(AssertionError, match="bit-identical"):
        assert_parity(np.array([0.0]), np.array([-0.0]))
