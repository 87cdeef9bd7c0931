"""The reference's intended property suite (pflow SPEC.md), on the GPU path.

pflow ships no tests; SPEC.md states the properties its evaluation must
have.  Each test cites the clause it checks:

* SPEC.md:257, 452 (acceptance 2): analytic Jacobian vs central finite
  differences, max relative entry error < 1e-6 at 100 random states on
  every bundled small case (pflow/cli.py:151-176 draws the states).
* device independence -- permuting the line order
  changes no residual or Jacobian entry beyond the reassociation tolerance;
  the permuted system is still bit-identical to wf1 run on the permuted
  order.
* SPEC.md:197, 457 (acceptance 7): allocation-free steady state -- after
  warm-up no evaluation entry point allocates device memory.
* complex-power oracle -- every line's (p + jq) at both
  terminals equals V conj(I) of the MATPOWER admittance form within 1e-12
  over >= 1000 randomised branches (taps and phase shifts included).
* pattern stability across plans and evaluations.
"""

import numpy as np
import pytest

import oracle
from _util import assert_parity, load, system_of
from paper_2011_11880_b200 import synth
from paper_2011_11880_b200.system_model import build_system, random_state

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _check_states(s, n, seed):
    """pflow check's random states (cli.py:151-159): theta + U(-0.3, 0.3),
    V * U(0.95, 1.05), Q_g / P_s + U(-0.5, 0.5) around the flat start."""
    from paper_2011_11880_b200.system_model import flat_start

    rng = np.random.default_rng(seed)
    y0 = flat_start(s)
    nb = s.n_bus
    for _ in range(n):
        y = y0.copy()
        y[:nb] += rng.uniform(-0.3, 0.3, nb)
        y[nb:2 * nb] *= rng.uniform(0.95, 1.05, nb)
        y[2 * nb:] += rng.uniform(-0.5, 0.5, s.n_var - 2 * nb)
        yield y


@pytest.mark.parametrize("name", ["case2", "case5_shift", "case14"])
def test_fd_agreement_100_random_states(name):
    from paper_2011_11880_b200.jacobian import JacobianWorkspace, finite_difference_jacobian
    from paper_2011_11880_b200.residual import ResidualWorkspace

    s = system_of(load(name))
    jws = JacobianWorkspace(s)
    rws = ResidualWorkspace(s, jws.plan)
    worst = 0.0
    for y in _check_states(s, 100, seed=11):
        jac = jws.run(y).toarray()
        fd = finite_difference_jacobian(s, y, workspace=rws)
        worst = max(worst, float((np.abs(jac - fd) / np.maximum(1.0, np.abs(fd))).max()))
    assert worst < 1e-6, worst


def _permuted_case(raw, seed):
    """The same network with its branch rows listed in a shuffled order (bus
    numbering and device order unchanged, so y and g index alike)."""
    import dataclasses

    rng = np.random.default_rng(seed)
    pb = rng.permutation(len(raw.from_bus))
    cols = {f.name: getattr(raw, f.name) for f in dataclasses.fields(raw)}
    for k in ("from_bus", "to_bus", "r", "x", "b", "ratio", "angle", "br_status"):
        if k in cols:
            cols[k] = np.ascontiguousarray(cols[k][pb])
    return type(raw)(**cols)


def test_device_permutation_invariance():
    from paper_2011_11880_b200.plan import Plan

    raw = synth.synth_case(400, 700, seed=21, pq_frac=0.6, pv_frac=0.15, shunt_frac=0.1,
                           shift_frac=0.2, hub_frac=0.02, hub_degree=25)
    s1 = build_system(raw)
    s2 = build_system(_permuted_case(raw, 5))
    p1, p2 = Plan(s1), Plan(s2)
    c1, c2 = p1.pattern_csc(), p2.pattern_csc()
    assert np.array_equal(c1[0], c2[0]) and np.array_equal(c1[1], c2[1])
    o2 = oracle.Oracle(s2)
    for y in _check_states(s1, 10, seed=3):
        outs = []
        for p in (p1, p2):
            g, j, n = p.empty(p.n_var), p.empty(p.nnz), p.empty(1)
            p.eval(torch.as_tensor(y, device="cuda"), g, j, n)
            _, _, perm = p.pattern_csc()
            outs.append((g.cpu().numpy(), j.cpu().numpy()[perm]))
        (g1, j1), (g2, j2) = outs
        # reassociation only: the SPEC's normwise tolerance
        assert np.abs(g1 - g2).max() <= 1e-12 * max(1.0, np.abs(g1).max())
        assert np.abs(j1 - j2).max() <= 1e-12 * max(1.0, np.abs(j1).max())
        # and the permuted system is still wf1's own bits in its own order
        assert_parity(g2, o2.residual(y), "permuted g")
        assert_parity(j2, o2.jacobian(y), "permuted J")


def test_allocation_free_steady_state():
    """After warm-up, no entry point allocates device memory: the library's
    own allocation counter (every cudaMalloc it makes) and torch's allocator
    are both unchanged over 100 rounds of every evaluation call."""
    from paper_2011_11880_b200.batched import ScenarioBuffers
    from paper_2011_11880_b200.jacobian import JacobianWorkspace
    from paper_2011_11880_b200.plan import Plan, alloc_count, to_blocked
    from paper_2011_11880_b200.residual import ResidualWorkspace

    s = build_system(synth.config_case(0, seed=0))
    plan = Plan(s)
    y = random_state(s, 1)
    dy = torch.as_tensor(y, device="cuda")
    g, j, n = plan.empty(plan.n_var), plan.empty(plan.nnz), plan.empty(1)
    K = 40
    buf = ScenarioBuffers(plan, K)
    buf.upload(synth.make_scenarios(s, K, seed=2))
    jc = plan.empty(plan.nnz, K)
    rws, jws = ResidualWorkspace(s, plan), JacobianWorkspace(s, plan)
    yh = np.array(y)
    sb = synth.make_scenarios(s, K, seed=3)
    hy = to_blocked(sb.y.T)
    hg, hj, hn = np.zeros(hy.size), np.zeros(64 * plan.nnz), np.zeros(K)

    def every_call():
        plan.eval(dy, g, j, n)
        plan.eval(dy, g=g)
        plan.eval(dy, jval=j)
        buf.evaluate()
        plan.jac_to_csc(buf.jval, jc, K)
        rws.run(yh)
        jws.run(yh)
        plan.eval_batched_host(K, hy, g=hg, jval=hj, norms=hn)

    every_call()                        # warm-up: first-use staging is allocated here
    torch.cuda.synchronize()
    a0, t0 = alloc_count(), torch.cuda.memory_allocated()
    r0 = torch.cuda.memory_reserved()
    for _ in range(100):
        every_call()
    torch.cuda.synchronize()
    assert alloc_count() == a0
    assert torch.cuda.memory_allocated() == t0 and torch.cuda.memory_reserved() == r0


def test_complex_power_oracle_1000_draws():
    """(p_h + j q_h, p_k + j q_k) from the device line kernel equal
    V_h conj(I_h), V_k conj(I_k) with MATPOWER's branch admittances
    Yff = (ys + j bc/2) / |t|^2, Yft = -ys / conj(t), Ytf = -ys / t,
    Ytt = ys + j bc/2 (t = m e^{j phi}), over 1,200 random branches with
    taps and phase shifts, two random states each."""
    raw = synth.synth_case(300, 1200, seed=4, pq_frac=0.5, pv_frac=0.2, shift_frac=0.5,
                           shunt_frac=0.1)
    s = build_system(raw)
    from paper_2011_11880_b200.plan import Plan

    plan = Plan(s)
    assert plan.n_line == 1200
    idx = {b: i for i, b in enumerate(raw.bus_id)}
    f = np.array([idx[b] for b in raw.from_bus])
    t = np.array([idx[b] for b in raw.to_bus])
    ys = 1.0 / (raw.r + 1j * raw.x)
    tap = raw.ratio * np.exp(1j * np.deg2rad(raw.angle))
    assert np.count_nonzero(raw.angle) > 300 and np.count_nonzero(raw.ratio != 1.0) > 50
    ytt = ys + 0.5j * raw.b
    yff, yft, ytf = ytt / (tap * np.conj(tap)), -ys / np.conj(tap), -ys / tap
    nb = s.n_bus
    for seed in (1, 2):
        y = random_state(s, seed)
        ph, pk, qh, qk = (a.cpu().numpy() for a in plan.line_injections(
            torch.as_tensor(y, device="cuda")))
        V = y[nb:2 * nb] * np.exp(1j * y[:nb])
        sf = V[f] * np.conj(yff * V[f] + yft * V[t])
        st = V[t] * np.conj(ytf * V[f] + ytt * V[t])
        for got, ref in ((ph, sf.real), (qh, sf.imag), (pk, st.real), (qk, st.imag)):
            assert (np.abs(got - ref) <= 1e-12 * np.maximum(1.0, np.abs(ref))).all()


def test_pattern_stability():
    from paper_2011_11880_b200.plan import Plan

    s = build_system(synth.config_case(0, seed=0))
    a, b = Plan(s), Plan(s)
    pa, pb = a.pattern_csr(), b.pattern_csr()
    assert all(np.array_equal(x, z) for x, z in zip(pa, pb))
    y = torch.as_tensor(random_state(s, 2), device="cuda")
    for _ in range(3):
        a.eval(y, a.empty(a.n_var), a.empty(a.nnz), a.empty(1))
    assert all(np.array_equal(x, z) for x, z in zip(a.pattern_csr(), pa))
    assert all(np.array_equal(x, z) for x, z in zip(a.pattern_csc(), b.pattern_csc()))
