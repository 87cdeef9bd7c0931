"""The drop-in, executed: the reference's own caller driving this engine.

pflow's ``newton_solve(sys, y0, opts, solver, residual_ws, jacobian_ws)``
duck-types its workspaces (pflow/newton.py:49-70): it calls
``evaluate_residual`` (ws.bind / ws.run / ws.residual, residual.py:262-274)
and ``evaluate_jacobian`` (ws.sys is sys, ws.run -> csc_matrix,
jacobian.py:216-221).  Here the live pflow package (imported from
$PFLOW_SRC or baseline/_ref; skipped with the reason when absent) runs its
own Newton loop with this package's GPU workspaces, built straight from
pflow's own PowerSystem, and is compared with the same loop on pflow's own
wf1 workspaces.  Because the GPU residual and Jacobian are bit-identical to
wf1, every iterate -- and so the solution -- is bit-identical too.
"""

import numpy as np
import pytest

from oracle import live

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pflow():
    mod, why = live.import_pflow()
    if mod is None:
        pytest.skip(why)
    return mod


def _systems(pflow):
    from paper_2011_11880_b200 import synth

    out = [(n, live.pflow_fixture(pflow, n)) for n in ("case2", "case5_shift", "case14")]
    # BASELINE config 0 (2k buses) at light load so flat-start Newton converges
    raw = synth.config_case(0, seed=0)
    for col in (raw.pd, raw.qd, raw.pg):
        col *= 0.05
    out.append(("config0_light", live.pflow_system(pflow, raw)))
    return out


@pytest.mark.parametrize("fused", [False, True])
def test_pflow_newton_solve_with_gpu_workspaces(pflow, fused):
    """fused: JacobianWorkspace(..., residual_ws=rws) -- each Newton
    iteration's residual call also evaluates J in the same launch."""
    from paper_2011_11880_b200.jacobian import JacobianWorkspace
    from paper_2011_11880_b200.residual import ResidualWorkspace

    for name, psys in _systems(pflow):
        opts = pflow.NewtonOptions()
        rws = ResidualWorkspace(psys)
        jws = JacobianWorkspace(psys, residual_ws=rws) if fused else JacobianWorkspace(psys)
        assert jws.sys is psys
        ref = pflow.newton_solve(psys, pflow.flat_start(psys), opts)
        got = pflow.newton_solve(psys, pflow.flat_start(psys), opts, residual_ws=rws,
                                 jacobian_ws=jws)
        assert (got.converged, got.diverged, got.iterations) == \
            (ref.converged, ref.diverged, ref.iterations), name
        assert got.converged, name
        assert got.final_mismatch == ref.final_mismatch, name
        assert np.array_equal(got.y.view(np.int64), ref.y.view(np.int64)), name


def test_pflow_evaluate_calls_on_gpu_workspaces(pflow):
    """pflow's evaluate_residual / evaluate_jacobian with the GPU workspaces
    at random states: the same bits as pflow's own wf1 workspaces, the same
    csc_matrix object returned every call, pflow's ValueErrors preserved."""
    from paper_2011_11880_b200.jacobian import JacobianWorkspace
    from paper_2011_11880_b200.residual import ResidualWorkspace

    cfg = pflow.workflow_config(1)
    for name, psys in _systems(pflow):
        rws, jws = ResidualWorkspace(psys), JacobianWorkspace(psys)
        prws, pjws = pflow.ResidualWorkspace(psys), pflow.symbolic_pattern(psys)
        assert np.array_equal(jws.csc.indptr, pjws.csc.indptr)
        assert np.array_equal(jws.csc.indices, pjws.csc.indices)
        rng = np.random.default_rng(7)
        y = pflow.flat_start(psys)
        nb = psys.n_bus
        out = np.zeros(psys.n_var)
        first = None
        for _ in range(5):
            y[:nb] = rng.normal(0, 0.2, nb)
            y[nb:2 * nb] = rng.uniform(0.95, 1.05, nb)
            y[2 * nb:] = rng.uniform(-0.5, 0.5, psys.n_var - 2 * nb)
            g = pflow.evaluate_residual(psys, y, cfg, out, rws)
            g_ref = pflow.evaluate_residual(psys, y, cfg, None, prws).copy()
            assert np.array_equal(g.view(np.int64), g_ref.view(np.int64)), name
            J = pflow.evaluate_jacobian(psys, y, cfg, jws)
            J_ref = pflow.evaluate_jacobian(psys, y, cfg, pjws)
            assert np.array_equal(J.data.view(np.int64), J_ref.data.view(np.int64)), name
            first = J if first is None else first
            assert J is first
        with pytest.raises(ValueError):
            pflow.evaluate_residual(psys, np.zeros(psys.n_var + 1), cfg, None, rws)
        other = _systems(pflow)[0][1]
        with pytest.raises(ValueError):
            pflow.evaluate_jacobian(other, y, cfg, jws)
