"""Generate tests/golden/*.npz by running the REFERENCE (pflow) itself.

Run in the build container only (needs /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python scripts/make_golden.py

Each fixture holds the raw case columns, the reference's PowerSystem arrays
(to pin this package's build_system bit-for-bit), evaluation states, and the
reference's outputs: g and CSC Jacobian data under workflow 1 (the oracle,
pflow SPEC.md:192) and workflow 5, the CSC pattern, the contribution pool,
the join index arrays, the triplet slots and slot values, and the per-line
injections.  ``batch_*.npz`` holds scenario-batched outputs produced by
mutating the reference's PowerSystem arrays per scenario.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("PFLOW_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import pflow  # noqa: E402
from pflow.residual import ResidualWorkspace  # noqa: E402
from pflow.jacobian import symbolic_pattern  # noqa: E402

from paper_2011_11880_b200 import case as C  # noqa: E402
from paper_2011_11880_b200 import synth  # noqa: E402
from paper_2011_11880_b200.system_model import random_state  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"
CASES = Path(REF) / "pflow" / "cases"


def sys_arrays(s) -> dict:
    d = {}
    for grp in ("pq", "pv", "slack", "shunts", "lines"):
        g = getattr(s, grp)
        for f in g.__dataclass_fields__:
            v = getattr(g, f)
            if v is not None and f not in ("ph", "pk", "qh", "qk"):
                d[f"sys_{grp}_{f}"] = v
    d["sys_lines_shift"] = np.array(s.lines.gl2 is not s.lines.gl)
    d["sys_n_bus"] = np.array(s.n_bus)
    return d


def tiny_edge_case() -> C.RawCase:
    """Hand-made 5-bus case: parallel and reversed branches, tap+shift,
    out-of-service rows, an isolated bus, two gens on one bus, a second gen
    on the slack bus, a generator on a PQ bus."""
    bus = dict(bus_id=[10, 20, 30, 40, 50], bus_type=[3, 2, 1, 1, 1],
               pd=[0.0, 20.0, 45.0, 10.0, 0.0], qd=[0.0, 5.0, 15.0, 2.0, 0.0],
               gs=[0.0, 0.0, 0.0, 3.0, 1.5], bs=[0.0, 0.0, 0.0, 12.0, -8.0],
               vm=[1.04, 1.02, 1.0, 1.0, 1.0], va=[2.5, 0.0, 0.0, 0.0, 0.0],
               base_kv=[230.0] * 5)
    gen = dict(gen_bus=[10, 10, 20, 20, 30, 50], pg=[50.0, 10.0, 40.0, 15.0, 12.0, 5.0],
               qg=[0.0, 0.0, 0.0, 0.0, 3.0, 0.0], qmax=[99.0] * 6, qmin=[-99.0] * 6,
               vg=[1.04, 1.03, 1.02, 1.01, 1.0, 1.0], gen_status=[1, 1, 1, 1, 1, 0])
    branch = dict(from_bus=[10, 20, 10, 20, 30, 10, 50],
                  to_bus=[20, 10, 20, 30, 10, 30, 30],
                  r=[0.01, 0.02, 0.015, 0.03, 0.0, 0.05, 0.02],
                  x=[0.1, 0.12, 0.09, 0.15, 0.08, 0.2, 0.1],
                  b=[0.02, 0.01, 0.0, 0.03, 0.0, 0.01, 0.04],
                  ratio=[1.0, 1.0, 0.97, 1.0, 1.05, 1.0, 1.0],
                  angle=[0.0, 0.0, 0.0, 0.0, -4.0, 0.0, 0.0],
                  br_status=[1, 1, 1, 1, 1, 0, 1])
    return C.make_case(100.0, bus, gen, branch, name="tiny_edge")


def slack_only_case() -> C.RawCase:
    """Single slack bus with a shunt and a load, no branches."""
    bus = dict(bus_id=[1], bus_type=[3], pd=[5.0], qd=[1.0], gs=[1.0], bs=[2.0],
               vm=[1.0], va=[0.0], base_kv=[100.0])
    gen = dict(gen_bus=[1], pg=[5.0], qg=[0.0], qmax=[9.0], qmin=[-9.0], vg=[1.0],
               gen_status=[1])
    z = np.zeros(0)
    branch = dict(from_bus=z, to_bus=z, r=z, x=z, b=z, ratio=z, angle=z, br_status=z)
    return C.make_case(100.0, bus, gen, branch, name="slack_only")


def golden_single(name: str, raw_cols: C.RawCase, n_random: int, seed: int) -> None:
    ref_raw = C.to_rows(raw_cols)
    s = pflow.build_system(ref_raw)
    rws = ResidualWorkspace(s)
    jws = symbolic_pattern(s)
    ys = [pflow.flat_start(s)] + [random_state(s, seed + i) for i in range(n_random)]
    out = {"name": np.array(name)}
    out.update({f"case_{k}": v for k, v in raw_cols.to_arrays().items()})
    out.update(sys_arrays(s))
    out["ys"] = np.array(ys)
    g1, g5, j1, j5 = [], [], [], []
    for y in ys:
        y = y.copy()
        for wf, gl, jl in ((1, g1, j1), (5, g5, j5)):
            cfg = pflow.workflow_config(wf)
            g = np.zeros(s.n_eq)
            pflow.evaluate_residual(s, y, cfg, g, rws)
            gl.append(g.copy())
            jl.append(pflow.evaluate_jacobian(s, y, cfg, jws).data.copy())
    out["g_wf1"], out["g_wf5"] = np.array(g1), np.array(g5)
    out["j_wf1"], out["j_wf5"] = np.array(j1), np.array(j5)
    out["csc_indptr"] = jws.csc.indptr.astype(np.int32)
    out["csc_indices"] = jws.csc.indices.astype(np.int32)
    csr = jws.csc.tocsr()
    out["csr_indptr"] = csr.indptr.astype(np.int32)
    out["csr_indices"] = csr.indices.astype(np.int32)
    # internals at the last random state under wf1
    y = ys[-1].copy()
    cfg = pflow.workflow_config(1)
    pflow.evaluate_residual(s, y, cfg, np.zeros(s.n_eq), rws)
    out["pool"] = rws.pool.copy()
    pflow.evaluate_jacobian(s, y, cfg, jws)
    out["slot_vals"] = jws.vals.copy()
    out["join_ptr"], out["join_split"], out["join_idx"] = (
        rws._join_ptr, rws._join_split, rws._join_idx)
    out["slot_rows"], out["slot_cols"] = jws.rows, jws.cols
    out["slot_to_csc"], out["gather_ptr"] = jws.slot_to_csc, jws._gather_ptr
    pflow.line_injections(s, y)
    out["line_inj"] = np.array([s.lines.ph, s.lines.pk, s.lines.qh, s.lines.qk]).copy()
    out["dev_inj"] = np.concatenate([
        *pflow.pq_injections(s, y), *pflow.pv_injections(s, y),
        *pflow.slack_injections(s, y), *pflow.shunt_injections(s, y)])
    if s.n_var <= 400:
        out["fd_jac"] = pflow.finite_difference_jacobian(s, y)
    # the caller of the path: pflow's own Newton solve from flat start
    try:
        res = pflow.newton_solve(s, pflow.flat_start(s), pflow.NewtonOptions())
        out["newton_converged"] = np.array(res.converged)
        out["newton_iterations"] = np.array(res.iterations)
        out["newton_y"] = res.y
        out["newton_mismatch"] = np.array(res.final_mismatch)
    except pflow.SingularMatrixError:  # isolated buses: singular by construction
        out["newton_converged"] = np.array(False)
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(f"{name}: n_var={s.n_var} nnz={jws.nnz} slots={jws.vals.size} states={len(ys)}")


def golden_batch(name: str, raw_cols: C.RawCase, K: int, seed: int) -> None:
    """Scenario batch via in-place mutation of the reference PowerSystem."""
    s = pflow.build_system(C.to_rows(raw_cols))
    rws = ResidualWorkspace(s)
    jws = symbolic_pattern(s)
    sb = synth.make_scenarios(s, K, seed)
    ln = s.lines
    coef = [ln.gl, ln.bl, ln.gl2, ln.bl2, ln.g_self_h, ln.b_self_h, ln.g_self_k, ln.b_self_k]
    p0, q0, pv0 = s.pq.p0.copy(), s.pq.q0.copy(), s.pv.p0.copy()
    cfg = pflow.workflow_config(1)
    gs, js, norms = [], [], []
    for k in range(K):
        y, pq_p, pq_q, pv_p, l = sb.scenario(k)
        s.pq.p0[:] = pq_p
        s.pq.q0[:] = pq_q
        s.pv.p0[:] = pv_p
        saved = [c[l] for c in coef]
        for c in coef:
            c[l] = 0.0
        g = np.zeros(s.n_eq)
        pflow.evaluate_residual(s, y, cfg, g, rws)
        gs.append(g)
        js.append(pflow.evaluate_jacobian(s, y, cfg, jws).data.copy())
        norms.append(float(np.abs(g).max()))
        for c, v in zip(coef, saved):
            c[l] = v
    s.pq.p0[:], s.pq.q0[:], s.pv.p0[:] = p0, q0, pv0
    out = {"name": np.array(name), "K": np.array(K), "seed": np.array(seed)}
    out.update({f"case_{k}": v for k, v in raw_cols.to_arrays().items()})
    out["y"] = np.ascontiguousarray(sb.y.T)           # [K, n_var]
    out["pq_p"] = np.ascontiguousarray(sb.pq_p.T)
    out["pq_q"] = np.ascontiguousarray(sb.pq_q.T)
    out["pv_p"] = np.ascontiguousarray(sb.pv_p.T)
    out["outage"] = sb.outage
    out["g_wf1"], out["j_wf1"], out["norms"] = np.array(gs), np.array(js), np.array(norms)
    out["csc_indptr"] = jws.csc.indptr.astype(np.int32)
    out["csc_indices"] = jws.csc.indices.astype(np.int32)
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(f"{name}: K={K} n_var={s.n_var} nnz={jws.nnz}")


def main() -> None:
    OUT.mkdir(parents=True, exist_ok=True)
    for nm, seed in (("case2", 11), ("case5_shift", 12), ("case14", 13)):
        raw = C.from_rows(pflow.parse_case_file(CASES / f"{nm}.m"))
        golden_single(nm, raw, n_random=3, seed=seed)
    golden_single("tiny_edge", tiny_edge_case(), n_random=3, seed=21)
    golden_single("slack_only", slack_only_case(), n_random=2, seed=22)
    golden_single("edge300", synth.synth_case(300, 420, seed=5, pq_frac=0.5, pv_frac=0.2,
                                              shunt_frac=0.3, shift_frac=0.2,
                                              out_of_service_frac=0.05, hub_frac=0.02,
                                              hub_degree=20, name="edge300"),
                  n_random=2, seed=31)
    golden_single("config0", synth.config_case(0, seed=0), n_random=2, seed=41)
    golden_batch("batch_edge300", synth.synth_case(300, 420, seed=6, pq_frac=0.5, pv_frac=0.2,
                                                   shunt_frac=0.3, shift_frac=0.2,
                                                   name="batch_edge300"), K=6, seed=51)


if __name__ == "__main__":
    main()
