import sys
from pathlib import Path
import numpy as np, scipy.sparse as sp, scipy.sparse.linalg as spla, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2])); sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "tests"))
from test_gpu_parity import _light_case
from paper_2011_11880_b200 import synth, batched_lu as BL, _abi
from paper_2011_11880_b200.batched_newton import base_lu
from paper_2011_11880_b200.plan import Plan, from_blocked, to_blocked
from paper_2011_11880_b200.system_model import build_system, flat_start
s = build_system(_light_case(2000, 2500, seed=0)); plan = Plan(s)
for K in (64, 256):
    sb = synth.make_scenarios(s, K, seed=1, outages=False)
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
    t = lambda a: dev(to_blocked(np.ascontiguousarray(a.T)))
    n, nnz = plan.n_var, plan.nnz
    y = dev(to_blocked(np.tile(flat_start(s), (K, 1))))
    g, j = plan.empty(n, K), plan.empty(nnz, K)
    plan.eval_batched(K, y, t(sb.pq_p), t(sb.pq_q), t(sb.pv_p), None, g, j, None); torch.cuda.synchronize()
    indptr, indices = plan.pattern_csr()
    J = from_blocked(j.cpu().numpy(), K, nnz); G = from_blocked(g.cpu().numpy(), K, n)
    L, U, P, Q = base_lu(sp.csr_matrix((J[0], indices, indptr), shape=(n, n)).tocsc(), n_bus=plan.n_bus)
    sch = BL.analyze(indptr, indices, L, U, P, Q)
    lu = BL.DeviceSparseLU(sch, K); lu.factor(j); dx = lu.solve(g); torch.cuda.synchronize()
    X = from_blocked(dx.cpu().numpy(), K, n)
    errs = []
    for k in range(K):
        A = sp.csr_matrix((J[k], indices, indptr), shape=(n, n))
        errs.append(np.abs(A @ X[k] + G[k]).max() / np.abs(G[k]).max())
    errs = np.array(errs)
    print(K, "D", sch.D, "worst rel resid", errs.max(), "argmax", errs.argmax(), "n bad(>1e-6)", (errs > 1e-6).sum(), "bad idx", np.nonzero(errs > 1e-6)[0][:20])
