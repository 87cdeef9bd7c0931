import sys
from pathlib import Path
import numpy as np, scipy.sparse as sp, scipy.sparse.linalg as spla, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2])); sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "tests"))
from test_gpu_parity import _light_case
from paper_2011_11880_b200 import synth, batched_lu as BL
from paper_2011_11880_b200.batched_newton import base_lu
from paper_2011_11880_b200.plan import Plan, from_blocked, to_blocked
from paper_2011_11880_b200.system_model import build_system, flat_start
s = build_system(_light_case(300, 390, seed=3)); plan = Plan(s)
K = 24; sb = synth.make_scenarios(s, K, seed=4)
print("outages", sb.outage[:10], "branch 6:", sb.outage[6], "bus_h/k", s.lines.bus_h[sb.outage[6]], s.lines.bus_k[sb.outage[6]])
y0 = flat_start(s); Y = np.tile(y0, (K, 1))
dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
t = lambda a: dev(to_blocked(np.ascontiguousarray(a.T)))
y = dev(to_blocked(Y)); out = torch.as_tensor(sb.outage, device="cuda")
n, nnz = plan.n_var, plan.nnz
g, j = plan.empty(n, K), plan.empty(nnz, K)
plan.eval_batched(K, y, t(sb.pq_p), t(sb.pq_q), t(sb.pv_p), out, g, j, None); torch.cuda.synchronize()
J = from_blocked(j.cpu().numpy(), K, nnz); G = from_blocked(g.cpu().numpy(), K, n)
indptr, indices = plan.pattern_csr()
j0 = plan.empty(nnz, K); plan.eval_batched(K, y, t(sb.pq_p), t(sb.pq_q), t(sb.pv_p), None, None, j0, None); torch.cuda.synchronize()
J0 = from_blocked(j0.cpu().numpy(), K, nnz)
L, U, P, Q = base_lu(sp.csr_matrix((J0[0], indices, indptr), shape=(n, n)).tocsc())
sch = BL.analyze(indptr, indices, L, U, P, Q)
print("D", sch.D)
for k in (0, 5, 6, 7):
    A = sp.csr_matrix((J[k], indices, indptr), shape=(n, n))
    ref = spla.spsolve(A.tocsc(), -G[k])
    x = BL.reference_factor_solve(sch, J[k], -G[k])
    res = np.abs(A @ x + G[k]).max()
    print(k, "outage", sb.outage[k], "rel err vs scipy", np.abs(x - ref).max() / np.abs(ref).max(), "resid", res, "cond est", np.linalg.cond(A.toarray()) if n < 1500 else None)
