"""BatchedLU (cusolverRf per scenario) against scipy on config-0 Jacobians."""
import faulthandler; faulthandler.enable()
import sys, time
from pathlib import Path
import numpy as np, scipy.sparse as sp, scipy.sparse.linalg as spla, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2011_11880_b200.batched_newton as bn
from paper_2011_11880_b200 import synth
from paper_2011_11880_b200.plan import Plan
from paper_2011_11880_b200.system_model import build_system, random_state

s = build_system(synth.config_case(0, seed=0)); plan = Plan(s)
n, nnz = plan.n_var, plan.nnz
indptr, indices = plan.pattern_csr()
K = 4
mats = []
for k in range(K):
    y = torch.as_tensor(random_state(s, 10 + k), device="cuda")
    j = plan.empty(nnz); plan.eval(y, jval=j); torch.cuda.synchronize()
    mats.append(sp.csr_matrix((j[:nnz].cpu().numpy(), indices, indptr), shape=(n, n)))
rhs = [np.random.default_rng(k).normal(size=n) for k in range(K)]
ref = [spla.spsolve(m.tocsc(), b) for m, b in zip(mats, rhs)]
t0 = time.time()
lu = bn.BatchedLU(K, indptr, indices, mats[0].tocsc())
print("setup", time.time() - t0, "nnzLU", lu.nnz_lu, flush=True)
for k in range(K):
    lu.vals[k] = torch.as_tensor(mats[k].data, device="cuda")
    lu.rhs[k] = torch.as_tensor(rhs[k], device="cuda")
t0 = time.time(); lu.refactor_solve(); dt = time.time() - t0
err = [float(np.abs(lu.rhs[k].cpu().numpy() - ref[k]).max() / np.abs(ref[k]).max()) for k in range(K)]
print("refactor+solve", dt, "rel err", err, flush=True)
