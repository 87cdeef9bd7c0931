import sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "tests"))
from _util import load, system_of, csc_to_csr_perm
from paper_2011_11880_b200.plan import Plan
d = load("edge300"); s = system_of(d); plan = Plan(s)
to_csr = csc_to_csr_perm(d["csc_indptr"], d["csc_indices"], d["csr_indptr"], d["csr_indices"])
y = torch.as_tensor(d["ys"][0], device="cuda")
j = torch.full((plan.nnz,), -777.0, dtype=torch.float64, device="cuda")
g = plan.empty(plan.n_var); n = plan.empty(1)
plan.eval(y, g, j, n); torch.cuda.synchronize()
J = j.cpu().numpy(); R = d["j_wf1"][0][to_csr]
ip, ix = d["csr_indptr"], d["csr_indices"]
rows = np.repeat(np.arange(len(ip) - 1), np.diff(ip))
bad = np.nonzero(~(np.abs(J - R) <= np.maximum(1e-12 * np.abs(R), 1e-14)))[0]
N = s.n_bus
print("N", N, "L", len(s.lines.bus_h), "bad", len(bad))
bh, bk = s.lines.bus_h, s.lines.bus_k
for b in bad[:40]:
    r, c = rows[b], ix[b]
    bus = r % N if r < 2 * N else -1
    nb_ = c % N if c < 2 * N else -1
    cnt = np.sum(((bh == bus) & (bk == nb_)) | ((bh == nb_) & (bk == bus)))
    print(f"pos {b} row {r} col {c} bus {bus} nbr {nb_} got {J[b]} ref {R[b]} parallel {cnt} deg {np.sum(bh==bus)+np.sum(bk==bus)}")
