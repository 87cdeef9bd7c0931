import sys, time, statistics
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2011_11880_b200 import synth
from paper_2011_11880_b200.plan import Plan, pinned_zeros
from paper_2011_11880_b200.system_model import build_system, random_state
s = build_system(synth.config_case(2, seed=2)); plan = Plan(s)
y = random_state(s, 7)
_, g = pinned_zeros(plan.n_var); _, j = pinned_zeros(plan.nnz)
_, yp = pinned_zeros(plan.n_var); yp[:] = y
gpage = np.zeros(plan.n_var); jpage = np.zeros(plan.nnz)
def t(fn, n=50):
    for _ in range(5): fn()
    ts=[]
    for _ in range(n):
        a=time.perf_counter(); fn(); ts.append(time.perf_counter()-a)
    return statistics.median(ts)*1e6
print('y pageable, g+J pinned  ', t(lambda: plan.eval_host(y, g=g, jcsc=j)))
print('y pinned,   g+J pinned  ', t(lambda: plan.eval_host(yp, g=g, jcsc=j)))
print('y pinned,   g only      ', t(lambda: plan.eval_host(yp, g=g)))
print('y pinned,   J only      ', t(lambda: plan.eval_host(yp, jcsc=j)))
print('y pageable, g only      ', t(lambda: plan.eval_host(y, g=g)))
print('y pageable, g+J pageable', t(lambda: plan.eval_host(y, g=gpage, jcsc=jpage)))
# raw copy rates
dj = torch.empty(plan.nnz, dtype=torch.float64, device='cuda'); hj = torch.from_numpy(j)
def d2h(): hj.copy_(dj); 
print('D2H 8MB pinned          ', t(d2h))
dy = torch.empty(plan.n_var, dtype=torch.float64, device='cuda')
print('H2D 1.2MB pageable      ', t(lambda: dy.copy_(torch.from_numpy(y))))
print('H2D 1.2MB pinned        ', t(lambda: dy.copy_(torch.from_numpy(yp))))
