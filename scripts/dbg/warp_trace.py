import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2011_11880_b200.plan import Plan
from paper_2011_11880_b200 import _abi
for wl in ("config4", "config3"):
    K = bench.WORKLOADS[wl][1]
    s = bench.build_case(wl); plan = Plan(s)
    y, pq_p, pq_q, pv_p, out = bench.blocked_inputs(s, K, 1000)
    t = lambda a: torch.from_numpy(a).cuda()
    dy, dp, dq, dv, do = t(y), t(pq_p), t(pq_q), t(pv_p), t(out)
    g, j, n = plan.empty(plan.n_var, K), plan.empty(plan.nnz, K), plan.empty(K)
    lib = _abi.lib()
    buf = np.zeros(3 * 4096, dtype=np.uint64)
    for _ in range(3):
        plan.eval_batched(K, dy, dp, dq, dv, do, g, j, n)
    lib._lib.pf_debug_warp_trace(ctypes.c_void_p(buf.ctypes.data)) if hasattr(lib, '_lib') else None
    L = ctypes.CDLL(os.environ["PFGPU_LIB"])
    L.pf_debug_warp_trace(ctypes.c_void_p(buf.ctypes.data))
    plan.eval_batched(K, dy, dp, dq, dv, do, g, j, n)
    torch.cuda.synchronize()
    L.pf_debug_warp_trace(ctypes.c_void_p(buf.ctypes.data))
    W = 24; nw = 148 * W
    tot = buf[:nw].astype(np.float64) / 1e3; hub = buf[4096:4096 + nw].astype(np.float64) / 1e3
    nh = buf[8192:8192 + nw]
    print(wl, f"warp total us: mean {tot.mean():.1f} p50 {np.median(tot):.1f} max {tot.max():.1f} min {tot.min():.1f}")
    has = nh > 0
    print(f"  warps with hubs {has.sum()}: total mean {tot[has].mean() if has.any() else 0:.1f} vs without {tot[~has].mean():.1f}; hub items {nh.sum()} time per hub item {hub.sum()/max(nh.sum(),1):.2f} us")
