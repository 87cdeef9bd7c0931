import torch
n = 2283*2**20//256  # 256B rows
x = torch.empty(n, 32, dtype=torch.float64, device="cuda")
v = torch.ones(n, 32, dtype=torch.float64, device="cuda")
for name, idx in (("seq", torch.arange(n, device="cuda")), ("rand", torch.randperm(n, device="cuda"))):
    for _ in range(2): x.index_copy_(0, idx, v)
    a,b=torch.cuda.Event(True),torch.cuda.Event(True)
    a.record(); x.index_copy_(0, idx, v); b.record(); torch.cuda.synchronize()
    ms=a.elapsed_time(b); print(name, "index_copy 256B rows", ms, "ms", 2*x.numel()*8/ms/1e6, "GB/s (r+w)")
