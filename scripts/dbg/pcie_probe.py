import torch, time
n = 1 << 28  # 2 GB fp64
d = torch.empty(n, dtype=torch.float64, device='cuda')
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
for name, f in [("D2H", lambda: h.copy_(d, non_blocking=True)), ("H2D", lambda: d.copy_(h, non_blocking=True))]:
    for _ in range(2): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); f(); b.record(); torch.cuda.synchronize()
    print(name, n * 8 / a.elapsed_time(b) / 1e6, "GB/s")
# chunked D2H on 4 streams
ss = [torch.cuda.Stream() for _ in range(4)]
ch = n // 16
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(16):
    with torch.cuda.stream(ss[i % 4]):
        h[i*ch:(i+1)*ch].copy_(d[i*ch:(i+1)*ch], non_blocking=True)
torch.cuda.synchronize()
print("D2H 4 streams", n * 8 / (time.perf_counter() - t0) / 1e9, "GB/s")
# simultaneous: D2H of 2 GB and H2D of 0.5 GB on two streams
h2 = torch.empty(n // 4, dtype=torch.float64, pin_memory=True)
d2 = torch.empty(n // 4, dtype=torch.float64, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
e = [torch.cuda.Event(True) for _ in range(4)]
with torch.cuda.stream(s1):
    e[0].record(); h.copy_(d, non_blocking=True); e[1].record()
with torch.cuda.stream(s2):
    e[2].record(); d2.copy_(h2, non_blocking=True); e[3].record()
torch.cuda.synchronize()
print("concurrent: D2H", n * 8 / e[0].elapsed_time(e[1]) / 1e6, "GB/s; H2D", n * 2 / e[2].elapsed_time(e[3]) / 1e6, "GB/s")
# D2H in 64 MB pieces back to back on one stream
torch.cuda.synchronize()
a, b = torch.cuda.Event(True), torch.cuda.Event(True)
pc = 1 << 23
a.record()
for i in range(0, n, pc):
    h[i:i + pc].copy_(d[i:i + pc], non_blocking=True)
b.record(); torch.cuda.synchronize()
print("D2H 64MB pieces", n * 8 / a.elapsed_time(b) / 1e6, "GB/s")
