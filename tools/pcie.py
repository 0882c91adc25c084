"""PCIe copy throughput: contiguous vs 2D-strided (the e2e chunking pattern)."""
import time, torch
rows, S, w = 100_000, 65_536, 3584
h = torch.empty((rows, S), dtype=torch.int64, pin_memory=True)
d = torch.empty((rows, w), dtype=torch.int64, device="cuda")
dc = torch.empty(rows * w, dtype=torch.int64, device="cuda")
hc = torch.empty(rows * w, dtype=torch.int64, pin_memory=True)
def t(fn, n=3):
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / n
gb = rows * w * 8 / 1e9
print("D2H contiguous GB/s", gb / t(lambda: hc.copy_(dc, non_blocking=True)))
print("H2D contiguous GB/s", gb / t(lambda: dc.copy_(hc, non_blocking=True)))
print("D2H 2D strided GB/s", gb / t(lambda: h[:, :w].copy_(d, non_blocking=True)))
print("H2D 2D strided GB/s", gb / t(lambda: d.copy_(h[:, :w], non_blocking=True)))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    with torch.cuda.stream(s1): hc.copy_(dc, non_blocking=True)
    with torch.cuda.stream(s2): dc.copy_(hc, non_blocking=True)
print("duplex (each way) GB/s", gb / t(both))
