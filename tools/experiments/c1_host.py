"""Config 1 host overhead: wall time per simulate_batch_device call without /
with synchronisation, device time per call, and a cProfile of the Python side."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

import bench
from paper_2006_03318_b200.batch import simulate_batch_device

fz, table, _g, _i = bench.build_config(1, 0)
S, n, L = table.n_scenarios, fz.n, fz.L
st = torch.empty((n, S), dtype=torch.int64, device="cuda:0")
ms = torch.empty(S, dtype=torch.int64, device="cuda:0")
lb = torch.empty((S, max(L, 1)), dtype=torch.int64, device="cuda:0")
stream = torch.cuda.current_stream()


def step():
    simulate_batch_device(fz, table, makespan=ms, lane_busy=lb, start=st, stream=stream.cuda_stream)


for _ in range(20):
    step()
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for _ in range(N):
    step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host per call {1e6 * (t1 - t0) / N:.1f} us, incl drain {1e6 * (t2 - t0) / N:.1f} us")
t0 = time.perf_counter()
for _ in range(N):
    step()
    stream.synchronize()
print(f"synchronous per call {1e6 * (time.perf_counter() - t0) / N:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    step()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)

# the API calls of one call, recorded with this package's own CUPTI collector
from paper_2006_03318_b200 import cupti  # noqa: E402

with cupti.record() as rec:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
ct = rec.trace
c = ct.cols
names = [ct.names[i] for i in ct.name_id]
lanes = [str(c.lanes[i]) for i in c.lane]
rows = sorted(range(c.n), key=lambda i: c.start[i])
third = [i for i in rows if lanes[i].startswith("cpu")]
k = len(third) // 3
for i in third[-k:]:
    print(f"{c.start[i] / 1e3:10.1f} us {c.duration[i] / 1e3:7.1f} us  {names[i]}")
gpu = [i for i in rows if lanes[i].startswith("gpu")]
for i in gpu[-len(gpu) // 3:]:
    print(f"GPU {c.start[i] / 1e3:10.1f} us {c.duration[i] / 1e3:7.1f} us  {names[i][:60]}")
