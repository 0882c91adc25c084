"""Per-step config-4 kernel times (CUDA events around each launch) to see
whether slow windows are isolated steps or whole-process modes."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2006_03318_b200.batch import ScenarioTable, simulate_batch_device  # noqa: E402

torch.cuda.set_device(0)
w, fz = bench.build_workload(0)
S = bench.S_PER_GPU
rows, L = fz.n, fz.L
base = torch.from_numpy(fz.duration[fz.order].copy()).cuda()
dense = torch.empty((rows, S), dtype=torch.int32, device="cuda")
g = torch.Generator(device="cuda")
g.manual_seed(1000)
step_rows = max(1, (1 << 28) // S)
for r0 in range(0, rows, step_rows):
    r1 = min(rows, r0 + step_rows)
    k = torch.randint(900, 1101, (r1 - r0, S), generator=g, device="cuda", dtype=torch.int64)
    dense[r0:r1] = ((2 * base[r0:r1, None] * k + 1000) // 2000).to(torch.int32)
start = torch.empty((rows, S), dtype=torch.int64, device="cuda")
ms = torch.empty(S, dtype=torch.int64, device="cuda")
lb = torch.empty((S, L), dtype=torch.int64, device="cuda")
table = ScenarioTable(n_scenarios=S, dense=dense)
st = torch.cuda.current_stream().cuda_stream
n = 40
ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
for _ in range(3):
    simulate_batch_device(fz, table, makespan=ms, lane_busy=lb, start=start, stream=st)
torch.cuda.synchronize()
ev[0].record()
for i in range(n):
    simulate_batch_device(fz, table, makespan=ms, lane_busy=lb, start=start, stream=st)
    ev[i + 1].record()
torch.cuda.synchronize()
print(" ".join(f"{ev[i].elapsed_time(ev[i + 1]):.1f}" for i in range(n)), flush=True)
