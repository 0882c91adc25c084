"""Config-4 kernel time vs memory placement: a padding allocation of
0..N GB before the duration / start matrices shifts where they land."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2006_03318_b200.batch import ScenarioTable, simulate_batch_device  # noqa: E402

torch.cuda.set_device(0)
w, fz = bench.build_workload(0)
S = bench.S_PER_GPU
rows, L = fz.n, fz.L
base = torch.from_numpy(fz.duration[fz.order].copy()).cuda()
st = torch.cuda.current_stream().cuda_stream
ms = torch.empty(S, dtype=torch.int64, device="cuda")
lb = torch.empty((S, L), dtype=torch.int64, device="cuda")
for pad_mb in [0, 2, 64, 1024, 3 * 1024 + 2, 10 * 1024 + 6, 0, 2]:
    pad = torch.empty(pad_mb * (1 << 20) // 8 + 1, dtype=torch.int64, device="cuda")
    dense = torch.randint(900, 1101, (rows, S), dtype=torch.int32, device="cuda")
    start = torch.empty((rows, S), dtype=torch.int64, device="cuda")
    table = ScenarioTable(n_scenarios=S, dense=dense)

    def step():
        simulate_batch_device(fz, table, makespan=ms, lane_busy=lb, start=start, stream=st)
    step()
    torch.cuda.synchronize()
    res = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            step()
        b.record()
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / 5)
    print(f"pad {pad_mb:6d} MB dense@{dense.data_ptr() % (1 << 30):#x} start@{start.data_ptr() % (1 << 30):#x}: "
          f"{' '.join('%.2f' % x for x in res)} ms", flush=True)
    del pad, dense, start, table
    torch.cuda.empty_cache()
