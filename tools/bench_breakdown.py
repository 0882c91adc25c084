"""Batched breakdown (ks_breakdown) throughput on the config-4 workload:
65,536 jittered scenarios x 100k tasks, start matrix resident from the
simulate launch.  Algorithmic bytes per (task, scenario): start 8 + dur 4."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import bench  # noqa: E402
from paper_2006_03318_b200.batch import (ScenarioTable, breakdown_batch_device,  # noqa: E402
                                         layer_names_of, simulate_batch_device)

S = int(os.environ.get("S", 65536))
w, fz = bench.build_workload(0)
rows, L = fz.n, fz.L
base = torch.from_numpy(fz.duration[fz.order].copy()).cuda()
dense = torch.empty((rows, S), dtype=torch.int32, device="cuda")
g = torch.Generator(device="cuda")
g.manual_seed(1)
step = max(1, (1 << 28) // S)
for r0 in range(0, rows, step):
    r1 = min(rows, r0 + step)
    k = torch.randint(900, 1101, (r1 - r0, S), generator=g, device="cuda", dtype=torch.int64)
    dense[r0:r1] = ((2 * base[r0:r1, None] * k + 1000) // 2000).to(torch.int32)
start = torch.empty((rows, S), dtype=torch.int64, device="cuda")
ms = torch.empty(S, dtype=torch.int64, device="cuda")
table = ScenarioTable(n_scenarios=S, dense=dense)
st = torch.cuda.current_stream().cuda_stream
simulate_batch_device(fz, table, makespan=ms, start=start, stream=st)
parts = torch.empty((S, 4), dtype=torch.int64, device="cuda")
names = layer_names_of(fz)
lbz = torch.empty((len(names), 2, S), dtype=torch.int64, device="cuda")
out = {"scenarios": S, "tasks": rows, "lanes": L, "layers": len(names)}
for label, lb in (("parts", None), ("parts+layers", lbz)):
    def call():
        breakdown_batch_device(fz, table, start=start, makespan=ms, parts=parts, layer_busy=lb,
                               stream=st)
    call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        call()
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 3 / 1e3
    out[label] = {"s": t, "updates_per_s": rows * S / t, "GBps_12B": rows * S * 12 / t / 1e9}
# parity spot check of scenario 0 and S-1 against the breakdown oracle
from breakdown_oracle import breakdown as ora  # noqa: E402
P = parts.cpu().numpy()
for s in (0, S - 1):
    col = start[:, s].cpu().numpy()
    d = dense[:, s].cpu().numpy().astype(np.int64)
    gg = w.graph.copy()
    for r in range(rows):
        gg.tasks[int(fz.row_ids[r])].duration = int(d[r])
    st_of = {int(fz.row_ids[r]): int(col[r]) for r in range(rows)}
    want = ora(gg.tasks, st_of, int(ms[s].item()))
    got = P[s].tolist()
    assert got == [want["cpu_only_ns"], want["gpu_only_ns"], want["parallel_ns"], want["idle_ns"]], (s, got, want)
out["checked"] = [0, S - 1]
print(json.dumps(out))
