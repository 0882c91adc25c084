"""Breakdown time of a bench config's sweep (parts only / with per-layer busy)
against the windowed merge's window count (DDSIM_BD_WINDOWS)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2006_03318_b200.batch import (breakdown_batch_device, layer_names_of,  # noqa: E402
                                         simulate_batch_device)

c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
fz, table, graph_of, info = bench.build_config(c, 0)
S = table.n_scenarios
st = torch.empty((fz.n, S), dtype=torch.int64, device="cuda")
ms = torch.empty(S, dtype=torch.int64, device="cuda")
simulate_batch_device(fz, table, makespan=ms, start=st)
parts = torch.empty((S, 4), dtype=torch.int64, device="cuda")
names = layer_names_of(fz)
lbz = torch.empty((len(names), 2, S), dtype=torch.int64, device="cuda")
print("config", c, "S", S, "rows", fz.n, "lanes", fz.L, "chains", fz.info.n_chains if hasattr(fz.info, "n_chains") else "?")
for K in ("", "16", "57", "152", "400"):
    if K:
        os.environ["DDSIM_BD_WINDOWS"] = K
    else:
        os.environ.pop("DDSIM_BD_WINDOWS", None)
    for label, lb in (("parts", None), ("parts+layers", lbz)):
        def call():
            breakdown_batch_device(fz, table, start=st, makespan=ms, parts=parts, layer_busy=lb)
        call()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            call()
        b.record()
        torch.cuda.synchronize()
        print(f"windows {K or 'auto'} {label}: {a.elapsed_time(b) / 5:.3f} ms")
