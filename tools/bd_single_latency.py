"""Latency of the single-scenario breakdown (the drop-in Analysis.whatif path:
a one-point table) on the config-1 graph against the number of time windows
(DDSIM_BD_WINDOWS; default: >= 512 rows per window)."""
import os
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2006_03318_b200 import workloads as W  # noqa: E402
from paper_2006_03318_b200.batch import (ScenarioTable, breakdown_batch_device,  # noqa: E402
                                         layer_names_of, simulate_batch_device)
from paper_2006_03318_b200.frozen import FrozenGraph  # noqa: E402

for name, g in (("resnet50 (config 1)", W.resnet50_trace().graph),
                ("gpt 100k (config 4)", W.gpt_trace(seed=0, n_tasks=100_000).graph)):
    fz = FrozenGraph.from_graph(g, device=0)
    S = 1
    tab = ScenarioTable(n_scenarios=S)
    st = torch.empty((fz.n, S), dtype=torch.int64, device="cuda")
    ms = torch.empty(S, dtype=torch.int64, device="cuda")
    simulate_batch_device(fz, tab, makespan=ms, start=st)
    parts = torch.empty((S, 4), dtype=torch.int64, device="cuda")
    names = layer_names_of(fz)
    lbz = torch.empty((len(names), 2, S), dtype=torch.int64, device="cuda")
    ref = None
    for K in ("", "19", "64", "256", "1024"):
        if K:
            os.environ["DDSIM_BD_WINDOWS"] = K
        else:
            os.environ.pop("DDSIM_BD_WINDOWS", None)
        ts = []
        for _ in range(12):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            breakdown_batch_device(fz, tab, start=st, makespan=ms, parts=parts, layer_busy=lbz)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        got = parts.cpu().tolist()
        ref = ref or got
        assert got == ref, (K, got, ref)
        print(f"{name}: windows {K or 'default'}: {statistics.median(ts[2:]) * 1e3:.3f} ms  parts {got[0]}")
