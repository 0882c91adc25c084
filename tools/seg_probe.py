"""Time the segment-parallel lanes path against the single-pass kernel.

    python tools/seg_probe.py config4 8192 [16384 ...]   (jitter, device-resident)
    python tools/seg_probe.py config2                     (400 per-layer Shrink)
    python tools/seg_probe.py config3                     (4,000 bucket-order x network)

Each line: workload, S, mode (env), ms per launch (CUDA events, 10 launches
after 3 warm-up), G updates/s, and whether the result equals the other mode.
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import numpy as np
import torch

import bench
from paper_2006_03318_b200 import workloads as W
from paper_2006_03318_b200.batch import ScenarioTable, compile_scale_sweep, simulate_batch_device
from paper_2006_03318_b200.frozen import FrozenGraph
from paper_2006_03318_b200.transform import GPU_TASKS, And, ByLayer

MODES = {"seg": {}, "seqscan": {"DDSIM_SEG_SEQSCAN": "1"}, "single": {"DDSIM_NO_SEG": "1"}}


def timed(fz, table, S, env, reps=10):
    for k, v in env.items():
        os.environ[k] = v
    try:
        st = torch.empty((fz.n, S), dtype=torch.int64, device="cuda:0")
        ms = torch.empty(S, dtype=torch.int64, device="cuda:0")
        lb = torch.empty((S, fz.L), dtype=torch.int64, device="cuda:0")
        stream = torch.cuda.current_stream()
        run = lambda: simulate_batch_device(fz, table, makespan=ms, lane_busy=lb, start=st,
                                            stream=stream.cuda_stream)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            run()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps, st, ms
    finally:
        for k in env:
            os.environ.pop(k, None)


def main():
    what = sys.argv[1]
    extra = {}
    for a in sys.argv[2:]:
        if "=" in a:
            k, v = a.split("=", 1)
            extra[k] = v
    sizes = [int(a) for a in sys.argv[2:] if "=" not in a]
    cases = []
    if what == "config4":
        w, fz = bench.build_workload(0)
        for S in sizes or [8192]:
            cases.append((f"config4", S, fz, ScenarioTable(n_scenarios=S,
                                                          dense=bench.make_jitter_dense(fz, S, 5, 0))))
    elif what == "config2":
        w = W.bert_trace(buckets_mb=None)
        scen = [[(And([GPU_TASKS, ByLayer(l)]), "1/2")] for l in w.layers] + [[]]
        group_of, ptr, steps = compile_scale_sweep(w.graph, scen)
        fz = FrozenGraph.from_graph(w.graph, group_of=group_of)
        cases.append(("config2", len(scen), fz,
                      ScenarioTable(n_scenarios=len(scen), scale_ptr=ptr, scale=steps)))
    elif what == "config3":
        fz, table, _g, _i = bench.build_config(3, 0)
        cases.append(("config3", table.n_scenarios, fz, table))
    for name, S, fz, table in cases:
        out = {}
        for mode, env in MODES.items():
            t, st, ms = timed(fz, table, S, {**env, **extra})
            out[mode] = (t, st.cpu(), ms.cpu())
            print(json.dumps({"workload": name, "S": S, "mode": mode, "env": extra, "ms": round(t, 4),
                              "G_updates_per_s": round(fz.n * S / t / 1e6, 2)}), flush=True)
        same = all(torch.equal(out[m][1], out["single"][1]) and torch.equal(out[m][2], out["single"][2])
                   for m in out)
        print(json.dumps({"workload": name, "S": S, "identical": bool(same),
                          "speedup": round(out["single"][0] / out["seg"][0], 3)}), flush=True)


if __name__ == "__main__":
    main()
