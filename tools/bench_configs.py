"""Measure BASELINE configs 1, 2, 3 and 5 (config 4 is bench.py's headline).

    python tools/bench_configs.py [--out profiles/r01_configs.json]

Device times are CUDA events around the batched call with device-resident
inputs/outputs (after warm-up); CPU times are the C oracle port of the
reference algorithm (16 threads) on the same scenarios, or the drop-in
Python path where stated.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from fractions import Fraction
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def dev_time(fn, reps=5, warm=2):
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3  # seconds


def run_table(fz, table, S, device_out=True):
    import torch

    from paper_2006_03318_b200.batch import simulate_batch_device

    ms = torch.empty(S, dtype=torch.int64, device="cuda")
    lb = torch.empty((S, max(fz.L, 1)), dtype=torch.int64, device="cuda")
    st = torch.empty((fz.n, S), dtype=torch.int64, device="cuda")

    def call():
        simulate_batch_device(fz, table, makespan=ms, lane_busy=lb, start=st,
                              stream=torch.cuda.current_stream().cuda_stream)

    t = dev_time(call)
    return t, ms.cpu().numpy()


def config1():
    from oracle import OracleGraph
    from paper_2006_03318_b200 import workloads as W
    from paper_2006_03318_b200.batch import ScenarioTable, compile_scale_sweep
    from paper_2006_03318_b200.frozen import FrozenGraph
    from paper_2006_03318_b200.scenarios import whatif_amp
    from paper_2006_03318_b200.transform import Selector, apply_pipeline

    w = W.resnet50_trace()
    g = w.graph
    amp = whatif_amp(g)
    steps = [(Selector.from_object(s["selector"]), s["factor"]) for s in amp.steps]
    group_of, ptr, sc = compile_scale_sweep(g, [[], steps])
    fz = FrozenGraph.from_graph(g, group_of=group_of)
    t, ms = run_table(fz, ScenarioTable(n_scenarios=2, scale_ptr=ptr, scale=sc), 2)
    # CPU: the reference algorithm on the transformed graphs (C port)
    t0 = time.perf_counter()
    o = [OracleGraph.from_graph(g).simulate("default")[1],
         OracleGraph.from_graph(apply_pipeline(g, amp)).simulate("default")[1]]
    tc = time.perf_counter() - t0
    assert list(ms) == o, (ms, o)
    # drop-in API end to end (device ingest + layers + simulate + amp what-if)
    from paper_2006_03318_b200 import Analysis
    t1 = time.perf_counter()
    rep = Analysis.from_trace(w.trace).whatif("amp")
    t_api = time.perf_counter() - t1
    return {"config": "1 resnet50-like 10k tasks, baseline + AMP", "tasks": fz.n, "scenarios": 2,
            "device_s": t, "updates_per_s": 2 * fz.n / t, "cpu_port_s_incl_pipeline": tc,
            "dropin_analysis_whatif_s": t_api, "makespans_ns": [int(x) for x in ms],
            "predicted_speedup": rep["speedup"], "bound": "latency (S=2)"}


def config2():
    from paper_2006_03318_b200 import workloads as W
    from paper_2006_03318_b200.batch import ScenarioTable, compile_scale_sweep
    from paper_2006_03318_b200.frozen import FrozenGraph
    from paper_2006_03318_b200.transform import GPU_TASKS, And, ByLayer

    w = W.bert_trace(buckets_mb=None)
    g = w.graph
    scen = [[(And([GPU_TASKS, ByLayer(l)]), "1/2")] for l in w.layers]
    group_of, ptr, sc = compile_scale_sweep(g, scen)
    fz = FrozenGraph.from_graph(g, group_of=group_of)
    S = len(scen)
    t, ms = run_table(fz, ScenarioTable(n_scenarios=S, scale_ptr=ptr, scale=sc), S)
    cpu = cpu_check_scale(g, scen, ms, sample=16)
    return {"config": "2 BERT-large-like per-layer Shrink 2x sweep", "tasks": fz.n, "scenarios": S,
            "device_s": t, "updates_per_s": S * fz.n / t, "bytes_per_update": 8,
            "achieved_GBps": S * fz.n * 8 / t / 1e9, **cpu, "bound": "latency (S=400)"}


def cpu_check_scale(g, scen, ms, sample):
    from oracle import OracleGraph
    from paper_2006_03318_b200.transform import scale_durations

    idx = np.linspace(0, len(scen) - 1, sample).astype(int)
    t = 0.0
    for s in idx:
        h = g.copy()
        for sel, f in scen[s]:
            scale_durations(h, sel, Fraction(str(f)))
        og = OracleGraph.from_graph(h)
        t0 = time.perf_counter()
        m = og.simulate("default")[1]
        t += time.perf_counter() - t0
        assert m == ms[s], (s, m, ms[s])
    n = len(g.tasks)
    return {"cpu_port_updates_per_s_1core": sample * n / t, "checked_scenarios": int(sample)}


def config3():
    from oracle import OracleGraph
    from paper_2006_03318_b200 import workloads as W
    from paper_2006_03318_b200.batch import distributed_sweep
    from paper_2006_03318_b200.scenarios import whatif_distributed
    from paper_2006_03318_b200.transform import TransformPipeline, apply_pipeline

    w = W.bert_trace(buckets_mb=25.0)
    g = w.graph
    buckets = w.trace.gradient_buckets
    B = len([b for b in buckets.buckets() if buckets.layers_of_bucket(b)])
    rng = np.random.default_rng(0)
    configs, perms = [], []
    for bw in (1, 5, 10, 25, 50, 100, 200, 400, 800, 1600):
        for workers in (1, 2, 4, 8, 16, 32, 64, 128):
            for _ in range(50):
                configs.append({"bandwidth_gbps": bw, "workers": workers})
                perms.append(rng.permutation(B))
    perms = np.array(perms, np.int16)
    t0 = time.perf_counter()
    sw = distributed_sweep(g, buckets, configs, perms)
    t_compile = time.perf_counter() - t0
    S = len(configs)
    t, ms = run_table(sw.frozen, sw.table, S)
    # spot-check against the reference-equivalent pipelines on the C port
    tc = 0.0
    chk = [0, 1, 777, 1999, 3999]
    for s in chk:
        pipe = whatif_distributed(g, buckets=buckets, **configs[s])
        steps = [pipe.steps[k] for k in perms[s]] if pipe.steps else []
        h = apply_pipeline(g, TransformPipeline(steps=steps))
        og = OracleGraph.from_graph(h)
        t1 = time.perf_counter()
        m = og.simulate("default")[1]
        tc += time.perf_counter() - t1
        assert m == ms[s], (s, m, ms[s])
    n = sw.frozen.n
    return {"config": "3 data-parallel: bandwidth x workers x bucket order", "tasks": n,
            "buckets": B, "scenarios": S, "device_s": t, "updates_per_s": S * n / t,
            "bytes_per_update": 8, "achieved_GBps": S * n * 8 / t / 1e9,
            "table_compile_s": t_compile, "cpu_port_updates_per_s_1core": len(chk) * n / tc,
            "checked_scenarios": len(chk), "bound": "latency (S=4000)"}


def config5(n_records: int):
    """Trace ingest from document TEXT: native reader (host C++, all cores) ->
    device ingest (joins, sync links, gaps) -> device layer mapping ->
    device-resident frozen graph (CSR + topological order)."""
    import os

    import torch

    from paper_2006_03318_b200.columnar import (dump_trace_columns, frozen_from_ingest,
                                                 load_trace_columns)
    from paper_2006_03318_b200.ingest import ingest_arrays, map_layers_arrays
    from paper_2006_03318_b200.workloads import ingest_document_columns

    t0 = time.perf_counter()
    ct0 = ingest_document_columns(n_records, seed=0)
    text = dump_trace_columns(ct0)
    t_gen = time.perf_counter() - t0
    del ct0
    # warm-up of every stage (allocator, CUB plans, NVRTC-free)
    # warm-up at full size (device memory pool growth, CUB plans, host huge pages)
    ct = load_trace_columns(text)
    res = ingest_arrays(ct.cols)
    tag_m, _ = ct.marker_tags()
    map_layers_arrays(ct.cols, res.launcher, ct.m_lane, ct.m_start, ct.m_end, tag_m)
    frozen_from_ingest(ct, res).close()
    del ct, res
    torch.cuda.synchronize()
    stages = {}
    t0 = time.perf_counter()
    ct = load_trace_columns(text)
    stages["parse_s"] = time.perf_counter() - t0
    t1 = time.perf_counter()
    res = ingest_arrays(ct.cols)
    stages["ingest_s"] = time.perf_counter() - t1
    t2 = time.perf_counter()
    tag_m, tags = ct.marker_tags()
    tag = map_layers_arrays(ct.cols, res.launcher, ct.m_lane, ct.m_start, ct.m_end, tag_m)
    stages["layer_map_s"] = time.perf_counter() - t2
    t3 = time.perf_counter()
    fz = frozen_from_ingest(ct, res)
    torch.cuda.synchronize()
    stages["freeze_s"] = time.perf_counter() - t3
    total = time.perf_counter() - t0
    n = ct.n_events
    return {"config": f"5 ingest from JSON text: {n} records, {len(ct.cols.lanes)} lanes, "
                      f"{ct.n_markers} markers",
            "records": n, "json_bytes": len(text), "edges": int(res.edge_src.shape[0]),
            "mapped_events": int((tag >= 0).sum()), "layers": len(tags), **stages,
            "total_s": total, "records_per_s": n / total,
            "parse_GBps": len(text) / stages["parse_s"] / 1e9,
            "device_stages_records_per_s": n / (stages["ingest_s"] + stages["layer_map_s"]),
            "frozen_chained": bool(fz.chained), "frozen_levels": int(fz.info.n_levels),
            "host_threads": os.cpu_count(), "generate_and_dump_s_untimed": t_gen,
            "bytes_per_record": 80,
            "achieved_GBps_algorithmic_device": n * 80 / (stages["ingest_s"] + stages["layer_map_s"]) / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r01_configs.json"))
    ap.add_argument("--ingest-records", type=int, default=10_000_000)
    ap.add_argument("--only", default="1,2,3,5")
    args = ap.parse_args()
    out = {}
    for c in args.only.split(","):
        fn = {"1": config1, "2": config2, "3": config3,
              "5": lambda: config5(args.ingest_records)}[c]
        t0 = time.perf_counter()
        out[c] = fn()
        out[c]["harness_s"] = time.perf_counter() - t0
        print(json.dumps({c: out[c]}), flush=True)
    Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
