"""BASELINE configs at their full graph sizes (the bench's own workloads),
spot-checked scenario by scenario against the C oracle (Alg. 1, sim.py:89-142)
plus size-independent properties over every scenario:

* config 4: 100k-task GPT-style graph, 2,048 jitter scenarios (bench uses 65,536);
  exact for sampled scenarios; for all: makespan >= every lane busy total and
  makespan == max over rows of start + duration (gap excluded, sim.py:125);
* config 2: 400 per-layer Shrink scenarios on the 30k-task BERT-like graph;
  shrinking never lengthens a lane-chained schedule (monotone max-plus);
* config 3: 4,000 bandwidth x workers x bucket-order scenarios; workers == 1
  equals the baseline (scenarios.py:197-199) and makespan is non-increasing in
  bandwidth for a fixed worker count and bucket order.
"""

from fractions import Fraction

import numpy as np
import pytest

from oracle import OracleGraph
from paper_2006_03318_b200 import workloads as W
from paper_2006_03318_b200.batch import (ScenarioTable, compile_scale_sweep, distributed_sweep,
                                         simulate_batch)
from paper_2006_03318_b200.frozen import FrozenGraph
from paper_2006_03318_b200.scenarios import whatif_distributed
from paper_2006_03318_b200.transform import (GPU_TASKS, And, ByLayer, TransformPipeline,
                                             apply_pipeline, scale_durations)

pytestmark = pytest.mark.gpu


def test_config4_full_graph():
    w = W.gpt_trace(seed=0, n_tasks=100_000)
    fz = FrozenGraph.from_graph(w.graph)
    assert fz.chained and fz.n >= 99_000
    S = 2048
    base = fz.duration[fz.order]
    rng = np.random.default_rng(11)
    k = rng.integers(900, 1101, size=(fz.n, S))
    dense = ((2 * base[:, None] * k + 1000) // 2000).astype(np.int32)
    res = simulate_batch(fz, ScenarioTable(n_scenarios=S, dense=dense))
    og = OracleGraph.from_graph(w.graph)
    for s in (0, 777, S - 1):
        d = np.empty(fz.n, np.int64)
        d[fz.order] = dense[:, s]
        st, ms, lb, _ = og.simulate("default", dur=d)
        assert res.makespan[s] == ms
        assert res.start_of(s) == st
    # properties over every scenario
    fin = res.start + dense.astype(np.int64)
    assert np.array_equal(res.makespan, fin.max(axis=0))
    assert np.all(res.makespan[:, None] >= res.lane_busy)
    assert np.array_equal(res.lane_busy.sum(axis=1), dense.astype(np.int64).sum(axis=0))


@pytest.mark.parametrize("durations", ["expanded", "expanded64", "derived"])
def test_config2_full_sweep(durations, monkeypatch):
    monkeypatch.setenv("DDSIM_FORCE_DERIVED" if durations == "derived" else "DDSIM_NO_DERIVED", "1")
    if durations == "expanded64":  # int64 matrix (default: int32, the durations fit)
        monkeypatch.setenv("DDSIM_EXPAND64", "1")
    w = W.bert_trace(buckets_mb=None)
    g = w.graph
    scen = [[(And([GPU_TASKS, ByLayer(l)]), "1/2")] for l in w.layers]
    group_of, ptr, steps = compile_scale_sweep(g, scen + [[]])
    fz = FrozenGraph.from_graph(g, group_of=group_of)
    S = len(scen) + 1
    res = simulate_batch(fz, ScenarioTable(n_scenarios=S, scale_ptr=ptr, scale=steps))
    base = int(res.makespan[-1])
    assert np.all(res.makespan[:-1] <= base)          # shrinking never hurts
    for s in (0, len(scen) // 2, len(scen) - 1):
        h = g.copy()
        for sel, f in scen[s]:
            scale_durations(h, sel, Fraction(f))
        st, ms, _lb, _ = OracleGraph.from_graph(h).simulate("default")
        assert res.makespan[s] == ms and res.start_of(s) == st


@pytest.mark.parametrize("durations", ["expanded", "derived"])
def test_config3_full_sweep(durations, monkeypatch):
    monkeypatch.setenv("DDSIM_FORCE_DERIVED" if durations == "derived" else "DDSIM_NO_DERIVED", "1")
    w = W.bert_trace(buckets_mb=25.0)
    g = w.graph
    buckets = w.trace.gradient_buckets
    B = len([b for b in buckets.buckets() if buckets.layers_of_bucket(b)])
    bws = (1, 5, 10, 25, 50, 100, 200, 400, 800, 1600)
    workers = (1, 2, 4, 8, 16, 32, 64, 128)
    rng = np.random.default_rng(0)
    orders = [rng.permutation(B) for _ in range(50)]
    configs, perms = [], []
    for o in orders:
        for nw in workers:
            for bw in bws:
                configs.append({"bandwidth_gbps": bw, "workers": nw})
                perms.append(o)
    sw = distributed_sweep(g, buckets, configs, np.array(perms, np.int16))
    res = simulate_batch(sw.frozen, sw.table)
    ms = res.makespan.reshape(len(orders), len(workers), len(bws))
    baseline = OracleGraph.from_graph(g).simulate("default")[1]
    assert np.all(ms[:, 0, :] == baseline)              # one worker: no allreduce inserted
    assert np.all(np.diff(ms, axis=2) <= 0)             # more bandwidth never hurts
    for s in (1, 1234, len(configs) - 1):
        pipe = whatif_distributed(g, buckets=buckets, **configs[s])
        steps = [pipe.steps[k] for k in perms[s]] if pipe.steps else []
        h = apply_pipeline(g, TransformPipeline(steps=steps))
        st, m, _lb, _ = OracleGraph.from_graph(h).simulate("default")
        assert res.makespan[s] == m and res.start_of(s) == st


def test_config4_bench_variant_vs_oracle():
    """The exact launch the config-4 bench times: 65,536 scenarios, int32
    jitter durations from bench.make_jitter_dense, default environment (V = 2
    scenarios per thread, NVRTC if-chain handler, global spill slots).  Five
    scenarios against the C oracle's Alg. 1 (every start, makespan, lane busy)
    and every (task, scenario) against the max-plus recurrence on the device."""
    import os

    import torch

    import bench
    from helpers import check_recurrence_device
    from paper_2006_03318_b200 import _native as N
    from paper_2006_03318_b200.batch import simulate_batch_device

    for k in ("DDSIM_LANES_V", "DDSIM_LANES_DYN", "DDSIM_NO_JIT", "DDSIM_NO_LANES"):
        assert k not in os.environ, k
    w, fz = bench.build_workload(0)
    S = bench.S_PER_GPU
    dense = bench.make_jitter_dense(fz, S, 1000, 0)
    start = torch.empty((fz.n, S), dtype=torch.int64, device="cuda:0")
    ms = torch.empty(S, dtype=torch.int64, device="cuda:0")
    lb = torch.empty((S, fz.L), dtype=torch.int64, device="cuda:0")
    simulate_batch_device(fz, ScenarioTable(n_scenarios=S, dense=dense), makespan=ms,
                          lane_busy=lb, start=start,
                          stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    log = (N.lib().ks_jit_log() or b"").decode()
    assert "compiled 0:1:2:" in log, log        # device 0, int32 tiles, V = 2, if-chain
    assert fz.info.n_slots > fz.info.n_slots_smem  # global spill slots in use
    cols = [0, 1, 18_945, S // 2 + 1, S - 1]
    assert bench.oracle_check(w, fz, dense, start, ms, lb, cols) == cols
    check_recurrence_device(fz, dense, start, ms, lb)


def test_config1_full_baseline_and_amp():
    """Config 1 at its bench size: the ~10k-task ResNet-50-like iteration,
    baseline + AMP (whatif_amp, scenarios.py:141-149) in one launch; every
    start time, makespan and lane busy of both scenarios against the oracle
    on the reference-equivalent transformed graph."""
    from paper_2006_03318_b200.scenarios import whatif_amp
    from paper_2006_03318_b200.transform import Selector

    w = W.resnet50_trace()
    g = w.graph
    amp = whatif_amp(g)
    scen = [[], [(Selector.from_object(x["selector"]), x["factor"]) for x in amp.steps]]
    group_of, ptr, steps = compile_scale_sweep(g, scen)
    fz = FrozenGraph.from_graph(g, group_of=group_of)
    assert fz.n >= 9_000
    res = simulate_batch(fz, ScenarioTable(n_scenarios=2, scale_ptr=ptr, scale=steps))
    amp_graph = apply_pipeline(g, amp)
    for s, h in enumerate((g, amp_graph)):
        st, ms, lb, _ = OracleGraph.from_graph(h).simulate("default")
        assert res.makespan[s] == ms, s
        assert res.start_of(s) == st, s
        assert {str(k): v for k, v in res.lane_busy_of(s).items()} == \
            {str(k): v for k, v in lb.items()}, s
    assert res.makespan[1] < res.makespan[0]
