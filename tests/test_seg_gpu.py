"""Segment-parallel lanes path (SegParams, csrc/lanes_body.cuh + lanes_seg.cuh):
small scenario counts cut the record stream into K segments, compute each
segment's (max,+) transfer per scenario, compose them, and replay every
segment from its true input.  Results must equal Alg. 1 (sim.py:89-142) --
checked against the C oracle on sampled scenarios, against the single-pass
kernel on the whole matrix, and against the max-plus recurrence on every
(task, scenario) on the device."""

import os

import numpy as np
import pytest

from helpers import check_recurrence_device
from oracle import OracleGraph
from paper_2006_03318_b200 import _native as N
from paper_2006_03318_b200 import workloads as W
from paper_2006_03318_b200.batch import ScenarioTable, compile_scale_sweep, simulate_batch
from paper_2006_03318_b200.frozen import FrozenGraph
from paper_2006_03318_b200.graph import DependencyGraph, EdgeKind, Task
from paper_2006_03318_b200.trace import LaneId, TaskKind
from paper_2006_03318_b200.transform import GPU_TASKS, And, ByLayer, scale_durations

pytestmark = pytest.mark.gpu


def slot_graph(n=4000, lanes=3, seed=0, reach=6):
    """A lane-chained graph whose cross-lane edges often come from a task
    that is no longer its lane's head (shared-memory value slots in the lanes
    program), with short live ranges so segment cuts exist."""
    rng = np.random.default_rng(seed)
    g = DependencyGraph()
    lane_ids = [LaneId.parse("cpu:0")] + [LaneId.parse(f"gpu:0:{7 + k}") for k in range(lanes - 1)]
    lane_of = rng.integers(0, lanes, n)
    order = {ln: [] for ln in lane_ids}
    edges = set()
    for i in range(n):
        ln = lane_ids[lane_of[i]]
        kind = TaskKind.CPU_OTHER if lane_of[i] == 0 else TaskKind.GPU_KERNEL
        g.tasks[i] = Task(id=i, kind=kind, name=f"t{i}", lane=ln,
                          duration=int(rng.integers(1000, 50_000)),
                          gap=int(rng.integers(0, 3000)) if lane_of[i] == 0 else 0)
        if order[ln]:
            edges.add((order[ln][-1], i, EdgeKind.LANE_SEQ_CPU if lane_of[i] == 0
                       else EdgeKind.LANE_SEQ_GPU))
        order[ln].append(i)
        for _ in range(int(rng.integers(0, 3))):
            j = i - int(rng.integers(1, reach))
            if j >= 0 and lane_of[j] != lane_of[i]:
                edges.add((j, i, EdgeKind.INJECTED))
    g.edges = edges
    g.lane_order = {ln: v for ln, v in order.items() if v}
    return g


def _dense(fz, S, seed, lo=900, hi=1101):
    rng = np.random.default_rng(seed)
    base = fz.duration[fz.order]
    return ((2 * base[:, None] * rng.integers(lo, hi, (fz.n, S)) + 1000) // 2000).astype(np.int32)


def _oracle_cols(g, fz, dense, res, cols):
    og = OracleGraph.from_graph(g)
    for s in cols:
        d = np.empty(fz.n, np.int64)
        d[fz.order] = dense[:, s]
        st, ms, lb, _ = og.simulate("default", dur=d)
        assert res.makespan[s] == ms, s
        assert res.start_of(s) == st, s
        assert {str(k): v for k, v in res.lane_busy_of(s).items()} == \
            {str(k): v for k, v in lb.items()}, s


def _plain(fz, table, monkeypatch):
    monkeypatch.setenv("DDSIM_NO_SEG", "1")
    try:
        return simulate_batch(fz, table)
    finally:
        monkeypatch.delenv("DDSIM_NO_SEG")


def _seg_engaged():
    log = (N.lib().ks_jit_log() or b"").decode()
    return "seg_t:" in log or "seg_t2:" in log or "seg_f:" in log


@pytest.mark.parametrize("scan", ["block", "warp", "sequential"])
@pytest.mark.parametrize("S,K", [(1, 40), (5, 600), (16, 1100), (17, 300)])
def test_seg_scan_kernels_many_segments(S, K, scan, monkeypatch):
    """The three compositions of the segment transfers -- one CTA per scenario
    (S <= 16: warp chunks + a scan of the chunk products, several 512-segment
    rounds at K = 600 / 1100), one warp per scenario, one thread per scenario
    -- give the single-pass kernel's result."""
    if scan == "warp":
        monkeypatch.setenv("DDSIM_SEG_WSCAN", "1")
    elif scan == "sequential":
        monkeypatch.setenv("DDSIM_SEG_SEQSCAN", "1")
    g = slot_graph(n=100_000, seed=5, reach=4)
    fz = FrozenGraph.from_graph(g)
    assert fz.info.n_lane_cuts >= 600
    K = min(K, fz.info.n_lane_cuts)
    dense = _dense(fz, S, 11)
    table = ScenarioTable(n_scenarios=S, dense=dense)
    monkeypatch.setenv("DDSIM_SEG_K", str(K))
    res = simulate_batch(fz, table)
    assert _seg_engaged()
    ref = _plain(fz, table, monkeypatch)
    assert np.array_equal(res.start, ref.start)
    assert np.array_equal(res.makespan, ref.makespan)
    assert np.array_equal(res.lane_busy, ref.lane_busy)
    _oracle_cols(g, fz, dense, res, [S - 1])


@pytest.mark.parametrize("passes", ["fused", "3pass"])
@pytest.mark.parametrize("K", ["", "2", "7"])
@pytest.mark.parametrize("S", [1, 96, 333])
def test_seg_slot_graph_vs_oracle_and_single_pass(S, K, passes, monkeypatch):
    """Both segment drivers: the transfer / scan / replay kernels (default)
    and the fused look-back kernel (DDSIM_SEG_FUSED)."""
    if passes == "fused":
        monkeypatch.setenv("DDSIM_SEG_FUSED", "1")
    g = slot_graph()
    fz = FrozenGraph.from_graph(g)
    info = fz.info
    assert info.has_lanes and info.n_lane_slots_smem > 0 and info.n_lane_slots_global == 0
    assert info.n_lane_cuts > 10
    dense = _dense(fz, S, 3)
    table = ScenarioTable(n_scenarios=S, dense=dense)
    if K:
        monkeypatch.setenv("DDSIM_SEG_K", K)
    res = simulate_batch(fz, table)
    assert _seg_engaged()
    ref = _plain(fz, table, monkeypatch)
    assert np.array_equal(res.start, ref.start)
    assert np.array_equal(res.makespan, ref.makespan)
    assert np.array_equal(res.lane_busy, ref.lane_busy)
    _oracle_cols(g, fz, dense, res, sorted({0, S // 2, S - 1}))


def test_seg_config4_strong_shard_full_check():
    """Config 4 as one of 8 strong-scaling shards (8,192 scenarios of the
    100k-task graph): every (task, scenario) against the recurrence, sampled
    scenarios against the oracle."""
    import torch

    import bench
    from paper_2006_03318_b200.batch import simulate_batch_device

    w, fz = bench.build_workload(0)
    S = 8192
    dense = bench.make_jitter_dense(fz, S, 77, 0)
    start = torch.empty((fz.n, S), dtype=torch.int64, device="cuda:0")
    ms = torch.empty(S, dtype=torch.int64, device="cuda:0")
    lb = torch.empty((S, fz.L), dtype=torch.int64, device="cuda:0")
    simulate_batch_device(fz, ScenarioTable(n_scenarios=S, dense=dense), makespan=ms,
                          lane_busy=lb, start=start,
                          stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert _seg_engaged()
    assert bench.oracle_check(w, fz, dense, start, ms, lb, [0, 4097, S - 1]) == [0, 4097, S - 1]
    check_recurrence_device(fz, dense, start, ms, lb)


def test_seg_config2_layer_sweep_vs_oracle(monkeypatch):
    """Config 2 (per-layer Shrink, derived durations expanded on the device)
    through the segment path: equal to the single-pass kernel and the oracle."""
    w = W.bert_trace(buckets_mb=None)
    g = w.graph
    scen = [[(And([GPU_TASKS, ByLayer(l)]), "1/2")] for l in w.layers] + [[]]
    group_of, ptr, steps = compile_scale_sweep(g, scen)
    fz = FrozenGraph.from_graph(g, group_of=group_of)
    table = ScenarioTable(n_scenarios=len(scen), scale_ptr=ptr, scale=steps)
    res = simulate_batch(fz, table)
    assert _seg_engaged()
    ref = _plain(fz, table, monkeypatch)
    assert np.array_equal(res.start, ref.start) and np.array_equal(res.makespan, ref.makespan)
    assert np.array_equal(res.lane_busy, ref.lane_busy)
    from fractions import Fraction
    for s in (0, 211, len(scen) - 1):
        h = g.copy()
        for sel, f in scen[s]:
            scale_durations(h, sel, Fraction(f))
        st, ms, _lb, _ = OracleGraph.from_graph(h).simulate("default")
        assert res.makespan[s] == ms and res.start_of(s) == st


def test_seg_overflow_certificate_reruns_exact(monkeypatch):
    """Durations whose per-segment sums pass 2^30 void the int32 coefficient
    certificate: the device flags the launch and the exact kernel reruns it."""
    g = slot_graph(n=3000, seed=5)
    fz = FrozenGraph.from_graph(g)
    S = 64
    rng = np.random.default_rng(2)
    dense = rng.integers(0, 2**31 - 1, size=(fz.n, S)).astype(np.int32)
    dense[:, : S // 2] //= 1 << 16   # half the scenarios stay small
    res = simulate_batch(fz, ScenarioTable(n_scenarios=S, dense=dense))
    assert _seg_engaged()
    assert int(res.makespan.max()) > 2**31
    _oracle_cols(g, fz, dense, res, [0, S // 2 - 1, S // 2, S - 1])


def test_seg_negative_durations_rerun_exact():
    g = slot_graph(n=3000, seed=6)
    fz = FrozenGraph.from_graph(g)
    S = 40
    rng = np.random.default_rng(4)
    base = fz.duration[fz.order]
    dense = (base[:, None] + rng.integers(-30_000, 3000, size=(fz.n, S))).astype(np.int32)
    res = simulate_batch(fz, ScenarioTable(n_scenarios=S, dense=dense))
    _oracle_cols(g, fz, dense, res, [0, 13, S - 1])


@pytest.mark.parametrize("seed,K", [(1, 6), (2, 17), (3, 40)])
@pytest.mark.parametrize("durations", ["derived", "expanded"])
def test_seg_chain_carries_vs_single_pass_and_oracle(seed, K, durations, monkeypatch):
    """Data-parallel sweeps (one permutable AllReduce chain whose member
    predecessors live through the backward pass) on random training traces:
    the segment path with carries and the chain segment replayed between two
    scans equals the single-pass kernel on every start, makespan and lane busy,
    and sampled scenarios equal the oracle on the reference-equivalent graph."""
    from paper_2006_03318_b200 import transform as TR
    from paper_2006_03318_b200 import workloads as W
    from paper_2006_03318_b200.batch import distributed_sweep
    from paper_2006_03318_b200.scenarios import whatif_distributed

    w = W.training_trace(n_layers=60, kernels_fwd=4, kernels_bwd=8, n_wu=300, n_streams=1,
                         sync_every=200, seed=seed, buckets_mb=8.0)
    g, buckets = w.graph, w.trace.gradient_buckets
    B = len([b for b in buckets.buckets() if buckets.layers_of_bucket(b)])
    rng = np.random.default_rng(seed)
    configs, perms = [], []
    for _ in range(24):
        o = rng.permutation(B)
        for nw in (1, 4, 16):
            for bw in (1, 10, 100):
                configs.append({"bandwidth_gbps": bw, "workers": nw})
                perms.append(o)
    monkeypatch.setenv("DDSIM_FORCE_DERIVED" if durations == "derived" else "DDSIM_NO_DERIVED", "1")
    sw = distributed_sweep(g, buckets, configs, np.array(perms, np.int16))
    assert sw.frozen.info.n_carries > 0
    monkeypatch.setenv("DDSIM_SEG_K", str(K))
    l0 = N.launch_count()
    seg = simulate_batch(sw.frozen, sw.table)
    l1 = N.launch_count()
    monkeypatch.setenv("DDSIM_NO_SEG", "1")
    single = simulate_batch(sw.frozen, sw.table)
    l2 = N.launch_count()
    monkeypatch.delenv("DDSIM_NO_SEG")
    assert (l1 - l0) >= (l2 - l1) + 3  # transfer, two scans, two replays vs one pass
    assert np.array_equal(seg.start, single.start)
    assert np.array_equal(seg.makespan, single.makespan)
    assert np.array_equal(seg.lane_busy, single.lane_busy)
    for s in (1, len(configs) // 2, len(configs) - 1):
        pipe = whatif_distributed(g, buckets=buckets, **configs[s])
        steps = [pipe.steps[k] for k in perms[s]] if pipe.steps else []
        h = g.copy()
        TR._DEFER["on"] = True
        try:
            for stp in steps:
                TR.apply_step(h, stp)
        finally:
            TR._DEFER["on"] = False
        st, ms, _lb, _ = OracleGraph.from_graph(h).simulate("default")
        assert seg.makespan[s] == ms and seg.start_of(s) == st, s
