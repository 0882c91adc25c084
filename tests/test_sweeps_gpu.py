"""Batched sweep tables (BASELINE configs 2 and 3) against the C oracle run on
the equivalent reference pipelines, scenario by scenario."""

import numpy as np
import pytest

from oracle import OracleGraph
from paper_2006_03318_b200 import workloads as W
from paper_2006_03318_b200.batch import (ScenarioTable, compile_scale_sweep, distributed_sweep,
                                         simulate_batch)
from paper_2006_03318_b200.frozen import FrozenGraph
from paper_2006_03318_b200.scenarios import whatif_distributed
from paper_2006_03318_b200.trace import Phase
from paper_2006_03318_b200.transform import GPU_TASKS, And, ByLayer, TransformPipeline, apply_pipeline

pytestmark = pytest.mark.gpu


def _small_training(seed=3, buckets_mb=6.0):
    return W.training_trace(n_layers=24, kernels_fwd=3, kernels_bwd=5, n_wu=40, n_streams=1,
                            sync_every=60, seed=seed, buckets_mb=buckets_mb)


@pytest.mark.parametrize("mode", ["expand+lanes", "general"])
def test_per_layer_shrink_sweep_vs_oracle(mode, monkeypatch):
    if mode == "general":
        monkeypatch.setenv("DDSIM_NO_EXPAND", "1")
    w = _small_training()
    g = w.graph
    scen = [[(And([GPU_TASKS, ByLayer(l)]), "1/2")] for l in w.layers] + [[]]
    group_of, ptr, steps = compile_scale_sweep(g, scen)
    fz = FrozenGraph.from_graph(g, group_of=group_of)
    res = simulate_batch(fz, ScenarioTable(n_scenarios=len(scen), scale_ptr=ptr, scale=steps))
    for s in range(0, len(scen), 5):
        steps_s = [{"op": "scale", "selector": sel.to_object(), "factor": f} for sel, f in scen[s]]
        h = apply_pipeline(g, TransformPipeline(steps=steps_s))
        st, ms, lb, _ = OracleGraph.from_graph(h).simulate("default")
        assert res.makespan[s] == ms, s
        assert res.start_of(s) == st, s
        assert {str(k): v for k, v in res.lane_busy_of(s).items()} == {str(k): v for k, v in lb.items()}


def test_distributed_sweep_vs_oracle():
    w = _small_training()
    g = w.graph
    buckets = w.trace.gradient_buckets
    configs = []
    for bw in ("1", "10", "2.5", "400"):
        for workers in (1, 2, 8):
            configs.append({"bandwidth_gbps": bw, "workers": workers, "latency_us": "1.5"})
    rng = np.random.default_rng(0)
    B = len([b for b in buckets.buckets() if buckets.layers_of_bucket(b)])
    assert B >= 3
    perms = np.stack([rng.permutation(B) for _ in configs]).astype(np.int16)
    sw = distributed_sweep(g, buckets, configs, perms)
    res = simulate_batch(sw.frozen, sw.table)
    for s, cfg in enumerate(configs):
        pipe = whatif_distributed(g, buckets=buckets, **cfg)
        steps = [pipe.steps[k] for k in perms[s]] if pipe.steps else []
        h = apply_pipeline(g, TransformPipeline(steps=steps))
        st, ms, lb, _ = OracleGraph.from_graph(h).simulate("default")
        assert res.makespan[s] == ms, (s, cfg)
        assert res.start_of(s) == st, (s, cfg)
        present = set(range(len(sw.frozen.lanes)))
        got = {str(k): v for k, v in res.lane_busy_of(s).items() if v or str(k) in
               {str(x) for x in lb}}
        assert got == {str(k): v for k, v in lb.items()}, (s, cfg)


def test_distributed_sweep_reorders_change_makespan():
    w = _small_training(seed=5, buckets_mb=3.0)
    buckets = w.trace.gradient_buckets
    B = len([b for b in buckets.buckets() if buckets.layers_of_bucket(b)])
    cfg = {"bandwidth_gbps": "1", "workers": 8}
    perms = np.stack([np.arange(B), np.arange(B)[::-1]]).astype(np.int16)
    sw = distributed_sweep(w.graph, buckets, [cfg, cfg], perms)
    res = simulate_batch(sw.frozen, sw.table)
    assert res.makespan[0] > 0 and res.makespan[1] > 0


def test_removal_steps_vs_remove_task():
    """KS_STEP_REMOVE scenarios (batched remove_task, transform.py:249-265)
    against the oracle on graphs where remove_task was applied structurally:
    layer removals, kind removals, a whole lane removed, removal mixed with
    Shrink."""
    from paper_2006_03318_b200.batch import REMOVE
    from paper_2006_03318_b200.trace import TaskKind
    from paper_2006_03318_b200.transform import ByKind, ByLane, LaneClass, Not
    w = _small_training(seed=11)
    g = w.graph
    mem = ByKind(TaskKind.GPU_MEMCPY)
    scen = [[], [(ByLayer(w.layers[3]), REMOVE)], [(And([GPU_TASKS, ByLayer(w.layers[7])]), REMOVE)],
            [(mem, REMOVE)], [(ByLane(LaneClass.GPU_STREAM), REMOVE)],
            [(GPU_TASKS, "1/2"), (ByLayer(w.layers[1]), REMOVE), (GPU_TASKS, "3/2")],
            [(ByKind(TaskKind.SYNC), REMOVE), (ByLayer(w.layers[2]), "0.25")],
            [(And([ByLayer(w.layers[5]), Not(GPU_TASKS)]), REMOVE)]]
    group_of, ptr, steps = compile_scale_sweep(g, scen)
    fz = FrozenGraph.from_graph(g, group_of=group_of)
    res = simulate_batch(fz, ScenarioTable(n_scenarios=len(scen), scale_ptr=ptr, scale=steps))
    for s, sc in enumerate(scen):
        pipe = [{"op": "remove", "selector": sel.to_object()} if f == REMOVE else
                {"op": "scale", "selector": sel.to_object(), "factor": f} for sel, f in sc]
        h = apply_pipeline(g, TransformPipeline(steps=pipe))
        st, ms, lb, _ = OracleGraph.from_graph(h).simulate("default")
        assert res.makespan[s] == ms, s
        assert res.start_of(s) == st, s
        assert {str(k): v for k, v in res.lane_busy_of(s).items()} == {str(k): v for k, v in lb.items()}, s


def test_removal_inside_permutable_chain():
    """Removing chain members (inserted allReduces) per scenario: equals the
    reference's sequenced inserts in perm order followed by remove_task."""
    from paper_2006_03318_b200.batch import REMOVE  # noqa: F401  (num=den=0 steps)
    from paper_2006_03318_b200 import _native as N
    from paper_2006_03318_b200.comm import COLLECTIVE_LANE, earliest_weight_update_task
    from paper_2006_03318_b200.comm import last_backward_gpu_task
    from paper_2006_03318_b200.frozen import ChainSpec
    from paper_2006_03318_b200.graph import EdgeKind, Task
    from paper_2006_03318_b200.trace import TaskKind
    from paper_2006_03318_b200.transform import remove_task
    w = _small_training(seed=5)
    g = w.graph.copy()
    wu = earliest_weight_update_task(g)
    head_order = list(g.lane_order.get(COLLECTIVE_LANE, []))
    nid = g.next_id()
    members = []
    for k, layer in enumerate(w.layers[:5]):
        tid = nid + k
        g.tasks[tid] = Task(id=tid, kind=TaskKind.COMM, name=f"ar{k}", lane=COLLECTIVE_LANE,
                            duration=1000 * (k + 1), gap=7 * k)
        g.edges.add((last_backward_gpu_task(w.graph, layer).id, tid, EdgeKind.INJECTED))
        g.edges.add((tid, wu.id, EdgeKind.INJECTED))
        members.append(tid)
    group_of = np.zeros(len(g.tasks), np.uint32)
    ids = list(g.tasks)
    for k, tid in enumerate(members):
        group_of[ids.index(tid)] = k + 1
    fz = FrozenGraph.from_graph(g, group_of=group_of, chains=[ChainSpec(members=members, head=head_order[-1] if head_order else None)])
    rng = np.random.default_rng(1)
    S = 12
    perms = np.array([rng.permutation(5) for _ in range(S)], np.int16)
    removed = [sorted(rng.choice(5, size=rng.integers(0, 4), replace=False).tolist())
               for _ in range(S)]
    removed[0], removed[1] = [], [0, 1, 2, 3, 4]
    ptr, steps = [0], []
    for rm in removed:
        steps += [(k + 1, k + 1, 0, 0) for k in rm]
        ptr.append(len(steps))
    arr = np.zeros(max(len(steps), 1), N.SCALE_STEP_DTYPE)
    for i, st in enumerate(steps):
        arr[i] = st
    res = simulate_batch(fz, ScenarioTable(n_scenarios=S, scale_ptr=np.array(ptr, np.int32),
                                           scale=arr[:len(steps)], chain_perm=perms))
    for s in range(S):
        h = g.copy()
        order = head_order + [members[k] for k in perms[s]]
        h.lane_order[COLLECTIVE_LANE] = list(order)
        for a, b in zip(order, order[1:]):
            h.edges.add((a, b, EdgeKind.COMM_ORDER))
        for k in removed[s]:
            remove_task(h, members[k])
        st, ms, lb, _ = OracleGraph.from_graph(h).simulate("default")
        assert res.makespan[s] == ms, s
        assert res.start_of(s) == st, s
        assert {str(k): v for k, v in res.lane_busy_of(s).items()} == {str(k): v for k, v in lb.items()}, s


@pytest.mark.parametrize("S", [1, 7, 64])
def test_multi_device_shards_match_single(S):
    """simulate_batch(devices=...) (ks_simulate_host_multi): contiguous
    scenario shards per device (two shards on device 0 here -- one GPU per
    box) give exactly the single-call results, for dense jitter, scale
    programs and the inserted-task table."""
    w = _small_training()
    g = w.graph
    fz = FrozenGraph.from_graph(g)
    rng = np.random.default_rng(S)
    base = fz.duration[fz.order]
    dense = ((2 * base[:, None] * rng.integers(900, 1101, (fz.n, S)) + 1000) // 2000).astype(np.int32)
    tabs = [(fz, ScenarioTable(n_scenarios=S, dense=dense))]
    scen = [[(And([GPU_TASKS, ByLayer(w.layers[s % len(w.layers)])]), "1/2")] for s in range(S)]
    group_of, ptr, steps = compile_scale_sweep(g, scen)
    fz2 = FrozenGraph.from_graph(g, group_of=group_of)
    tabs.append((fz2, ScenarioTable(n_scenarios=S, scale_ptr=ptr, scale=steps)))
    buckets = w.trace.gradient_buckets
    B = len([b for b in buckets.buckets() if buckets.layers_of_bucket(b)])
    cfgs = [{"bandwidth_gbps": bw, "workers": 1 + s % 4} for s, bw in
            zip(range(S), np.tile([1, 10, 40], S))]
    perms = np.stack([rng.permutation(B) for _ in range(S)]).astype(np.int16)
    sw = distributed_sweep(g, buckets, cfgs, perms)
    tabs.append((sw.frozen, sw.table))
    for f, t in tabs:
        one = simulate_batch(f, t)
        two = simulate_batch(f, t, devices=[0, 0])
        assert np.array_equal(one.makespan, two.makespan)
        assert np.array_equal(one.lane_busy, two.lane_busy)
        assert np.array_equal(one.start, two.start)
