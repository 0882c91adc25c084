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
