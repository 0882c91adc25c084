"""Batched runtime breakdown on the device (ks_breakdown) against the
reference's own reports (golden whatif records) and the breakdown oracle
(oracle/breakdown_oracle.py, a restatement of breakdown.py:42-111) on
transformed graphs: Shrink / remove sweeps, inserted-allReduce chains with
per-scenario order, and every compute_breakdown keyword."""

import itertools
import random

import numpy as np
import pytest

from breakdown_oracle import breakdown as ora_breakdown
from helpers import graph_from_obj
from oracle import OracleGraph
from paper_2006_03318_b200 import build_graph, generate_synthetic_trace
from paper_2006_03318_b200 import workloads as W
from paper_2006_03318_b200.batch import (REMOVE, ScenarioTable, compile_scale_sweep,
                                         distributed_sweep, simulate_batch)
from paper_2006_03318_b200.frozen import FrozenGraph
from paper_2006_03318_b200.scenarios import whatif_distributed
from paper_2006_03318_b200.transform import (GPU_TASKS, And, ByLayer, TransformPipeline,
                                             apply_pipeline)
from randspec import make_spec

pytestmark = pytest.mark.gpu

# merge kernels: auto choice, the row-order streaming sweep forced (full FIFO,
# and a one-run FIFO that hands most scenarios back to the windowed merge),
# and the windowed merge alone
SWEEP_MODES = {"auto": {}, "sweep": {"DDSIM_BD_SWEEP": "1"},
               "sweep_depth1": {"DDSIM_BD_SWEEP": "1", "DDSIM_BD_SWEEP_DEPTH": "1"},
               "windowed": {"DDSIM_BD_SWEEP": "-1"}}


@pytest.fixture(params=list(SWEEP_MODES))
def bd_mode(request, monkeypatch):
    for k, v in SWEEP_MODES[request.param].items():
        monkeypatch.setenv(k, v)
    return request.param


def test_breakdown_matches_reference_reports(golden, bd_mode):
    n = 0
    for rec in golden["whatif"]:
        if "graph" not in rec or "error" in rec.get("sim", {}):
            continue
        g = graph_from_obj(rec["graph"])
        fz = FrozenGraph.from_graph(g)
        if not fz.chained:
            continue
        res = simulate_batch(fz, ScenarioTable(n_scenarios=1), breakdown=True)
        assert res.makespan[0] == rec["sim"]["makespan"]
        assert res.breakdown_of(0).to_object() == rec["report"]["predicted_breakdown"], (
            rec["case"], rec["scenario"])
        n += 1
    assert n >= 15


@pytest.mark.parametrize("opts", list(itertools.product([True, False], repeat=3)))
def test_breakdown_keywords_on_random_traces(opts, bd_mode):
    comm_as_gpu, dataload_as_cpu, gaps = opts
    rng = random.Random(7)
    for i in range(12):
        doc, _ = generate_synthetic_trace(make_spec(rng, rng.randint(20, 600)), seed=i)
        g = build_graph(doc)
        fz = FrozenGraph.from_graph(g)
        assert fz.chained
        res = simulate_batch(fz, ScenarioTable(n_scenarios=1), breakdown=True,
                             comm_as_gpu=comm_as_gpu, dataload_as_cpu=dataload_as_cpu,
                             gaps_as_cpu_busy=gaps)
        st, ms, _lb, _ = OracleGraph.from_graph(g).simulate("default")
        want = ora_breakdown(g.tasks, st, ms, comm_as_gpu, dataload_as_cpu, gaps)
        assert res.breakdown_of(0).to_object() == want, (i, opts)


def test_breakdown_of_shrink_and_remove_sweep(bd_mode):
    w = W.training_trace(n_layers=16, kernels_fwd=3, kernels_bwd=4, n_wu=20, n_streams=2,
                         sync_every=50, seed=4)
    g = w.graph
    scen = ([[(And([GPU_TASKS, ByLayer(l)]), "1/2")] for l in w.layers[:6]]
            + [[(ByLayer(w.layers[2]), REMOVE)], [(GPU_TASKS, "1/3"), (ByLayer(w.layers[5]), REMOVE)],
               [(GPU_TASKS, REMOVE)], []])
    group_of, ptr, steps = compile_scale_sweep(g, scen)
    fz = FrozenGraph.from_graph(g, group_of=group_of)
    res = simulate_batch(fz, ScenarioTable(n_scenarios=len(scen), scale_ptr=ptr, scale=steps),
                         breakdown=True)
    for s, sc in enumerate(scen):
        pipe = [{"op": "remove", "selector": sel.to_object()} if f == REMOVE else
                {"op": "scale", "selector": sel.to_object(), "factor": f} for sel, f in sc]
        h = apply_pipeline(g, TransformPipeline(steps=pipe))
        st, ms, _lb, _ = OracleGraph.from_graph(h).simulate("default")
        assert res.makespan[s] == ms
        assert res.breakdown_of(s).to_object() == ora_breakdown(h.tasks, st, ms), s


def test_breakdown_of_distributed_sweep_with_chains():
    w = W.training_trace(n_layers=12, kernels_fwd=2, kernels_bwd=3, n_wu=16, n_streams=1,
                         sync_every=40, seed=9, buckets_mb=5.0)
    g, buckets = w.graph, w.trace.gradient_buckets
    configs = [{"bandwidth_gbps": bw, "workers": n} for bw in (5, 50) for n in (1, 4, 16)]
    B = len([b for b in buckets.buckets() if buckets.layers_of_bucket(b)])
    rng = np.random.default_rng(2)
    perms = np.array([rng.permutation(B) for _ in configs], np.int16)
    sw = distributed_sweep(g, buckets, configs, perms)
    res = simulate_batch(sw.frozen, sw.table, breakdown=True)
    for s, cfg in enumerate(configs):
        pipe = whatif_distributed(g, buckets=buckets, **cfg)
        steps = [pipe.steps[k] for k in perms[s]] if pipe.steps else []
        h = apply_pipeline(g, TransformPipeline(steps=steps))
        st, ms, _lb, _ = OracleGraph.from_graph(h).simulate("default")
        assert res.makespan[s] == ms, s
        assert res.breakdown_of(s).to_object() == ora_breakdown(h.tasks, st, ms), s


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("depth", ["1", "2", "8"])
def test_breakdown_sweep_jittered_batch(depth, dtype, monkeypatch):
    """100 jittered scenarios (int32 and int64 tables) of a multi-stream training trace through the
    forced streaming sweep: every scenario's four parts equal the oracle's
    (scenarios the sweep hands back are recomputed by the windowed merge), and
    a scenario with one negative duration reports -1."""
    monkeypatch.setenv("DDSIM_BD_SWEEP", "1")
    monkeypatch.setenv("DDSIM_BD_SWEEP_DEPTH", depth)
    w = W.training_trace(n_layers=10, kernels_fwd=3, kernels_bwd=4, n_wu=12, n_streams=3,
                         sync_every=30, seed=5)
    g = w.graph
    fz = FrozenGraph.from_graph(g)
    assert fz.chained and fz.L <= 4
    S = 100  # int32 tables need dense_ld % 4 == 0
    rng = np.random.default_rng(int(depth))
    base = fz.duration[fz.order]
    dense = ((2 * base[:, None] * rng.integers(500, 1501, (fz.n, S)) + 1000) // 2000).astype(dtype)
    dense[rng.integers(0, fz.n), S - 3] = -5  # negative duration: precondition fails
    res = simulate_batch(fz, ScenarioTable(n_scenarios=S, dense=dense), breakdown=True)
    for s in range(S):
        if s == S - 3:
            assert res.parts[s].tolist() == [-1, -1, -1, -1]
            continue
        h = g.copy()
        for r in range(fz.n):
            h.tasks[int(fz.row_ids[r])].duration = int(dense[r, s])
        st, ms, _lb, _ = OracleGraph.from_graph(h).simulate("default")
        assert res.makespan[s] == ms
        assert res.breakdown_of(s).to_object() == ora_breakdown(h.tasks, st, ms), (s, depth, dtype)
