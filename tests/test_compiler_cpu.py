"""The host graph compiler (ks_graph_create) without a device:
DDSIM_COMPILE_ONLY=1 runs the compile passes and skips uploads."""

import os

import numpy as np
import pytest

from helpers import graph_from_obj


@pytest.fixture(autouse=True)
def compile_only(monkeypatch):
    monkeypatch.setenv("DDSIM_COMPILE_ONLY", "1")


def _is_topological(fz, graph):
    pos = {int(t): r for r, t in enumerate(fz.row_ids)}
    return all(pos[u] < pos[v] for u, v, _ in graph.edges)


def test_frozen_order_is_topological_and_chaining_detected(golden):
    from paper_2006_03318_b200.frozen import FrozenGraph
    for case in golden["cases"]:
        g = graph_from_obj(case["graph"])
        fz = FrozenGraph.from_graph(g)
        assert fz.n_ordered == fz.n
        assert _is_topological(fz, g), case["name"]
        assert fz.chained, case["name"]            # traced graphs are lane-chained
        assert fz.info.n_levels >= 1
    for rec in golden["unsequenced"]:
        g = graph_from_obj(rec["graph"])
        fz = FrozenGraph.from_graph(g)
        assert not fz.chained                      # unsequenced inserts break chaining
        assert _is_topological(fz, g)


def test_cycle_leaves_unordered_rows(golden):
    from paper_2006_03318_b200.frozen import FrozenGraph
    from paper_2006_03318_b200.graph import EdgeKind
    g = graph_from_obj(golden["cases"][0]["graph"])
    ids = sorted(g.tasks)
    g.edges.add((ids[-1], ids[0], EdgeKind.INJECTED))
    fz = FrozenGraph.from_graph(g)
    assert fz.n_ordered < fz.n


def test_chain_compilation_places_members_together():
    from paper_2006_03318_b200 import workloads as W
    from paper_2006_03318_b200.batch import distributed_sweep
    w = W.training_trace(n_layers=12, kernels_fwd=2, kernels_bwd=3, n_wu=10, n_streams=1,
                         sync_every=30, seed=1, buckets_mb=4.0)
    sw = distributed_sweep(w.graph, w.trace.gradient_buckets, [{"workers": 2}, {"workers": 1}])
    fz = sw.frozen
    assert fz.n_ordered == fz.n
    rows = [int(np.nonzero(fz.row_ids == m)[0][0]) for m in sw.member_ids]
    assert rows == list(range(rows[0], rows[0] + len(rows)))   # one macro record
