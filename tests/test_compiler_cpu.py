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


def _slot_scan(order, preds):
    """Restatement of the records builder's live-range scan (graph.cu): values
    are tasks in frozen order; a value read only within 48 records takes a
    shared slot while fewer than 24 are live, else a global one; a slot frees
    after its last read. Returns (shared slots, global slots)."""
    import heapq
    pos = {t: i for i, t in enumerate(order)}
    last = {}
    for i, v in enumerate(order):
        for u in preds.get(v, ()):
            last[u] = max(last.get(u, -1), i)
    free_s, free_g, ns, ng = [], [], 0, 0
    slot, glob = {}, {}
    for i, v in enumerate(order):
        lu = last.get(v, -1)
        if lu >= 0:
            if lu - i <= 48 and free_s:
                slot[v], glob[v] = heapq.heappop(free_s), False
            elif lu - i <= 48 and ns < 24:
                slot[v], glob[v], ns = ns, False, ns + 1
            elif free_g:
                slot[v], glob[v] = heapq.heappop(free_g), True
            else:
                slot[v], glob[v], ng = ng, True, ng + 1
        for u in sorted(set(preds.get(v, ())), key=lambda t: pos[t]):
            if last.get(u) == i and u in slot:
                heapq.heappush(free_g if glob[u] else free_s, slot[u])
    return ns, ng


def test_slot_counts_match_linear_scan(golden):
    from paper_2006_03318_b200.frozen import FrozenGraph
    for case in golden["cases"]:
        g = graph_from_obj(case["graph"])
        fz = FrozenGraph.from_graph(g)
        order = [int(t) for t in fz.row_ids]
        preds = {}
        for u, v, _ in g.edges:
            preds.setdefault(int(v), set()).add(int(u))
        ns, ng = _slot_scan(order, preds)
        assert (fz.info.n_slots_smem, fz.info.n_slots) == (ns, ns + ng), case["name"]


def test_slot_counts_match_linear_scan_long_ranges():
    """A launch/kernel graph with far consumers (global slots, slot reuse)."""
    from paper_2006_03318_b200.frozen import FrozenGraph
    rng = np.random.default_rng(3)
    n, CPU, STREAMS = 6000, 2, 3
    half = n // 2
    lane = np.empty(n, np.int32)
    lane[:half] = np.arange(half) % CPU
    lane[half:] = CPU + rng.integers(0, STREAMS, n - half)
    pos = np.empty(n, np.int64)
    pos[np.arange(half)] = 2 * np.arange(half)
    pos[half + np.arange(n - half)] = 2 * np.arange(n - half) + 1
    order = np.lexsort((pos, lane)).astype(np.int32)
    L = CPU + STREAMS
    lop = np.zeros(L + 1, np.int32)
    lop[1:] = np.cumsum(np.bincount(lane, minlength=L))
    same = lane[order[1:]] == lane[order[:-1]]
    far = rng.integers(0, half, 200)                  # a few long-range reads
    es = np.concatenate([order[:-1][same], np.arange(half), far]).astype(np.int32)
    ed = np.concatenate([order[1:][same], half + np.arange(half),
                         np.minimum(far + rng.integers(100, 2000, far.size), half - 1) + half]
                        ).astype(np.int32)
    keep = es != ed
    es, ed = es[keep], ed[keep]
    fz = FrozenGraph(ids=np.arange(n), duration=rng.integers(1, 100, n), gap=np.zeros(n, np.int64),
                     ready=np.zeros(n, np.int64), lane=lane, priority=np.zeros(n, np.int32),
                     flags=np.zeros(n, np.uint8), group=np.zeros(n, np.uint32), edge_src=es,
                     edge_dst=ed, lane_order_ptr=lop, lane_order=order, lanes=list(range(L)))
    assert fz.n_ordered == n
    preds = {}
    for u, v in zip(es.tolist(), ed.tolist()):
        preds.setdefault(v, set()).add(u)
    ns, ng = _slot_scan([int(t) for t in fz.row_ids], preds)
    assert ng > 0
    assert (fz.info.n_slots_smem, fz.info.n_slots) == (ns, ns + ng)
