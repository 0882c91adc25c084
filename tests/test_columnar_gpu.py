"""Config-5 chain from document TEXT: native reader -> device ingest ->
device layer mapping -> frozen graph, against the reference's golden graphs
and simulations (build_graph + map_tasks_to_layers + simulate, graph.py:
198-312, layers.py:50-81, sim.py:89-142) and, at 1M records, against the
columns the document was written from."""

import json

import numpy as np
import pytest

from helpers import graph_from_obj
from paper_2006_03318_b200.batch import ScenarioTable, simulate_batch
from paper_2006_03318_b200.columnar import dump_trace_columns, ingest_document
from paper_2006_03318_b200.graph import EDGE_KIND_OF_CODE
from paper_2006_03318_b200.ingest import ingest_arrays, map_layers_arrays
from paper_2006_03318_b200.layers import GLOBAL_LAYER

pytestmark = pytest.mark.gpu


def _tag_names(ci):
    out = []
    for t in ci.layer_tag.tolist():
        if t < 0:
            out.append(None)
        else:
            layer, phase = ci.tags[t]
            out.append((GLOBAL_LAYER if layer == "*" else layer, phase))
    return out


@pytest.mark.parametrize("threads", [None, 3])
def test_text_to_graph_matches_reference(golden, threads):
    for case in golden["cases"]:
        text = json.dumps(case["doc"])
        ci = ingest_document(text, threads=threads)
        want = graph_from_obj(case["graph"])
        ids = ci.trace.cols.id
        edges = sorted([int(ids[u]), int(ids[v]), EDGE_KIND_OF_CODE[int(k)].value]
                       for u, v, k in zip(ci.ingest.edge_src, ci.ingest.edge_dst,
                                          ci.ingest.edge_kind))
        assert edges == sorted([u, v, k.value] for u, v, k in want.edges), case["name"]
        assert dict(zip(ids.tolist(), ci.ingest.gap.tolist())) == \
            {t.id: t.gap for t in want.tasks.values()}, case["name"]
        layers = dict(zip(ids.tolist(), _tag_names(ci)))
        assert layers == {t.id: (t.layer[0], t.layer[1].value) if t.layer else None
                          for t in want.tasks.values()}, case["name"]
        # the frozen graph built straight from the ingest output simulates like the reference
        if ci.frozen.n:
            r = simulate_batch(ci.frozen, ScenarioTable(n_scenarios=1))
            assert int(r.makespan[0]) == case["sim"]["default"]["makespan"], case["name"]
            assert {str(k): v for k, v in sorted(r.start_of(0).items())} == \
                case["sim"]["default"]["start"], case["name"]


def test_million_record_document_roundtrip():
    """1M events written to JSON and read back through the whole chain give
    the same edges, gaps and layers as ingesting the generator's columns."""
    from paper_2006_03318_b200.workloads import ingest_document_columns

    ct = ingest_document_columns(1_000_000, seed=5)
    text = dump_trace_columns(ct)
    ci = ingest_document(text, freeze=False)
    direct = ingest_arrays(ct.cols)
    # event order is document order in both; lane ids may be numbered differently
    assert np.array_equal(ci.trace.cols.id, ct.cols.id)
    for k in ("gap", "launcher"):
        assert np.array_equal(getattr(ci.ingest, k), getattr(direct, k)), k

    def edges(r):  # emission order follows lane numbering: compare as a sorted multiset
        e = np.stack([r.edge_src.astype(np.int64), r.edge_dst, r.edge_kind]).T
        return e[np.lexsort(e.T[::-1])]
    assert np.array_equal(edges(ci.ingest), edges(direct))
    tag_m, tags = ct.marker_tags()
    tag = map_layers_arrays(ct.cols, direct.launcher, ct.m_lane, ct.m_start, ct.m_end, tag_m)
    a = np.array([f"{l}/{p}" for l, p in tags] + ["-"])[tag]
    b = np.array([f"{l}/{p}" for l, p in ci.tags] + ["-"])[ci.layer_tag]
    assert np.array_equal(a, b)
    assert (ci.layer_tag >= 0).mean() > 0.5


def _host_frozen(ct, res_host):
    from paper_2006_03318_b200.columnar import frozen_from_ingest
    return frozen_from_ingest(ct, res_host)


@pytest.mark.parametrize("shift_kernel", [False, True])
def test_device_freeze_equals_host_freeze(shift_kernel):
    """ks_graph_create_from_ingest (device: radix-sorted CSR, trace-time order
    verified on every edge) against the host compiler on the same ingest: same
    chained flag, a topological row order, and identical simulations of jitter
    scenarios.  shift_kernel moves a lane's first kernel before its launch, so
    the trace-time order breaks an edge and the host compiler orders it."""
    from paper_2006_03318_b200.columnar import frozen_from_ingest
    from paper_2006_03318_b200.workloads import ingest_document_columns

    ct = ingest_document_columns(120_000, seed=5)
    cols = ct.cols
    if shift_kernel:
        kind = np.asarray(cols.kind)
        lane = np.asarray(cols.lane)
        gpu = np.nonzero(kind == 2)[0]
        first = gpu[np.argmin(np.asarray(cols.start)[gpu])]
        cols.start[first] = 0  # before its launch; still first on its stream
        assert np.sum((lane == lane[first]) & (np.asarray(cols.start) == 0)) == 1
    kept = ingest_arrays(cols, keep_device=True)
    host = ingest_arrays(cols)
    fz_d = frozen_from_ingest(ct, kept)
    fz_h = frozen_from_ingest(ct, host)
    assert fz_d.chained and fz_h.chained and fz_d.n_ordered == fz_h.n_ordered == cols.n
    pos = np.empty(cols.n, np.int64)
    pos[fz_d.order] = np.arange(cols.n)
    assert np.all(pos[host.edge_src] < pos[host.edge_dst])
    assert np.array_equal(kept.edge_src, host.edge_src) and np.array_equal(kept.gap, host.gap)
    S = 8
    rng = np.random.default_rng(2)
    base = np.asarray(cols.duration, np.int64)
    k = rng.integers(900, 1101, size=(cols.n, S))
    per_task = ((2 * base[:, None] * k + 1000) // 2000).astype(np.int64)
    rd = simulate_batch(fz_d, ScenarioTable(n_scenarios=S, dense=np.ascontiguousarray(per_task[fz_d.order])))
    rh = simulate_batch(fz_h, ScenarioTable(n_scenarios=S, dense=np.ascontiguousarray(per_task[fz_h.order])))
    assert np.array_equal(rd.makespan, rh.makespan)
    sd = np.empty_like(rd.start)
    sd[fz_d.order] = rd.start
    sh = np.empty_like(rh.start)
    sh[fz_h.order] = rh.start
    assert np.array_equal(sd, sh)
    assert np.array_equal(rd.lane_busy, rh.lane_busy)
    assert fz_d.info.n_edges_unique == fz_h.info.n_edges_unique
