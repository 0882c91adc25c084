"""Device trace ingest (build_graph, map_tasks_to_layers) and the end-to-end
Analysis API against the reference's golden vectors."""

import json

import numpy as np
import pytest

from helpers import graph_from_obj
from paper_2006_03318_b200 import Analysis, build_graph, errors, map_tasks_to_layers
from paper_2006_03318_b200.ingest import ingest_arrays
from paper_2006_03318_b200.synthetic import generate_synthetic_trace
from paper_2006_03318_b200.trace import TraceColumns, document_to_object, parse_trace
from paper_2006_03318_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _obj(g):
    return {
        "edges": sorted([u, v, k.value] for u, v, k in g.edges),
        "gaps": {t.id: t.gap for t in g.tasks.values()},
        "lane_order": {str(k): v for k, v in g.lane_order.items()},
        "layers": {t.id: (t.layer[0], t.layer[1].value) if t.layer else None
                   for t in g.tasks.values()},
    }


def _golden_obj(graph_obj):
    g = graph_from_obj(graph_obj)
    return _obj(g)


def test_build_graph_and_layers_match_reference(golden):
    for case in golden["cases"]:
        trace = parse_trace(json.dumps(case["doc"]))
        g = build_graph(trace)
        map_tasks_to_layers(g, list(trace.layer_markers))
        assert _obj(g) == _golden_obj(case["graph"]), case["name"]
        # lane_order insertion order follows the lane text (graph.py:222)
        assert list(map(str, g.lane_order)) == list(case["graph"]["lane_order"])


def test_strict_orphans(golden):
    for case in golden["cases"]:
        trace = parse_trace(json.dumps(case["doc"]))
        if case["graph_strict_error"] is None:
            build_graph(trace, strict=True)
        else:
            with pytest.raises(errors.OrphanKernel):
                build_graph(trace, strict=True)
    b = {"schema_version": 1, "time_unit": "microseconds", "events": [
        {"id": 0, "kind": "GpuKernel", "name": "k", "lane": "gpu:0:1", "start": 0, "duration": 1,
         "correlation": 99}]}
    tr = parse_trace(json.dumps(b))
    assert not build_graph(tr).edges
    with pytest.raises(errors.OrphanKernel):
        build_graph(tr, strict=True)


def test_device_overlap_check_matches_host(golden):
    ev = []
    for i, (lane, st, du) in enumerate([("cpu:1", 0, 4), ("cpu:0", 0, 4), ("cpu:0", 2, 1),
                                        ("cpu:1", 1, 1), ("gpu:0:1", 0, 3)]):
        ev.append({"id": 10 + i, "kind": "CpuOther" if lane.startswith("cpu") else "GpuKernel",
                   "name": "x", "lane": lane, "start": st, "duration": du, "correlation": 1})
    from paper_2006_03318_b200.trace import TraceEvent, LaneId, TaskKind
    evs = [TraceEvent(id=e["id"], kind=TaskKind(e["kind"]), name="x", lane=LaneId.parse(e["lane"]),
                      start=e["start"] * 1000, duration=e["duration"] * 1000,
                      correlation=e["correlation"]) for e in ev]
    with pytest.raises(errors.OverlapViolation) as exc:
        ingest_arrays(TraceColumns.from_events(evs), check_overlaps=True)
    assert (exc.value.first_id, exc.value.second_id) == (10, 13)
    for case in golden["cases"][:20]:
        trace = parse_trace(json.dumps(case["doc"]))
        ingest_arrays(TraceColumns.from_events(list(trace.events)), check_overlaps=True)


def test_layer_mapping_edge_cases():
    def doc(events, markers):
        return json.dumps({"schema_version": 1, "time_unit": "microseconds", "events": events,
                           "layer_markers": markers})
    ev = lambda i, s, d, k="CpuOther", corr=None, lane="cpu:0": dict(  # noqa: E731
        {"id": i, "kind": k, "name": "t", "lane": lane, "start": s, "duration": d},
        **({"correlation": corr} if corr is not None else {}))
    mk = lambda l, s, e, ph="Forward": {"layer": l, "phase": ph, "cpu_lane": "cpu:0",  # noqa: E731
                                         "start": s, "end": e}
    # innermost nested marker wins; launch inheritance; '*' -> _global
    t = parse_trace(doc([ev(0, 2, 1), ev(1, 20, 1, "CpuApi", 1), ev(2, 60, 5, "GpuKernel", 1,
                                                                    "gpu:0:1")],
                        [mk("outer", 0, 10), mk("inner", 1.5, 4), mk("*", 15, 30, "Backward")]))
    g = build_graph(t)
    map_tasks_to_layers(g, list(t.layer_markers))
    assert g.tasks[0].layer[0] == "inner"
    assert g.tasks[1].layer[0] == "_global" and g.tasks[2].layer == g.tasks[1].layer
    # non-nested overlap -> AmbiguousMarker
    t2 = parse_trace(doc([ev(0, 4, 0.5)], [mk("left", 0, 6), mk("right", 3, 9)]))
    g2 = build_graph(t2)
    with pytest.raises(errors.AmbiguousMarker):
        map_tasks_to_layers(g2, list(t2.layer_markers))


@pytest.mark.parametrize("make", [W.resnet50_trace, W.bert_trace, W.gpt_trace])
def test_ingest_at_scale_matches_construction(make):
    w = make()
    g = build_graph(w.trace)
    map_tasks_to_layers(g, list(w.trace.layer_markers))
    ref = w.graph
    assert g.edges == ref.edges
    assert {k: v for k, v in g.lane_order.items()} == {k: v for k, v in ref.lane_order.items()}
    assert all(g.tasks[i].gap == ref.tasks[i].gap for i in ref.tasks)
    for i, t in ref.tasks.items():
        if t.kind.value in ("CpuApi", "GpuKernel"):
            assert g.tasks[i].layer == t.layer


def test_generate_synthetic_trace_matches_reference(golden):
    for case in golden["cases"]:
        if "spec" not in case:
            continue
        doc, ms = generate_synthetic_trace(case["spec"], seed=case["gen_seed"])
        assert ms == case["gen_makespan"], case["name"]
        assert document_to_object(doc) == case["doc"], case["name"]


def test_analysis_whatif_reports_match_reference(golden):
    docs = {c["name"]: c["doc"] for c in golden["cases"]}
    n = 0
    for rec in golden["whatif"]:
        a = Analysis.from_text(json.dumps(docs[rec["case"]]))
        if "error" in rec:
            with pytest.raises(errors.KernsimError) as exc:
                a.whatif(rec["scenario"], rec["params"])
            assert exc.value.name == rec["error"]
            continue
        rep = a.whatif(rec["scenario"], rec["params"])
        want = rec["report"]
        for key in ("baseline_makespan_ns", "predicted_makespan_ns", "lane_busy_ns",
                    "baseline_breakdown", "predicted_breakdown"):
            assert rep[key] == want[key], (rec["case"], rec["scenario"], key)
        assert rep["speedup"] == pytest.approx(want["speedup"], abs=0, rel=1e-15)
        n += 1
    assert n >= 25


def test_apply_pipeline_graphs_match_reference(golden):
    """The transformed graphs themselves (tasks, edges, lane order)."""
    from paper_2006_03318_b200.transform import TransformPipeline, apply_pipeline
    cases = {c["name"]: c for c in golden["cases"]}
    for rec in golden["whatif"]:
        if "graph" not in rec:
            continue
        base = graph_from_obj(cases[rec["case"]]["graph"])
        out = apply_pipeline(base, TransformPipeline.from_object(rec["pipeline"]))
        want = graph_from_obj(rec["graph"])
        assert out.to_object() == want.to_object(), (rec["case"], rec["scenario"])


@pytest.mark.parametrize("n", [120_000])
def test_columnar_ingest_matches_oracle_at_scale(n):
    """Config-5 generator (8 CPU threads x 16 streams, memcpys incl. blocking
    dtoh, stream + device-wide syncs, data loads): device ingest + layer
    mapping vs the C oracle's restatement of the reference rules."""
    from oracle import build_graph_columns, map_layers_columns
    from paper_2006_03318_b200.ingest import map_layers_arrays
    cols = W.ingest_columns(n, seed=3)
    res = ingest_arrays(cols, check_overlaps=True)
    edges, gap, launcher = build_graph_columns(cols)
    got = set(zip(res.edge_src.tolist(), res.edge_dst.tolist(), res.edge_kind.tolist()))
    assert len(got) == len(res.edge_src)           # no duplicate triples
    assert got == edges
    assert np.array_equal(res.gap, gap)
    assert np.array_equal(res.launcher, launcher)
    m = cols.markers
    tags = map_layers_arrays(cols, res.launcher, m["lane"], m["start"], m["end"], m["tag"])
    want, bad = map_layers_columns(cols, launcher, m["lane"], m["start"], m["end"], m["tag"])
    assert bad == -1
    assert np.array_equal(tags, want)
