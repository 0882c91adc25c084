"""Host-side logic against the reference's golden vectors (CPU only):
trace parsing/serialisation, comm cost model, what-if generators, selectors."""

import json
from fractions import Fraction

import pytest

from helpers import graph_from_obj
from paper_2006_03318_b200 import comm, errors
from paper_2006_03318_b200.scenarios import generate_pipeline, registry
from paper_2006_03318_b200.trace import (
    TraceColumns,
    document_to_object,
    dump_trace,
    parse_trace,
    us_to_ns,
)
from paper_2006_03318_b200.transform import (
    All,
    And,
    ByKind,
    ByLayer,
    ByNameSubstring,
    Not,
    Or,
    Selector,
    TransformPipeline,
    round_half_up,
)
from paper_2006_03318_b200.trace import Phase, TaskKind


def test_us_to_ns_units(golden):
    for value, want in golden["units"]["us_to_ns"]:
        assert us_to_ns(value) == want, value


def test_parse_dump_roundtrip(golden):
    for case in golden["cases"]:
        doc = parse_trace(json.dumps(case["doc"]))
        assert document_to_object(doc) == case["doc"]
        assert parse_trace(dump_trace(doc)) == doc


def test_overlap_violation_reports_both_ids():
    ev = [{"id": 1, "kind": "CpuOther", "name": "a", "lane": "cpu:0", "start": 0, "duration": 5},
          {"id": 2, "kind": "CpuOther", "name": "b", "lane": "cpu:0", "start": 3, "duration": 1}]
    doc = {"schema_version": 1, "time_unit": "microseconds", "events": ev}
    with pytest.raises(errors.OverlapViolation) as exc:
        parse_trace(json.dumps(doc))
    assert (exc.value.first_id, exc.value.second_id) == (1, 2)


def test_zero_duration_adjacency_is_fine():
    ev = [{"id": 1, "kind": "CpuOther", "name": "a", "lane": "cpu:0", "start": 0, "duration": 5},
          {"id": 2, "kind": "CpuOther", "name": "b", "lane": "cpu:0", "start": 5, "duration": 0},
          {"id": 3, "kind": "CpuOther", "name": "c", "lane": "cpu:0", "start": 5, "duration": 2}]
    parse_trace(json.dumps({"schema_version": 1, "time_unit": "microseconds", "events": ev}))


@pytest.mark.parametrize("bad,err", [
    ("{", errors.MalformedDocument), ("[]", errors.MalformedDocument),
    ('{"schema_version": 2, "time_unit": "microseconds"}', errors.SchemaViolation),
    ('{"schema_version": 1, "time_unit": "ms"}', errors.SchemaViolation),
    ('{"schema_version": 1, "time_unit": "microseconds", "events": [{"id": 0, "kind": "GpuKernel",'
     ' "name": "k", "lane": "gpu:0:1", "start": 0, "duration": 1}]}', errors.SchemaViolation),
    ('{"schema_version": 1, "time_unit": "microseconds", "events": [{"id": 0, "kind": "CpuApi",'
     ' "name": "k", "lane": "gpu:0:1", "start": 0, "duration": 1}]}', errors.SchemaViolation),
    ('{"schema_version": 1, "time_unit": "microseconds", "events": [{"id": 0, "kind": "Nope",'
     ' "name": "k", "lane": "cpu:0", "start": 0, "duration": 1}]}', errors.SchemaViolation),
    ('{"schema_version": 1, "time_unit": "microseconds", "events": [{"id": 0, "kind": "CpuApi",'
     ' "name": "k", "lane": "cpu:0", "start": -1, "duration": 1}]}', errors.SchemaViolation),
])
def test_schema_errors(bad, err):
    with pytest.raises(err):
        parse_trace(bad)


def test_first_overlap_matches_reference_order():
    """First lane (by first appearance) with a violation, first pair within."""
    ev = []
    for i, (lane, st, du) in enumerate([("cpu:1", 0, 4), ("cpu:0", 0, 4), ("cpu:0", 2, 1),
                                        ("cpu:1", 1, 1)]):
        ev.append({"id": 10 + i, "kind": "CpuOther", "name": "x", "lane": lane, "start": st,
                   "duration": du})
    with pytest.raises(errors.OverlapViolation) as exc:
        parse_trace(json.dumps({"schema_version": 1, "time_unit": "microseconds", "events": ev}))
    assert (exc.value.first_id, exc.value.second_id) == (10, 13)


def test_comm_cost_model(golden):
    for rec in golden["units"]["comm"]:
        cfg = comm.NetworkConfig.from_object({"workers": rec["workers"],
                                              "bandwidth_gbps": rec["bw"], "latency_us": "1.5",
                                              "contention_factor": "1.34"})
        assert comm.allreduce_duration(rec["size"], cfg) == rec["allreduce"]
        assert comm.push_pull_duration(rec["size"], cfg) == rec["push_pull"]
        if rec["rs"] is not None:
            assert comm.reduce_scatter_duration(rec["size"], rec["workers"], cfg) == rec["rs"]
    assert comm.allreduce_duration(100_000_000, comm.NetworkConfig(4, 10 * 10**9)) == 120_000_000


def test_round_half_up():
    assert round_half_up(Fraction(5, 2)) == 3
    assert round_half_up(Fraction(-5, 2)) == -3
    assert round_half_up(Fraction(3, 2)) == 2


def test_selector_roundtrip():
    sel = And([ByKind(TaskKind.GPU_KERNEL),
               Not(Or([ByNameSubstring("sgemm"), ByLayer("conv1", Phase.FORWARD)]))])
    assert Selector.from_object(sel.to_object()) == sel
    assert Selector.from_object({"all": True}) == All()
    with pytest.raises(errors.BadSelector):
        Selector.from_object({"bogus": 1})
    with pytest.raises(errors.BadPipeline):
        TransformPipeline.from_object({"no_steps": []})


def test_registry():
    names = [e["name"] for e in registry()]
    assert len(names) == 11 and names[-1] == "custom" and names[:-1] == sorted(names[:-1])


def test_generators_emit_reference_pipelines(golden):
    """Each scenario generator, run on the reference's layer-mapped graph,
    emits exactly the reference's pipeline (or the same error)."""
    cases = {c["name"]: c for c in golden["cases"]}
    checked = 0
    for rec in golden["whatif"]:
        case = cases[rec["case"]]
        g = graph_from_obj(case["graph"])
        trace = parse_trace(json.dumps(case["doc"]))
        try:
            pipe = generate_pipeline(g, rec["scenario"], rec["params"], trace=trace)
        except errors.KernsimError as exc:
            assert rec.get("error") == exc.name, (rec["case"], rec["scenario"])
            continue
        assert "error" not in rec, (rec["case"], rec["scenario"], rec.get("error"))
        assert json.loads(json.dumps(pipe.to_object())) == rec["pipeline"], \
            (rec["case"], rec["scenario"], rec["params"])
        checked += 1
    assert checked >= 25


def test_trace_columns_roundtrip(golden):
    doc = parse_trace(json.dumps(golden["cases"][0]["doc"]))
    cols = TraceColumns.from_events(list(doc.events))
    assert cols.n == len(doc.events)
    assert cols.id.tolist() == [e.id for e in doc.events]
