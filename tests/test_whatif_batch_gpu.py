"""Analysis.whatif_batch / sweep (the `kernsim sweep` loop, cli.py:185-193,
batched) against the reference's own whatif reports and against the
point-by-point whatif on the same Analysis."""

import json

import pytest

from paper_2006_03318_b200 import Analysis
from paper_2006_03318_b200.batch import compile_pipelines
from paper_2006_03318_b200.errors import Unsupported

pytestmark = pytest.mark.gpu

KEYS = ("baseline_makespan_ns", "predicted_makespan_ns", "speedup", "lane_busy_ns",
        "baseline_breakdown", "predicted_breakdown")
BATCHABLE = {"amp", "fused_adam", "reconstruct_batchnorm", "metaflow", "custom"}


def test_whatif_batch_matches_reference_reports(golden):
    docs = {c["name"]: c["doc"] for c in golden["cases"]}
    by_case: dict = {}
    for rec in golden["whatif"]:
        if rec["scenario"] in BATCHABLE and "report" in rec:
            by_case.setdefault((rec["case"], rec["scenario"]), []).append(rec)
    n = 0
    for (case, scen), recs in by_case.items():
        a = Analysis.from_text(json.dumps(docs[case]))
        pipes = [a.pipeline_for(scen, r["params"]) for r in recs]
        compile_pipelines(a.graph, pipes)  # must compile (no per-point fallback)
        got = a.whatif_batch(scen, [r["params"] for r in recs])
        for g, r in zip(got, recs):
            assert {k: g[k] for k in KEYS} == r["report"], (case, scen, r["params"])
            n += 1
    assert n >= 10


def test_sweep_equals_pointwise_whatif(golden):
    docs = {c["name"]: c["doc"] for c in golden["cases"]}
    a = Analysis.from_text(json.dumps(docs["layered"]))
    layers = sorted({t.layer[0] for t in a.graph.tasks.values() if t.layer is not None})
    params = ([{"remove_layers": l} for l in layers] + [{"scale_layers": f"{l}:1/3"} for l in layers]
              + [{"remove_layers": ",".join(layers[:2]), "scale_layers": f"{layers[-1]}:5/2"}])
    got = a.whatif_batch("metaflow", params)
    want = [a.whatif("metaflow", p) for p in params]
    assert got == want
    pts = a.sweep("amp", "compute_factor", ["1/2", "1/3", "1/5", "1"], fixed={"memory_factor": "1/2"})
    assert pts == [(v, a.whatif("amp", {"compute_factor": v, "memory_factor": "1/2"})
                    ["predicted_makespan_ns"]) for v in ["1/2", "1/3", "1/5", "1"]]


def test_set_duration_scale_interplay(golden):
    """set_duration voids earlier scales of that task but not later ones
    (apply_step order, transform.py:285-326)."""
    docs = {c["name"]: c["doc"] for c in golden["cases"]}
    a = Analysis.from_text(json.dumps(docs["gpu_bound"]))
    tid = next(t.id for t in a.graph.tasks.values() if t.lane.is_gpu)
    every = {"all": True}
    pipes = [
        {"steps": [{"op": "scale", "selector": every, "factor": "1/2"},
                   {"op": "set_duration", "task_id": tid, "duration_ns": 12345},
                   {"op": "scale", "selector": every, "factor": "3"}]},
        {"steps": [{"op": "set_duration", "task_id": tid, "duration_ns": 7},
                   {"op": "remove", "task_id": tid}]},
        {"steps": [{"op": "set_priority", "task_id": tid, "priority": 9},
                   {"op": "scale", "selector": every, "factor": "0.75"}]},
    ]
    got = a.whatif_batch("custom", [{"pipeline": p} for p in pipes])
    want = [a.whatif("custom", {"pipeline": p}) for p in pipes]
    assert got == want


def test_insert_pipelines_fall_back_pointwise(golden):
    docs = {c["name"]: c["doc"] for c in golden["cases"]}
    a = Analysis.from_text(json.dumps(docs["distributed_2"]))
    params = [{"workers": 4, "bandwidth_gbps": b} for b in (10, 20)]
    with pytest.raises(Unsupported):
        compile_pipelines(a.graph, [a.pipeline_for("distributed", p) for p in params])
    assert a.whatif_batch("distributed", params) == [a.whatif("distributed", p) for p in params]
