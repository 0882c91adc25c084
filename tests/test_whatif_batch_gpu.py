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


INSERTS = {"distributed", "p3", "blueconnect", "vdnn", "gist", "dgc"}


def test_insert_generators_match_reference_reports(golden):
    """The insert / list-scheduled generators (scenarios.py:191-470) as
    scenario tables: every golden report of p3, blueconnect, vdnn, gist, dgc
    and distributed, one table per structure (batch.structure_key)."""
    from paper_2006_03318_b200.batch import structure_key

    docs = {c["name"]: c["doc"] for c in golden["cases"]}
    by_case: dict = {}
    for rec in golden["whatif"]:
        if rec["scenario"] in INSERTS and "report" in rec:
            by_case.setdefault((rec["case"], rec["scenario"]), []).append(rec)
    n, seen = 0, set()
    for (case, scen), recs in by_case.items():
        a = Analysis.from_text(json.dumps(docs[case]))
        pipes = [a.pipeline_for(scen, r["params"]) for r in recs]
        groups: dict = {}
        for p in pipes:
            groups.setdefault(structure_key(p), []).append(p)
        for ps in groups.values():
            fz, table = compile_pipelines(a.graph, ps)  # no per-point fallback
            seen.add((scen, fz.chained))
        got = a.whatif_batch(scen, [r["params"] for r in recs])
        for g, r in zip(got, recs):
            assert {k: g[k] for k in KEYS} == r["report"], (case, scen, r["params"])
            n += 1
    assert n >= 15
    assert {s for s, _c in seen} == INSERTS
    assert (("p3", False) in seen) and (("distributed", True) in seen)


@pytest.mark.parametrize("scen,case,param,values,fixed", [
    ("p3", "p3", "bandwidth_gbps", [1, 2, 8, 25, 100],
     {"layer_gradient_bytes": {"conv1": 1000, "fc2": 8000}, "workers": 2,
      "slice_size_bytes": 3000, "n_servers": 2}),
    ("dgc", "allreduce", "compression_ratio", ["1", "1/2", "1/4", "0.01", "3"], {}),
    ("vdnn", "layered", "pcie_bandwidth_gbps", [1, 16, 128, "1/1000", 10**9], {}),
    ("gist", "layered", "kernel_cost_ns", [0, 100, 5000, 12345], {"lossy": True}),
    ("blueconnect", "allreduce", "bandwidth_gbps", [1, 8, 100],
     {"factorization": "2,2", "workers": 4, "channels": 2}),
    ("distributed", "distributed_2", "bandwidth_gbps", [1, 10, 20, 40, 400], {"workers": 4}),
])
def test_insert_sweeps_one_table_equal_pointwise(golden, scen, case, param, values, fixed):
    """A parameter sweep of an insert generator is one structure (one table,
    one launch sequence) and equals the reference composition point by point
    (apply_pipeline + simulate + compute_breakdown)."""
    from paper_2006_03318_b200.batch import structure_key

    docs = {c["name"]: c["doc"] for c in golden["cases"]}
    a = Analysis.from_text(json.dumps(docs[case]))
    params = [{**fixed, param: v} for v in values]
    assert len({structure_key(a.pipeline_for(scen, p)) for p in params}) == 1
    got = a.whatif_batch(scen, params)
    want = [a._whatif_pointwise(scen, p) for p in params]
    assert got == want
    assert len({g["predicted_makespan_ns"] for g in got}) > 1


def test_whatif_is_the_batched_device_path(golden):
    """Analysis.whatif (api.py:43-62) is a one-point whatif_batch: same
    report as the reference composition, breakdowns computed by ks_breakdown."""
    from paper_2006_03318_b200 import _native as N

    docs = {c["name"]: c["doc"] for c in golden["cases"]}
    for case, scen, params in (("gpu_bound", "amp", None), ("p3", "p3", {
            "layer_gradient_bytes": {"conv1": 1000, "fc2": 8000}, "bandwidth_gbps": 8,
            "workers": 2, "slice_size_bytes": 3000, "n_servers": 2}),
            ("layered", "vdnn", None)):
        a = Analysis.from_text(json.dumps(docs[case]))
        a.baseline_breakdown()
        l0 = N.launch_count()
        got = a.whatif(scen, params)
        assert N.launch_count() > l0
        assert got == a._whatif_pointwise(scen, params)
