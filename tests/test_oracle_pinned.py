"""Pin the C oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import pytest

from helpers import graph_from_obj, policy_of, sim_as_obj, strip_trace
from oracle import OracleGraph, scale


def _oracle_obj(graph, policy, conv_order=None):
    og = OracleGraph.from_graph(graph, conv_order=conv_order)
    try:
        s, m, lb, tr = og.simulate(policy)
    except RuntimeError:
        return {"error": "Deadlock"}
    return sim_as_obj(s, m, lb, tr)


def test_oracle_simulate_matches_reference_cases(golden):
    for case in golden["cases"]:
        g = graph_from_obj(case["graph"])
        for pol in ("default", "priority"):
            assert _oracle_obj(g, pol) == case["sim"][pol], (case["name"], pol)


def test_oracle_toposort_and_longest_path(golden):
    for case in golden["cases"]:
        og = OracleGraph.from_graph(graph_from_obj(case["graph"]))
        assert og.toposort() == case["topo"], case["name"]
        assert og.longest_path() == case["longest"], case["name"]
        if "gen_makespan" in case:
            assert og.longest_path() == case["gen_makespan"]


def test_oracle_whatif_graphs(golden):
    n = 0
    for rec in golden["whatif"]:
        if "graph" not in rec:
            continue
        g = graph_from_obj(rec["graph"])
        name, params = policy_of(rec)
        got = _oracle_obj(g, name, params.get("conv_order"))
        assert got == rec["sim"], (rec["case"], rec["scenario"], rec["params"])
        assert _oracle_obj(g, "default") == rec["fifo"], (rec["case"], rec["scenario"])
        n += 1
    assert n >= 25


def test_oracle_unsequenced_list_scheduling(golden):
    for rec in golden["unsequenced"]:
        g = graph_from_obj(rec["graph"])
        for pol in ("default", "priority"):
            assert _oracle_obj(g, pol) == rec["sim"][pol], (rec["seed"], pol)


def test_oracle_scale_rounding(golden):
    """Durations are int64 ns on the device and in the oracle: cases whose
    exact result leaves int64 (the reference uses unbounded ints) are outside
    the simulated domain and skipped."""
    n = 0
    for d, num, den, want in golden["units"]["scale"]:
        if want >= 2**63:
            continue
        assert scale(d, num, den) == want
        n += 1
    assert n > 300


def test_known_answers_from_reference_tests(golden):
    """Values quoted from the reference's own tests."""
    by = {c["name"]: c for c in golden["cases"]}
    assert by["gpu_bound"]["sim"]["default"]["makespan"] == 78_790
    assert by["fused_adam"]["sim"]["default"]["makespan"] == 700_000
    assert by["p3"]["sim"]["default"]["makespan"] == 16_000
    reports = {}
    for w in golden["whatif"]:
        if "report" in w:
            reports.setdefault((w["case"], w["scenario"]), w)
    assert reports[("gpu_bound", "amp")]["report"]["predicted_makespan_ns"] == 29_227
    assert reports[("fused_adam", "fused_adam")]["report"]["predicted_makespan_ns"] == 205_000
    p3 = [w for w in golden["whatif"] if w["scenario"] == "p3" and "sim" in w]
    assert p3[0]["sim"]["makespan"] == 30_000 and p3[0]["fifo"]["makespan"] == 32_000
    dgc = [w for w in golden["whatif"] if w["scenario"] == "dgc" and "sim" in w]
    assert dgc[0]["report"]["predicted_makespan_ns"] == 6_000


@pytest.mark.parametrize("bw,expect", [(10, 5_422_000), (20, 2_722_000)])
def test_distributed_fixture_values(golden, bw, expect):
    for w in golden["whatif"]:
        if w["case"] == "distributed_2" and w["scenario"] == "distributed" \
                and w["params"].get("bandwidth_gbps") == bw:
            assert w["report"]["predicted_makespan_ns"] == expect
            return
    raise AssertionError("fixture missing")


EDGE_CODES = {"LaneSeqCpu": 0, "LaneSeqGpu": 1, "LaunchCorrelation": 2, "SyncBlock": 3,
              "CommOrder": 4}


def test_oracle_ingest_matches_reference_graphs(golden):
    """ora_build_graph / ora_map_layers reproduce the reference's build_graph
    + map_tasks_to_layers on every golden trace."""
    import json as _json
    from oracle import build_graph_columns, map_layers_columns
    from paper_2006_03318_b200.trace import TraceColumns, parse_trace
    for case in golden["cases"]:
        doc = parse_trace(_json.dumps(case["doc"]))
        cols = TraceColumns.from_events(list(doc.events))
        edges, gap, launcher = build_graph_columns(cols)
        ids = cols.id.tolist()
        got = {(ids[u], ids[v], k) for u, v, k in edges}
        want = {(u, v, EDGE_CODES[k]) for u, v, k in case["graph"]["edges"]}
        assert got == want, case["name"]
        gaps = {t["id"]: t["gap_ns"] for t in case["graph"]["tasks"]}
        assert dict(zip(ids, gap.tolist())) == gaps, case["name"]
        # layers: markers in list order, tags ranked by (layer, phase)
        markers = list(doc.layer_markers)
        tags = sorted({(m.layer, m.phase.value) for m in markers})
        tid = {t: i for i, t in enumerate(tags)}
        lane_ix = {ln: i for i, ln in enumerate(cols.lanes)}
        ml = [lane_ix.get(m.cpu_lane, -2) for m in markers]
        tag, bad = map_layers_columns(cols, launcher, ml, [m.start for m in markers],
                                      [m.end for m in markers],
                                      [tid[(m.layer, m.phase.value)] for m in markers])
        assert bad == -1
        lay = {t["id"]: (t["layer"], t["phase"]) for t in case["graph"]["tasks"]}
        for i, x in enumerate(ids):
            exp = lay[x]
            got_t = None if tag[i] < 0 else tags[tag[i]]
            if got_t is not None and got_t[0] == "*":
                got_t = ("_global", got_t[1])
            assert (got_t if got_t else (None, None)) == exp, (case["name"], x)


def test_breakdown_oracle_matches_reference_reports(golden):
    """oracle/breakdown_oracle.py against the reference's own whatif reports
    (predicted_breakdown of the transformed graph and its schedule)."""
    from breakdown_oracle import breakdown
    n = 0
    for rec in golden["whatif"]:
        if "graph" not in rec or "error" in rec.get("sim", {}):
            continue
        g = graph_from_obj(rec["graph"])
        start = {int(k): v for k, v in rec["sim"]["start"].items()}
        got = breakdown(g.tasks, start, rec["sim"]["makespan"])
        assert got == rec["report"]["predicted_breakdown"], (rec["case"], rec["scenario"])
        n += 1
    assert n >= 25
