"""Generate golden vectors by running the REFERENCE implementation (kernsim).

Run in the development container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference read-only (pkg/src on sys.path, plus pkg/ for the
reference's own test helpers crafted.py / genspec.py), runs it on

  * the reference's crafted traces (tests/crafted.py),
  * a seeded corpus of genspec random traces (tests/genspec.py) -- the same
    generator the reference's property/acceptance tests use,
  * every what-if scenario generator on the crafted traces,
  * unsequenced-insert pipelines on random traces (list-scheduling cases),
  * unit known answers (us_to_ns, scale rounding, comm durations),

and writes tests/golden/golden.json.gz.  Nothing at test time reads
/root/reference; the GPU box only sees the committed fixture.
"""

from __future__ import annotations

import gzip
import json
import random
import sys
from fractions import Fraction
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF))

from kernsim import comm as rcomm  # noqa: E402
from kernsim.api import Analysis  # noqa: E402
from kernsim.graph import build_graph, verify_acyclic  # noqa: E402
from kernsim.layers import map_tasks_to_layers  # noqa: E402
from kernsim.scenarios import generate_pipeline  # noqa: E402
from kernsim.sim import make_policy, simulate  # noqa: E402
from kernsim.synthetic import generate_synthetic_trace, longest_path_makespan  # noqa: E402
from kernsim.trace import dump_trace, parse_trace, us_to_ns  # noqa: E402
from kernsim.transform import TransformPipeline, apply_pipeline, round_half_up  # noqa: E402
from tests import crafted  # noqa: E402
from tests.genspec import random_spec  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden.json.gz"


def graph_obj(g) -> dict:
    obj = g.to_object()
    obj["trace_start"] = {str(t.id): t.trace_start for t in g.tasks.values()}
    obj["ready_time"] = {str(t.id): t.ready_time for t in g.tasks.values() if t.ready_time}
    return obj


def sim_obj(r) -> dict:
    return {
        "makespan": r.makespan,
        "start": {str(k): v for k, v in sorted(r.start_of.items())},
        "lane_busy": {str(k): v for k, v in r.lane_busy.items()},
        "trace": [list(x) for x in r.schedule_trace],
    }


def sim_or_error(g, policy):
    try:
        return sim_obj(simulate(g, policy))
    except Exception as exc:  # noqa: BLE001
        return {"error": type(exc).__name__}


def case_from_doc(name: str, doc: dict, extra: dict | None = None) -> dict:
    text = json.dumps(doc)
    trace = parse_trace(text)
    g = build_graph(trace)
    map_tasks_to_layers(g, list(trace.layer_markers))
    out = {
        "name": name,
        "doc": json.loads(dump_trace(trace)),
        "graph": graph_obj(g),
        "topo": verify_acyclic(g),
        "longest": longest_path_makespan(g),
        "sim": {"default": sim_or_error(g, make_policy("default")),
                "priority": sim_or_error(g, make_policy("priority"))},
    }
    try:
        out["graph_strict_error"] = None
        build_graph(trace, strict=True)
    except Exception as exc:  # noqa: BLE001
        out["graph_strict_error"] = type(exc).__name__
    if extra:
        out.update(extra)
    return out


def whatif_case(case: str, doc: dict, scenario: str, params: dict | None) -> dict:
    a = Analysis.from_text(json.dumps(doc))
    rec = {"case": case, "scenario": scenario, "params": params}
    try:
        pipeline = a.pipeline_for(scenario, params)
    except Exception as exc:  # noqa: BLE001
        rec["error"] = type(exc).__name__
        return rec
    rec["pipeline"] = pipeline.to_object()
    transformed = apply_pipeline(a.graph, pipeline)
    policy = make_policy(pipeline.schedule_policy, **pipeline.policy_params)
    rec["graph"] = graph_obj(transformed)
    rec["sim"] = sim_or_error(transformed, policy)
    rec["fifo"] = sim_or_error(transformed, make_policy("default"))
    rep = a.whatif(scenario, params)
    rec["report"] = {k: rep[k] for k in ("baseline_makespan_ns", "predicted_makespan_ns",
                                         "speedup", "lane_busy_ns", "baseline_breakdown",
                                         "predicted_breakdown")}
    return rec


def random_unsequenced_pipeline(g, rng: random.Random) -> TransformPipeline:
    """Inserts that are NOT sequenced (list-scheduling territory) with random
    comm priorities, plus a scale step and a removal."""
    ids = sorted(g.tasks)
    steps = []
    nxt = g.next_id()
    lanes = ["comm:send", "comm:recv", "gpu:9:1", "cpu:9"]
    kinds = {"comm:send": "Comm", "comm:recv": "Comm", "gpu:9:1": "GpuKernel", "cpu:9": "CpuOther"}
    for _ in range(rng.randint(2, 12)):
        lane = rng.choice(lanes)
        a = rng.choice(ids)
        task = {"id": nxt, "kind": kinds[lane], "name": f"ins_{nxt}", "lane": lane,
                "duration_ns": rng.choice([0, rng.randint(1, 30_000)]),
                "priority": rng.randint(-3, 3)}
        steps.append({"op": "insert", "task": task, "after": [a], "before": [],
                      "sequenced": False})
        ids.append(nxt)
        nxt += 1
    steps.append({"op": "scale", "selector": {"kind": "GpuKernel"}, "factor": "2/3"})
    return TransformPipeline(steps=steps)


def main() -> None:
    golden: dict = {"cases": [], "whatif": [], "unsequenced": [], "units": {}}
    docs = {
        "gpu_bound": crafted.gpu_bound_trace(),
        "cpu_bound": crafted.cpu_bound_trace(),
        "fused_adam": crafted.fused_adam_trace(),
        "fused_adam_1": crafted.fused_adam_trace(n_updates=1),
        "p3": crafted.p3_trace(),
        "distributed_2": crafted.distributed_trace(2),
        "distributed_4": crafted.distributed_trace(4),
        "allreduce": crafted.allreduce_trace(),
        "layered": crafted.layered_trace(),
    }
    for name, doc in docs.items():
        golden["cases"].append(case_from_doc(name, doc))

    # genspec corpus: same construction as the reference's property tests
    for seed in list(range(48)) + [1001, 1002, 1003]:
        rng = random.Random(seed)
        approx = rng.randint(8, 80) if seed < 1000 else rng.randint(1500, 2500)
        spec = random_spec(rng, approx_tasks=approx)
        gen_seed = rng.randint(0, 10**9)
        doc, expected = generate_synthetic_trace(spec, seed=gen_seed)
        golden["cases"].append(case_from_doc(
            f"genspec_{seed}", json.loads(dump_trace(doc)),
            {"spec": spec, "gen_seed": gen_seed, "gen_makespan": expected}))

    scen = [
        ("gpu_bound", "amp", None),
        ("gpu_bound", "amp", {"compute_factor": "1", "memory_factor": "1"}),
        ("cpu_bound", "amp", None),
        ("gpu_bound", "custom", {"pipeline": {"steps": [
            {"op": "scale", "selector": {"all": True}, "factor": "1/2"}]}}),
        ("fused_adam", "fused_adam", None),
        ("fused_adam_1", "fused_adam", None),
        ("gpu_bound", "fused_adam", None),
        ("layered", "reconstruct_batchnorm", None),
        ("layered", "reconstruct_batchnorm", {"include_backward": True}),
        ("gpu_bound", "reconstruct_batchnorm", None),
        ("distributed_2", "distributed", {"workers": 4, "bandwidth_gbps": 10}),
        ("distributed_2", "distributed", {"workers": 4, "bandwidth_gbps": 20}),
        ("distributed_2", "distributed", {"workers": 4, "bandwidth_gbps": 40}),
        ("distributed_2", "distributed", {"workers": 1}),
        ("distributed_4", "distributed", {"workers": 8, "bandwidth_gbps": "2.5",
                                          "latency_us": 3, "contention_factor": "1.34"}),
        ("p3", "p3", crafted.P3_PARAMS),
        ("p3", "p3", dict(crafted.P3_PARAMS, slice_size_bytes=3_000)),
        ("p3", "p3", {"workers": 2}),
        ("allreduce", "blueconnect", {"factorization": "2,2", "workers": 4, "channels": 2,
                                      "bandwidth_gbps": 8}),
        ("allreduce", "blueconnect", {"factorization": "2,3", "workers": 4, "channels": 2}),
        ("layered", "metaflow", None),
        ("layered", "metaflow", {"remove_layers": "relu1", "scale_layers": "conv1:1/2"}),
        ("layered", "vdnn", None),
        ("layered", "vdnn", {"pcie_bandwidth_gbps": 10 ** 9, "launch_cost_ns": 0}),
        ("layered", "vdnn", {"pcie_bandwidth_gbps": "1/1000"}),
        ("gpu_bound", "vdnn", None),
        ("layered", "gist", None),
        ("layered", "gist", {"lossy": True}),
        ("layered", "gist", {"kernel_cost_ns": 5_000, "launch_cost_ns": 0}),
        ("allreduce", "dgc", {"compression_ratio": "1/4"}),
        ("allreduce", "dgc", {"compression_ratio": "1"}),
        ("allreduce", "dgc", {"compression_ratio": "0"}),
        ("gpu_bound", "nope", None),
    ]
    for case, scenario, params in scen:
        golden["whatif"].append(whatif_case(case, docs[case], scenario, params))

    # list-scheduling corpus: random unsequenced inserts on genspec traces
    for seed in range(24):
        rng = random.Random(10_000 + seed)
        spec = random_spec(rng, approx_tasks=rng.randint(10, 60))
        doc, _ = generate_synthetic_trace(spec, seed=rng.randint(0, 10**9))
        trace = parse_trace(dump_trace(doc))
        g = build_graph(trace)
        pipe = random_unsequenced_pipeline(g, rng)
        try:
            out = apply_pipeline(g, pipe)
        except Exception as exc:  # noqa: BLE001
            golden["unsequenced"].append({"seed": seed, "error": type(exc).__name__})
            continue
        golden["unsequenced"].append({
            "seed": seed, "doc": json.loads(dump_trace(doc)), "pipeline": pipe.to_object(),
            "graph": graph_obj(out),
            "sim": {"default": sim_or_error(out, make_policy("default")),
                    "priority": sim_or_error(out, make_policy("priority"))},
        })

    units = golden["units"]
    units["us_to_ns"] = [[v, us_to_ns(v)] for v in
                         [0, 1, 1.5, 0.0005, 0.0015, 0.0025, 2.4994, 2.4995, 123.456789, "7.0005",
                          1e-3, 1234567.8915]]
    rng = random.Random(7)
    scales = []
    for _ in range(400):
        d = rng.choice([0, 1, 2, 3, 5, 7, rng.randint(0, 10**6), rng.randint(0, 10**12),
                        rng.randint(0, 2**62)])
        num = rng.randint(1, 2000)
        den = rng.randint(1, 2000)
        scales.append([d, num, den, round_half_up(Fraction(d) * Fraction(num, den))])
    units["scale"] = scales
    comm = []
    for size in (1, 1500, 12_000_000, 100_000_000, 25 * 2**20):
        for workers in (1, 2, 3, 4, 8, 64):
            for bw in ("1", "8", "10", "2.5", "1/3", "400"):
                cfg = rcomm.NetworkConfig.from_object({"workers": workers, "bandwidth_gbps": bw,
                                                       "latency_us": "1.5",
                                                       "contention_factor": "1.34"})
                comm.append({"size": size, "workers": workers, "bw": bw,
                             "allreduce": rcomm.allreduce_duration(size, cfg),
                             "push_pull": rcomm.push_pull_duration(size, cfg),
                             "rs": (rcomm.reduce_scatter_duration(size, workers, cfg)
                                    if workers >= 2 else None)})
    units["comm"] = comm
    with gzip.open(OUT, "wt") as fh:
        json.dump(golden, fh, separators=(",", ":"))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes): {len(golden['cases'])} cases, "
          f"{len(golden['whatif'])} what-ifs, {len(golden['unsequenced'])} unsequenced")


if __name__ == "__main__":
    main()
