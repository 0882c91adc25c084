"""Shared test helpers: fixture objects -> package objects, comparisons."""

from __future__ import annotations

from paper_2006_03318_b200.graph import DependencyGraph, EdgeKind, Task
from paper_2006_03318_b200.trace import LaneId, Phase, TaskKind


def graph_from_obj(obj: dict) -> DependencyGraph:
    """Rebuild a DependencyGraph from the reference's graph.to_object() dump
    (+ trace_start / ready_time added by make_golden.py)."""
    g = DependencyGraph()
    ts = obj.get("trace_start", {})
    rt = obj.get("ready_time", {})
    for t in obj["tasks"]:
        layer = (t["layer"], Phase(t["phase"])) if t["layer"] is not None else None
        g.tasks[t["id"]] = Task(id=t["id"], kind=TaskKind(t["kind"]), name=t["name"],
                                lane=LaneId.parse(t["lane"]), duration=t["duration_ns"],
                                gap=t["gap_ns"], correlation=t["correlation"], layer=layer,
                                priority=t["priority"], size_bytes=t["size_bytes"],
                                trace_start=ts.get(str(t["id"])),
                                ready_time=rt.get(str(t["id"]), 0))
    g.edges = {(u, v, EdgeKind(k)) for u, v, k in obj["edges"]}
    g.lane_order = {LaneId.parse(k): list(v) for k, v in obj["lane_order"].items()}
    return g


def sim_as_obj(start_of, makespan, lane_busy, trace=None) -> dict:
    out = {"makespan": makespan,
           "start": {str(k): v for k, v in sorted(start_of.items())},
           "lane_busy": {str(k): v for k, v in lane_busy.items()}}
    if trace is not None:
        out["trace"] = [list(x) for x in trace]
    return out


def result_obj(r, with_trace=True) -> dict:
    return sim_as_obj(r.start_of, r.makespan, r.lane_busy, r.schedule_trace if with_trace else None)


def strip_trace(obj: dict) -> dict:
    return {k: v for k, v in obj.items() if k != "trace"}


def policy_of(rec: dict) -> tuple[str, dict]:
    pol = (rec.get("pipeline") or {}).get("schedule_policy") or {}
    return pol.get("name", "default"), dict(pol.get("params", {}))
