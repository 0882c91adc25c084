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


def check_recurrence_device(fz, dense, start, makespan, lane_busy, col_block: int = 4096):
    """Every (task, scenario) of a device max-plus result against the
    recurrence start(v) = max(ready(v), max_{u->v} start(u)+dur(u)+gap(u)),
    floored at 0 (sim.py:89-142 on lane-chained graphs == synthetic.py:35-48),
    plus makespan = max(start + dur) (gap excluded, sim.py:125) and lane busy
    = per-lane duration sums (sim.py:124).  Torch on the result's device, in
    scenario blocks; raises AssertionError on the first difference."""
    import numpy as np
    import torch

    dev = start.device
    rows, S = start.shape[0], makespan.shape[0]
    src = torch.from_numpy(fz.row_of[fz.edge_src].astype(np.int64)).to(dev)
    dst = torch.from_numpy(fz.row_of[fz.edge_dst].astype(np.int64)).to(dev)
    gap = torch.from_numpy(fz.gap[fz.order]).to(dev)
    ready = torch.from_numpy(fz.ready[fz.order]).to(dev)
    lane = torch.from_numpy(fz.lane[fz.order].astype(np.int64)).to(dev)
    for c0 in range(0, S, col_block):
        c1 = min(S, c0 + col_block)
        st = start[:rows, c0:c1]
        d = dense[:rows, c0:c1].to(torch.int64)
        rel = st + d + gap[:, None]
        want = ready[:, None].clamp(min=0).expand(rows, c1 - c0).contiguous()
        want.index_reduce_(0, dst, rel[src], "amax", include_self=True)
        bad = (want != st).nonzero()
        assert bad.numel() == 0, f"recurrence violated at (row, scenario) {bad[0].tolist()}"
        fin = (st + d).amax(dim=0)
        assert torch.equal(fin, makespan[c0:c1]), "makespan != max(start + dur)"
        lb = torch.zeros((fz.L, c1 - c0), dtype=torch.int64, device=dev)
        lb.index_add_(0, lane, d)
        assert torch.equal(lb.t(), lane_busy[c0:c1, :fz.L]), "lane busy != per-lane sums"
