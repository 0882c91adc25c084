"""Seeded synthetic traces with analytically known makespan (kernsim.synthetic).

Reference: pkg/src/kernsim/synthetic.py.  ``generate_synthetic_trace`` turns a
spec (per-lane chains of (kind, duration, gap) plus correlation / sync
structure) into a trace that is a pure function of (spec, seed): durations are
drawn from ``random.Random(seed)`` in the reference's order, starts come from
the same greedy placement rule.  ``longest_path_makespan`` -- the reference's
own max-plus statement (synthetic.py:35-48) -- runs on the device as the
max-plus kernel on a single scenario.
"""

from __future__ import annotations

import json
import random
from typing import Any

import numpy as np

from . import _native as N
from .errors import InvalidSpec
from .graph import DependencyGraph, build_graph
from .trace import (
    GPU_KINDS,
    GradientBucketMap,
    LaneId,
    LayerMarker,
    Phase,
    TaskKind,
    TraceDocument,
    TraceEvent,
    us_to_ns,
)


def longest_path_makespan(graph: DependencyGraph) -> int:
    """Longest weighted path (edge weight = parent duration + gap) on the
    device: the max-plus kernel run once over the frozen topological order."""
    from .errors import CycleDetected
    from .frozen import FrozenGraph
    from .graph import _cycle_among

    if not graph.tasks:
        return 0
    fz = FrozenGraph.from_graph(graph)
    try:
        if fz.n_ordered < fz.n:
            stuck = set(int(i) for i in fz.row_ids[fz.n_ordered:])
            cyc = _cycle_among(graph, stuck)
            raise CycleDetected(f"dependency cycle: {cyc}", cyc)
        sc = N.ScenariosDesc()
        sc.n_scenarios = 1
        ms = np.zeros(1, np.int64)
        out = N.SimOut()
        out.makespan = ms.ctypes.data
        N.check(N.lib().ks_simulate_host(fz.handle, sc, N.KS_POLICY_DEFAULT, N.KS_PATH_MAXPLUS,
                                         out), "longest_path_makespan")
        return int(ms[0])
    finally:
        fz.close()


def _draw(value: Any, rng: random.Random, where: str) -> int:
    if isinstance(value, dict):
        lo, hi = us_to_ns(value.get("min", 0)), us_to_ns(value.get("max", 0))
        if lo < 0 or hi < lo:
            raise InvalidSpec(f"{where}: bad random range {value!r}")
        return rng.randint(lo, hi)
    ns = us_to_ns(value)
    if ns < 0:
        raise InvalidSpec(f"{where}: negative time {value!r}")
    return ns


def _read_spec(spec: dict | str, rng: random.Random):
    if isinstance(spec, str):
        try:
            spec = json.loads(spec)
        except json.JSONDecodeError as exc:
            raise InvalidSpec(f"spec is not valid JSON: {exc}") from None
    if not isinstance(spec, dict) or "lanes" not in spec:
        raise InvalidSpec("spec must be an object with a 'lanes' array")
    lanes = []
    for i, entry in enumerate(spec["lanes"]):
        lane = LaneId.parse(entry["lane"])
        rows = []
        for j, t in enumerate(entry.get("tasks", [])):
            where = f"lanes[{i}].tasks[{j}]"
            kind = TaskKind(t["kind"])
            dur = _draw(t.get("duration_us", 0), rng, where)
            gap = _draw(t.get("gap_us", 0), rng, where)
            rows.append({"kind": kind, "name": t.get("name", f"{kind.value.lower()}_{i}_{j}"),
                         "duration": dur, "gap": gap, "correlation": t.get("correlation"),
                         "sync_target": t.get("sync_target"), "size_bytes": t.get("size_bytes"),
                         "layer": t.get("layer"), "phase": t.get("phase")})
        lanes.append((lane, rows))
    return spec, lanes


def _validate_correlations(lanes) -> None:
    seen = {"gpu": set(), "cpu": set()}
    for _lane, rows in lanes:
        for t in rows:
            c = t["correlation"]
            if c is None:
                continue
            side = "gpu" if t["kind"] in GPU_KINDS else "cpu"
            if c in seen[side]:
                raise InvalidSpec(f"duplicate {side.upper()} correlation {c}")
            seen[side].add(c)
    dangling = seen["gpu"] ^ seen["cpu"]
    if dangling:
        raise InvalidSpec(f"dangling correlation ids: {sorted(dangling)}")
    for _lane, rows in lanes:
        if any(t["kind"] in GPU_KINDS and t["correlation"] is None for t in rows):
            raise InvalidSpec("GPU tasks need a correlation id")


def _placement(lanes) -> dict[tuple[int, int], int]:
    """Greedy consistent execution: repeatedly place the ready task with the
    smallest (tentative start, (lane, position)) (synthetic.py:164-238)."""
    gpu_at: dict[int, tuple[int, int]] = {}
    cpu_at: dict[int, tuple[int, int]] = {}
    for li, (_lane, rows) in enumerate(lanes):
        for ti, t in enumerate(rows):
            if t["correlation"] is not None:
                (gpu_at if t["kind"] in GPU_KINDS else cpu_at)[t["correlation"]] = (li, ti)
    deps: dict[tuple[int, int], list[tuple[int, int]]] = {}
    for li, (_lane, rows) in enumerate(lanes):
        for ti, t in enumerate(rows):
            d = [(li, ti - 1)] if ti > 0 else []
            if t["kind"] in GPU_KINDS:
                d.append(cpu_at[t["correlation"]])
            if t["kind"] is TaskKind.SYNC:
                newest: dict[str, tuple[int, int]] = {}
                for prev in rows[:ti]:
                    c = prev["correlation"]
                    if prev["kind"] not in GPU_KINDS and c in gpu_at:
                        g = gpu_at[c]
                        name = str(lanes[g[0]][0])
                        if t["sync_target"] is None or name == t["sync_target"]:
                            newest[name] = g
                d.extend(newest.values())
            deps[(li, ti)] = d
    waiting = {n: len(d) for n, d in deps.items()}
    kids: dict[tuple[int, int], list[tuple[int, int]]] = {}
    for n, d in deps.items():
        for p in d:
            kids.setdefault(p, []).append(n)
    lane_free = [0] * len(lanes)
    finish: dict[tuple[int, int], int] = {}
    starts: dict[tuple[int, int], int] = {}
    ready = [n for n, c in waiting.items() if c == 0]

    def earliest(node):
        li, ti = node
        s = lane_free[li]
        for p in deps[node]:
            extra = lanes[p[0]][1][p[1]]["gap"] if p == (li, ti - 1) else 0
            s = max(s, finish[p] + extra)
        return s

    while ready:
        node = min(ready, key=lambda n: (earliest(n), n))
        ready.remove(node)
        li, ti = node
        t = lanes[li][1][ti]
        s = earliest(node)
        starts[node] = s
        finish[node] = s + t["duration"]
        lane_free[li] = finish[node] + t["gap"]
        for k in kids.get(node, []):
            waiting[k] -= 1
            if waiting[k] == 0:
                ready.append(k)
    if len(starts) != len(waiting):
        raise InvalidSpec("circular structure in synthetic spec")
    return starts


def _markers(lanes, starts, spec) -> list[LayerMarker]:
    spans: dict[tuple[str, str, str], list[int]] = {}
    for li, (lane, rows) in enumerate(lanes):
        if not lane.is_cpu:
            continue
        for ti, t in enumerate(rows):
            if t["layer"] is None:
                continue
            s = starts[(li, ti)]
            e = s + t["duration"]
            cur = spans.setdefault((t["layer"], t["phase"] or "Forward", str(lane)), [s, e])
            cur[0], cur[1] = min(cur[0], s), max(cur[1], e)
    out = [LayerMarker(layer=l, phase=Phase(p), cpu_lane=LaneId.parse(ln), start=s,
                       end=max(e, s + 1)) for (l, p, ln), (s, e) in sorted(spans.items())]
    for m in spec.get("layer_markers", []):
        out.append(LayerMarker(layer=m["layer"], phase=Phase(m["phase"]),
                               cpu_lane=LaneId.parse(m["cpu_lane"]), start=us_to_ns(m["start"]),
                               end=us_to_ns(m["end"])))
    return out


def generate_synthetic_trace(spec: dict | str, seed: int) -> tuple[TraceDocument, int]:
    """(trace, makespan) as a pure function of (spec, seed)."""
    rng = random.Random(seed)
    spec, lanes = _read_spec(spec, rng)
    _validate_correlations(lanes)
    starts = _placement(lanes)
    events = []
    eid = 0
    for li, (lane, rows) in enumerate(lanes):
        for ti, t in enumerate(rows):
            events.append(TraceEvent(
                id=eid, kind=t["kind"], name=t["name"], lane=lane, start=starts[(li, ti)],
                duration=t["duration"], correlation=t["correlation"], size_bytes=t["size_bytes"],
                sync_target=LaneId.parse(t["sync_target"]) if t["sync_target"] else None))
            eid += 1
    buckets = None
    if spec.get("gradient_buckets"):
        raw = spec["gradient_buckets"]
        buckets = GradientBucketMap(
            bucket_of_layer=dict(raw["bucket_of_layer"]),
            bucket_size_bytes={int(k): v for k, v in raw["bucket_size_bytes"].items()})
    doc = TraceDocument(events=tuple(events), layer_markers=tuple(_markers(lanes, starts, spec)),
                        gradient_buckets=buckets,
                        metadata={str(k): str(v) for k, v in spec.get("metadata", {}).items()})
    return doc, longest_path_makespan(build_graph(doc))
