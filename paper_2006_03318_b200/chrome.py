"""Chrome-trace-format export of simulated schedules (kernsim/chrome.py:17-38).

``export_chrome_trace(result, graph)`` is the reference's export: one "X"
event per task, ts/dur in microseconds, one row (tid) per lane, pid by lane
class.  ``export_chrome_trace_scenario(batch, s, graph)`` renders scenario s
of a batched run straight from the device start rows (frozen row order), with
that scenario's durations when the table carried dense ones; removed /
absent tasks (start -1) are omitted.
"""

from __future__ import annotations

import numpy as np

from .errors import MismatchedInput

_PID_OF_CLASS = {"CpuThread": 1, "GpuStream": 2, "CommChannel": 3}


def _event(task, start: int, duration: int) -> dict:
    return {
        "name": task.name,
        "ph": "X",
        "ts": start / 1000,
        "dur": duration / 1000,
        "pid": _PID_OF_CLASS[task.lane.lane_class.value],
        "tid": str(task.lane),
        "args": {
            "id": task.id,
            "kind": task.kind.value,
            "layer": task.layer[0] if task.layer else None,
            "phase": task.layer[1].value if task.layer else None,
            "gap_ns": task.gap,
        },
    }


def export_chrome_trace(result, graph) -> dict:
    if set(result.start_of) != set(graph.tasks):
        raise MismatchedInput("simulation result and graph disagree on task ids")
    return {"traceEvents": [_event(graph.tasks[tid], start, graph.tasks[tid].duration)
                            for tid, start in sorted(result.start_of.items())]}


def export_chrome_trace_scenario(batch, s: int, graph, durations=None) -> dict:
    """Scenario ``s`` of a BatchResult as a Chrome trace.  ``durations``: the
    scenario's per-frozen-row durations (e.g. ``table.dense[:, s]``); default
    the graph's own."""
    fz = batch.frozen
    if batch.start is None:
        raise ValueError("the batch was simulated without start times")
    col = np.asarray(batch.start[:, s])
    ids = fz.row_ids
    if set(ids.tolist()) != set(graph.tasks):
        raise MismatchedInput("frozen graph and graph disagree on task ids")
    dur = None if durations is None else np.asarray(durations)
    keep = np.nonzero(col >= 0)[0]
    order = keep[np.argsort(ids[keep], kind="stable")]
    events = []
    for r in order.tolist():
        task = graph.tasks[int(ids[r])]
        d = task.duration if dur is None else int(dur[r])
        events.append(_event(task, int(col[r]), d))
    return {"traceEvents": events}


__all__ = ["export_chrome_trace", "export_chrome_trace_scenario"]
