"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's runtime
breakdown, used as the checker of the device kernel (ks_breakdown).

Follows pkg/src/kernsim/breakdown.py:42-111 step by step:
  * compute_breakdown (:42-98): +1/-1 deltas at interval endpoints per class
    (CPU lanes [start, end + gap) with gaps_as_cpu_busy, DataLoad skipped
    unless dataload_as_cpu; GPU lanes [start, end); comm lanes count as GPU
    unless comm_as_gpu is False), then a sweep over the sorted endpoint set
    restricted to [0, makespan] classifying each span.
  * per_layer_breakdown (:100-111): summed CPU / GPU durations per layer of
    the scheduled tasks, comm lanes excluded, untagged -> "_unmapped".
Pure-Python loops: small cases only.  Pinned against the reference's own
reports in tests/golden/golden.json.gz (whatif[*].report.*_breakdown).
"""

from __future__ import annotations

UNMAPPED = "_unmapped"  # layers.py UNMAPPED_LAYER


def breakdown(tasks, start_of: dict, makespan: int, comm_as_gpu=True, dataload_as_cpu=True,
              gaps_as_cpu_busy=True) -> dict:
    """tasks: id -> object with .lane (.is_cpu/.is_gpu/.is_comm), .kind.value,
    .duration, .gap, .layer.  Returns the reference's to_object() dict."""
    cpu_d: dict[int, int] = {}
    gpu_d: dict[int, int] = {}

    def mark(dd, a, b):
        if b > a:
            dd[a] = dd.get(a, 0) + 1
            dd[b] = dd.get(b, 0) - 1

    for tid, st in start_of.items():
        t = tasks[tid]
        end = st + t.duration
        if t.lane.is_cpu:
            if t.kind.value == "DataLoad" and not dataload_as_cpu:
                continue
            mark(cpu_d, st, end + (t.gap if gaps_as_cpu_busy else 0))
        elif t.lane.is_gpu:
            mark(gpu_d, st, end)
        else:
            mark(gpu_d if comm_as_gpu else cpu_d, st, end)
    pts = sorted(set(cpu_d) | set(gpu_d) | {0, makespan})
    pts = [x for x in pts if 0 <= x <= makespan]
    acc = {"cpu": 0, "gpu": 0, "par": 0, "idle": 0}
    cl = gl = 0
    for a, b in zip(pts, pts[1:]):
        cl += cpu_d.get(a, 0)
        gl += gpu_d.get(a, 0)
        k = "par" if cl > 0 and gl > 0 else "cpu" if cl > 0 else "gpu" if gl > 0 else "idle"
        acc[k] += b - a
    per: dict[str, list[int]] = {}
    for tid in start_of:
        t = tasks[tid]
        if t.lane.is_comm:
            continue
        name = t.layer[0] if t.layer is not None else UNMAPPED
        slot = per.setdefault(name, [0, 0])
        slot[0 if t.lane.is_cpu else 1] += t.duration
    return {"cpu_only_ns": acc["cpu"], "gpu_only_ns": acc["gpu"], "parallel_ns": acc["par"],
            "idle_ns": acc["idle"], "total_ns": makespan,
            "per_layer": {k: {"cpu_ns": c, "gpu_ns": g} for k, (c, g) in sorted(per.items())}}
