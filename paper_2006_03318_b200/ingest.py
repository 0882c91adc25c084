"""Device trace ingest: TraceDocument/columns -> dependency graph, layers.

Host orchestration of two C-ABI entry points:

* ks_ingest      -- rules 1/2/5 (lane sequencing), 3 (launch correlation,
                    last CPU launch of a correlation wins), 4 (sync blocking +
                    blocking memcpy_dtoh launches) and CPU gaps
                    (pkg/src/kernsim/graph.py:189-312), plus the lane overlap
                    check (trace.py:255-265);
* ks_map_layers  -- innermost-marker containment + launch inheritance
                    (layers.py:30-81).

``build_graph_device`` materialises the reference object graph from the
device output; ``ingest_arrays`` keeps everything columnar (config 5, no
Python objects per task).
"""

from __future__ import annotations

import os
import sys
import time
from dataclasses import dataclass

import ctypes as C

import numpy as np

from . import _native as N
from .errors import AmbiguousMarker, OrphanKernel, OverlapViolation
from .graph import EDGE_KIND_OF_CODE, DependencyGraph, Task, verify_acyclic
from .trace import (
    CPU_KINDS,
    GPU_KINDS,
    KIND_CODE,
    KIND_OF_CODE,
    LaneId,
    LayerMarker,
    Phase,
    TraceColumns,
    TraceDocument,
)


@dataclass
class IngestResult:
    cols: TraceColumns
    edge_src: np.ndarray    # event indices
    edge_dst: np.ndarray
    edge_kind: np.ndarray   # uint8 KS_EDGE_*
    lane_order: np.ndarray  # event indices grouped by lane index
    lane_order_ptr: np.ndarray
    gap: np.ndarray         # int64 per event
    launcher: np.ndarray    # int32 per event (-1 none)

    def edge_triples(self):
        ids = self.cols.id
        kinds = [EDGE_KIND_OF_CODE[k] for k in self.edge_kind.tolist()]
        return list(zip(ids[self.edge_src].tolist(), ids[self.edge_dst].tolist(), kinds))

    def gaps_by_id(self) -> dict[int, int]:
        return dict(zip(self.cols.id.tolist(), self.gap.tolist()))


def _trace_cols_struct(cols: TraceColumns, strict: bool, keep: list) -> N.TraceCols:
    tc = N.TraceCols()
    tc.n = cols.n
    arrs = {
        "id": N.c_i64(cols.id), "kind": np.ascontiguousarray(cols.kind, np.uint8),
        "lane": N.c_i32(cols.lane), "start": N.c_i64(cols.start),
        "duration": N.c_i64(cols.duration), "correlation": N.c_i64(cols.correlation),
        "sync_target": N.c_i32(cols.sync_target),
        "is_dtoh": np.ascontiguousarray(cols.is_dtoh, np.uint8),
    }
    for k, a in arrs.items():
        keep.append(a)
        setattr(tc, k, N.ptr(a))
    lc, lr = cols.lane_class_codes(), cols.lane_str_rank()
    keep += [lc, lr]
    tc.n_lanes = len(cols.lanes)
    tc.lane_class, tc.lane_rank = N.ptr(lc), N.ptr(lr)
    tc.strict = 1 if strict else 0
    return tc


_T = [0.0]


def _tick(what):
    """DDSIM_INGEST_TIMING=1: wall time of the host-side steps."""
    if not os.environ.get("DDSIM_INGEST_TIMING"):
        return
    t = time.perf_counter()
    if what is not None:
        print(f"[ingest_arrays] {what:12s} {1e3 * (t - _T[0]):8.3f} ms", file=sys.stderr)
    _T[0] = t


class KeptIngest:
    """ks_ingest_keep output: edges, lane order and gaps stay on the device
    for a device freeze (frozen_from_ingest); the IngestResult fields are
    copied to the host on first access."""

    def __init__(self, cols: TraceColumns, handle, n_edges: int, lane_order_ptr, launcher,
                 device: int):
        self.cols = cols
        self.device = device
        self.handle = handle
        self.n_edges = n_edges
        self.lane_order_ptr = lane_order_ptr
        self.launcher = launcher
        self._host = None

    def _fetch(self) -> IngestResult:
        if self._host is None:
            n, m = self.cols.n, self.n_edges
            src, dst = np.empty(max(m, 1), np.int32), np.empty(max(m, 1), np.int32)
            kind, lo = np.empty(max(m, 1), np.uint8), np.empty(max(n, 1), np.int32)
            gap = np.empty(max(n, 1), np.int64)
            N.check(N.lib().ks_ingest_dev_copy(self.handle, N.ptr(src), N.ptr(dst), N.ptr(kind),
                                               N.ptr(lo), N.ptr(gap)), "ks_ingest_dev_copy")
            self._host = IngestResult(cols=self.cols, edge_src=src[:m], edge_dst=dst[:m],
                                      edge_kind=kind[:m], lane_order=lo[:n],
                                      lane_order_ptr=self.lane_order_ptr, gap=gap[:n],
                                      launcher=self.launcher)
        return self._host

    def __getattr__(self, name):
        if name in ("edge_src", "edge_dst", "edge_kind", "lane_order", "gap", "edge_triples",
                    "gaps_by_id"):
            return getattr(self._fetch(), name)
        raise AttributeError(name)

    def close(self):
        h = self.__dict__.get("handle")
        if h is not None and h.value:
            N.lib().ks_ingest_dev_free(h)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def ingest_arrays(cols: TraceColumns, strict: bool = False, check_overlaps: bool = False,
                  device: int | None = None, keep_device: bool = False):
    """ks_ingest on the columns.  keep_device=True: a KeptIngest whose edges /
    lane order / gaps stay on the device for frozen_from_ingest's device
    freeze (ks_ingest_keep)."""
    device = N.env_device() if device is None else device
    _tick(None)
    N.require_device(device)
    keep: list = []
    tc = _trace_cols_struct(cols, strict, keep)
    n = cols.n
    n_gpu_lanes = int(np.sum(cols.lane_class_codes() == 1))
    n_sync = int(np.sum(cols.kind == KIND_CODE[next(k for k in KIND_CODE if k.value == "Sync")]))
    cap = 2 * n + n_sync * max(n_gpu_lanes, 1) + 16
    out = N.IngestOut()
    if keep_device:
        bufs = {"lane_order_ptr": np.empty(len(cols.lanes) + 1, np.int32),
                "launcher": np.empty(max(n, 1), np.int32)}
    else:
        bufs = {
            "edge_src": np.empty(cap, np.int32), "edge_dst": np.empty(cap, np.int32),
            "edge_kind": np.empty(cap, np.uint8), "lane_order": np.empty(max(n, 1), np.int32),
            "lane_order_ptr": np.empty(len(cols.lanes) + 1, np.int32),
            "gap": np.empty(max(n, 1), np.int64), "launcher": np.empty(max(n, 1), np.int32),
        }
    for k, a in bufs.items():
        setattr(out, k, a.ctypes.data)
    out.edge_cap = cap
    _tick("host prep")
    handle = C.c_void_p()
    if keep_device:
        rc = N.lib().ks_ingest_keep(tc, device, 1 if check_overlaps else 0, out, C.byref(handle))
    else:
        rc = N.lib().ks_ingest(tc, device, 1 if check_overlaps else 0, out)
    if rc == N.KS_ERR_OVERLAP:
        a, b = int(out.bad_a), int(out.bad_b)
        lane = cols.lanes[int(cols.lane[cols.index_of(a)])]
        raise OverlapViolation(f"events {a} and {b} overlap on lane {lane}", a, b)
    if rc == N.KS_ERR_ORPHAN:
        i = cols.index_of(int(out.bad_a))
        raise OrphanKernel(f"GPU task {int(out.bad_a)} correlation {int(cols.correlation[i])} "
                           "has no CPU launch")
    N.check(rc, "ks_ingest")
    _tick("ks_ingest")
    m = int(out.n_edges)
    if keep_device:
        return KeptIngest(cols, handle, m, bufs["lane_order_ptr"], bufs["launcher"][:n], device)
    return IngestResult(cols=cols, edge_src=bufs["edge_src"][:m].copy(),
                        edge_dst=bufs["edge_dst"][:m].copy(),
                        edge_kind=bufs["edge_kind"][:m].copy(), lane_order=bufs["lane_order"][:n],
                        lane_order_ptr=bufs["lane_order_ptr"], gap=bufs["gap"][:n],
                        launcher=bufs["launcher"][:n])


_INGEST_CACHE: dict[int, tuple[TraceDocument, bool, IngestResult]] = {}


def ingest_columns(trace: TraceDocument, strict: bool = False) -> IngestResult:
    hit = _INGEST_CACHE.get(id(trace))
    if hit is not None and hit[0] is trace and hit[1] == strict:
        return hit[2]
    res = ingest_arrays(TraceColumns.from_events(list(trace.events)), strict=strict)
    _INGEST_CACHE.clear()
    _INGEST_CACHE[id(trace)] = (trace, strict, res)
    return res


def build_graph_device(trace: TraceDocument, strict: bool = False) -> DependencyGraph:
    res = ingest_columns(trace, strict=strict)
    cols = res.cols
    g = DependencyGraph()
    gaps = res.gap.tolist()
    for i, e in enumerate(trace.events):
        g.tasks[e.id] = Task(id=e.id, kind=e.kind, name=e.name, lane=e.lane, duration=e.duration,
                             gap=gaps[i], correlation=e.correlation, size_bytes=e.size_bytes,
                             trace_start=e.start)
    g.edges = set(res.edge_triples())
    ids = cols.id
    lop = res.lane_order_ptr
    # lane_order insertion order: lanes sorted by their text (graph.py:222)
    for j in sorted(range(len(cols.lanes)), key=lambda j: str(cols.lanes[j])):
        if lop[j + 1] > lop[j]:  # lanes only named as a sync target carry no events
            g.lane_order[cols.lanes[j]] = ids[res.lane_order[lop[j]:lop[j + 1]]].tolist()
    verify_acyclic(g)
    return g


# ---------------------------------------------------------------- layer map

def _tag_tables(markers: list[LayerMarker]):
    """Intern (layer, phase) tags; tag id order == (layer, phase.value) order."""
    tags = sorted({(m.layer, m.phase.value) for m in markers})
    tag_id = {t: i for i, t in enumerate(tags)}
    return tags, tag_id


def map_layers_device(graph: DependencyGraph, markers: list[LayerMarker],
                      device: int | None = None) -> dict[int, tuple[str, Phase]]:
    device = N.env_device() if device is None else device
    from .layers import GLOBAL_LAYER

    tasks = list(graph.tasks.values())
    if not tasks:
        return {}
    N.require_device(device)
    lane_ix: dict[LaneId, int] = {}
    lanes: list[LaneId] = []

    def lix(ln):
        j = lane_ix.get(ln)
        if j is None:
            j = lane_ix[ln] = len(lanes)
            lanes.append(ln)
        return j

    n = len(tasks)
    ids = np.fromiter((t.id for t in tasks), np.int64, n)
    kind = np.fromiter((KIND_CODE[t.kind] for t in tasks), np.uint8, n)
    lane = np.fromiter((lix(t.lane) for t in tasks), np.int32, n)
    has_ts = np.fromiter((t.trace_start is not None for t in tasks), bool, n)
    start = np.fromiter((t.trace_start or 0 for t in tasks), np.int64, n)
    dur = np.fromiter((t.duration for t in tasks), np.int64, n)
    # tasks without a trace start are never mapped: give them an impossible lane
    mlane = np.array([lix(m.cpu_lane) for m in markers], np.int32)
    lane_task = np.where(has_ts, lane, -1).astype(np.int32)
    index = {t.id: i for i, t in enumerate(tasks)}
    launcher = np.full(n, -1, np.int32)
    for u, v, k in graph.edges:
        if k.value == "LaunchCorrelation" and v in index and u in index:
            launcher[index[v]] = index[u]
    tags, tag_id = _tag_tables(markers)
    cols = TraceColumns(id=ids, kind=kind, lane=lane_task, start=start, duration=dur,
                        correlation=np.full(n, -1, np.int64), sync_target=np.full(n, -1, np.int32),
                        is_dtoh=np.zeros(n, np.uint8), lanes=lanes)
    keep: list = []
    tc = _trace_cols_struct(cols, False, keep)
    mc = N.MarkerCols()
    marr = {"lane": mlane, "start": np.array([m.start for m in markers], np.int64),
            "end": np.array([m.end for m in markers], np.int64),
            "tag": np.array([tag_id[(m.layer, m.phase.value)] for m in markers], np.int32)}
    mc.n = len(markers)
    for k, a in marr.items():
        keep.append(a)
        setattr(mc, k, N.ptr(a))
    tag_out = np.full(n, -1, np.int32)
    bad = np.zeros(1, np.int64)
    rc = N.lib().ks_map_layers(tc, launcher.ctypes.data, mc, device, tag_out.ctypes.data,
                               bad.ctypes.data)
    if rc == N.KS_ERR_AMBIGUOUS:
        raise AmbiguousMarker(f"task {int(bad[0])} falls inside overlapping markers")
    N.check(rc, "ks_map_layers")
    out: dict[int, tuple[str, Phase]] = {}
    for i in np.nonzero(tag_out >= 0)[0].tolist():
        layer, phase = tags[tag_out[i]]
        out[int(ids[i])] = (GLOBAL_LAYER if layer == "*" else layer, Phase(phase))
    return out


def map_layers_arrays(cols: TraceColumns, launcher: np.ndarray, m_lane, m_start, m_end, m_tag,
                      device: int | None = None) -> np.ndarray:
    """Columnar layer mapping (config 5): tag id per event or -1."""
    device = N.env_device() if device is None else device
    N.require_device(device)
    keep: list = []
    tc = _trace_cols_struct(cols, False, keep)
    mc = N.MarkerCols()
    arrs = {"lane": N.c_i32(m_lane), "start": N.c_i64(m_start), "end": N.c_i64(m_end),
            "tag": N.c_i32(m_tag)}
    mc.n = len(arrs["lane"])
    for k, a in arrs.items():
        keep.append(a)
        setattr(mc, k, N.ptr(a))
    la = N.c_i32(launcher)
    tag = np.full(cols.n, -1, np.int32)
    bad = np.zeros(1, np.int64)
    rc = N.lib().ks_map_layers(tc, la.ctypes.data, mc, device, tag.ctypes.data, bad.ctypes.data)
    if rc == N.KS_ERR_AMBIGUOUS:
        raise AmbiguousMarker(f"task {int(bad[0])} falls inside overlapping markers")
    N.check(rc, "ks_map_layers")
    return tag


__all__ = ["map_layers_arrays","IngestResult", "ingest_arrays", "ingest_columns", "build_graph_device",
           "map_layers_device", "CPU_KINDS", "GPU_KINDS", "KIND_OF_CODE"]
