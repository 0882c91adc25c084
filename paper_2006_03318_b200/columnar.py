"""Columnar trace documents: the native reader/writer (include/ddsim.h
``ks_trace_parse`` / ``ks_trace_write``) and the config-5 ingest pipeline.

``load_trace_columns(text)`` is ``parse_trace`` (pkg/src/kernsim/trace.py:
281-328) for traces too large for Python objects: the JSON text is parsed by
multi-threaded host C++ straight into the columns ``ks_ingest`` /
``ks_map_layers`` consume, with the reference's validation and error
precedence (MalformedDocument > SchemaViolation (document order) >
duplicate id > OverlapViolation > marker errors > gradient_buckets >
metadata).  ``dump_trace_columns`` is ``dump_trace`` (trace.py:331-379) from
columns.  ``ColumnarTrace.to_document()`` materialises the reference's
TraceDocument for small traces (parity tests).

``ingest_document(text)`` chains parse -> device ingest (graph.py:198-312) ->
device layer mapping (layers.py:50-81) -> device-resident frozen graph
(graph.py:75-148), without a Python object per event.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import MalformedDocument, OverlapViolation, SchemaViolation
from .trace import (
    KIND_CODE,
    KIND_OF_CODE,
    GradientBucketMap,
    LaneId,
    LayerMarker,
    Phase,
    TaskKind,
    TraceColumns,
    TraceDocument,
    TraceEvent,
    _buckets_from,
)

PHASES = (Phase.FORWARD, Phase.BACKWARD, Phase.WEIGHT_UPDATE)  # ks_trace_marker_cols.phase
PHASE_CODE = {p: i for i, p in enumerate(PHASES)}


@dataclass
class ColumnarTrace:
    """A trace document as columns.  ``cols.lanes`` holds every lane: the
    first ``n_event_lanes`` in TraceColumns.from_events order, then lanes named
    only by layer markers."""

    cols: TraceColumns
    name_id: np.ndarray            # int32 per event
    names: list                    # distinct names, first-appearance order
    size_bytes: np.ndarray         # int64 per event, -1 = none
    n_event_lanes: int
    m_lane: np.ndarray             # int32 per marker (index into cols.lanes)
    m_start: np.ndarray
    m_end: np.ndarray
    m_layer: np.ndarray            # int32 index into layers
    m_phase: np.ndarray            # uint8 PHASE_CODE
    layers: list
    gradient_buckets: GradientBucketMap | None = None
    metadata: dict = field(default_factory=dict)

    @property
    def n_events(self) -> int:
        return self.cols.n

    @property
    def n_markers(self) -> int:
        return int(self.m_start.shape[0])

    # ---- conversions --------------------------------------------------------
    @staticmethod
    def from_document(doc: TraceDocument) -> "ColumnarTrace":
        events = list(doc.events)
        cols = TraceColumns.from_events(events)
        n_ev_lanes = len(cols.lanes)
        name_ix: dict[str, int] = {}
        name_id = np.fromiter((name_ix.setdefault(e.name, len(name_ix)) for e in events),
                              np.int32, len(events))
        lanes = list(cols.lanes)
        lane_ix = {ln: i for i, ln in enumerate(lanes)}
        layer_ix: dict[str, int] = {}
        ms = list(doc.layer_markers)
        m_lane = np.array([lane_ix.setdefault(m.cpu_lane, len(lane_ix)) for m in ms], np.int32)
        for ln, i in lane_ix.items():
            if i >= len(lanes):
                lanes.append(ln)
        cols.lanes = lanes
        cols.names = None
        return ColumnarTrace(
            cols=cols, name_id=name_id, names=list(name_ix),
            size_bytes=np.array([-1 if e.size_bytes is None else e.size_bytes for e in events],
                                np.int64),
            n_event_lanes=n_ev_lanes, m_lane=m_lane,
            m_start=np.array([m.start for m in ms], np.int64),
            m_end=np.array([m.end for m in ms], np.int64),
            m_layer=np.array([layer_ix.setdefault(m.layer, len(layer_ix)) for m in ms], np.int32),
            m_phase=np.array([PHASE_CODE[m.phase] for m in ms], np.uint8),
            layers=list(layer_ix), gradient_buckets=doc.gradient_buckets,
            metadata=dict(doc.metadata))

    def to_document(self) -> TraceDocument:
        c = self.cols
        lanes = c.lanes
        ev = []
        for i in range(c.n):
            st = int(c.sync_target[i])
            cr = int(c.correlation[i])
            sz = int(self.size_bytes[i])
            ev.append(TraceEvent(id=int(c.id[i]), kind=KIND_OF_CODE[int(c.kind[i])],
                                 name=self.names[int(self.name_id[i])], lane=lanes[int(c.lane[i])],
                                 start=int(c.start[i]), duration=int(c.duration[i]),
                                 correlation=None if cr < 0 else cr,
                                 size_bytes=None if sz < 0 else sz,
                                 sync_target=None if st < 0 else lanes[st]))
        mk = [LayerMarker(layer=self.layers[int(self.m_layer[j])], phase=PHASES[int(self.m_phase[j])],
                          cpu_lane=lanes[int(self.m_lane[j])], start=int(self.m_start[j]),
                          end=int(self.m_end[j])) for j in range(self.n_markers)]
        return TraceDocument(events=tuple(ev), layer_markers=tuple(mk),
                             gradient_buckets=self.gradient_buckets, metadata=dict(self.metadata))

    def marker_tags(self) -> tuple[np.ndarray, list]:
        """(tag id per marker, tags): tags are the distinct (layer, phase.value)
        pairs in sorted order, the ranking ks_map_layers expects
        (layers.py:41-47 tie-break on (layer, phase.value))."""
        if self.n_markers == 0:
            return np.zeros(0, np.int32), []
        pair = self.m_layer.astype(np.int64) * 3 + self.m_phase
        uniq, inv = np.unique(pair, return_inverse=True)
        keys = [(self.layers[int(u) // 3], PHASES[int(u) % 3].value) for u in uniq]
        order = sorted(range(len(keys)), key=lambda k: keys[k])
        rank = np.empty(len(keys), np.int32)
        rank[order] = np.arange(len(keys), dtype=np.int32)
        return rank[inv].astype(np.int32), [keys[k] for k in order]


# ------------------------------------------------------------------ native I/O

def _strings(h, which: int, count: int, nbytes: int) -> list[str]:
    buf = np.empty(max(nbytes, 1), np.uint8)
    off = np.empty(count + 1, np.int64)
    N.check(N.lib().ks_trace_strings(h, which, buf.ctypes.data, off.ctypes.data), "ks_trace_strings")
    raw = buf.tobytes()
    return [raw[off[i]:off[i + 1]].decode("utf-8", "surrogatepass") for i in range(count)]


def load_trace_columns(text, threads: int | None = None) -> ColumnarTrace:
    """parse_trace into columns (native, multi-threaded host parser)."""
    if isinstance(text, str):
        data = text.encode("utf-8", "surrogatepass")
    else:
        data = bytes(text) if not isinstance(text, bytes) else text
    h = C.c_void_p()
    bad = np.full(2, -1, np.int64)
    rc = N.lib().ks_trace_parse(data, len(data), int(threads or 0), C.byref(h), bad.ctypes.data)
    if rc != N.KS_OK:
        detail = (N.lib().ks_last_error_detail() or b"").decode(errors="replace")
        if rc == N.KS_ERR_MALFORMED:
            raise MalformedDocument(detail)
        if rc == N.KS_ERR_SCHEMA:
            raise SchemaViolation(detail)
        if rc == N.KS_ERR_OVERLAP:
            raise OverlapViolation(detail, int(bad[0]), int(bad[1]))
        N.check(rc, "ks_trace_parse")
    try:
        info = N.TraceInfo()
        N.check(N.lib().ks_trace_get_info(h, C.byref(info)))
        n, m = int(info.n_events), int(info.n_markers)
        a = {"id": np.empty(n, np.int64), "kind": np.empty(n, np.uint8),
             "lane": np.empty(n, np.int32), "start": np.empty(n, np.int64),
             "duration": np.empty(n, np.int64), "correlation": np.empty(n, np.int64),
             "sync_target": np.empty(n, np.int32), "is_dtoh": np.empty(n, np.uint8),
             "name_id": np.empty(n, np.int32), "size_bytes": np.empty(n, np.int64)}
        ec = N.TraceEventCols(**{k: (v.ctypes.data if n else None) for k, v in a.items()})
        N.check(N.lib().ks_trace_events(h, C.byref(ec)))
        mk = {"lane": np.empty(m, np.int32), "start": np.empty(m, np.int64),
              "end": np.empty(m, np.int64), "layer_id": np.empty(m, np.int32),
              "phase": np.empty(m, np.uint8)}
        mc = N.TraceMarkerCols(**{k: (v.ctypes.data if m else None) for k, v in mk.items()})
        N.check(N.lib().ks_trace_markers(h, C.byref(mc)))
        lanes = [LaneId.parse(s) for s in _strings(h, 0, info.n_lanes, info.lane_bytes)]
        names = _strings(h, 1, int(info.n_names), info.name_bytes)
        layers = _strings(h, 2, int(info.n_layers), info.layer_bytes)
        b_off, b_len = int(info.buckets_off), int(info.buckets_len)
        m_off, m_len = int(info.metadata_off), int(info.metadata_len)
    finally:
        N.lib().ks_trace_destroy(h)
    # gradient_buckets then metadata, as parse_trace does (trace.py:317-326)
    buckets = None
    if b_off >= 0:
        raw = json.loads(data[b_off:b_off + b_len])
        if raw is not None:
            buckets = _buckets_from(raw)
    meta = json.loads(data[m_off:m_off + m_len]) if m_off >= 0 else {}
    if not isinstance(meta, dict):
        raise SchemaViolation("metadata must be an object")
    cols = TraceColumns(id=a["id"], kind=a["kind"], lane=a["lane"], start=a["start"],
                        duration=a["duration"], correlation=a["correlation"],
                        sync_target=a["sync_target"], is_dtoh=a["is_dtoh"], lanes=lanes)
    return ColumnarTrace(cols=cols, name_id=a["name_id"], names=names, size_bytes=a["size_bytes"],
                         n_event_lanes=int(info.n_event_lanes), m_lane=mk["lane"],
                         m_start=mk["start"], m_end=mk["end"], m_layer=mk["layer_id"],
                         m_phase=mk["phase"], layers=layers, gradient_buckets=buckets,
                         metadata={str(k): str(v) for k, v in meta.items()})


def _string_table(items: list[str]):
    enc = [s.encode("utf-8", "surrogatepass") for s in items]
    off = np.zeros(len(enc) + 1, np.int64)
    if enc:
        off[1:] = np.cumsum([len(b) for b in enc])
    raw = np.frombuffer(b"".join(enc) or b"\0", np.uint8).copy()
    return raw, off


def dump_trace_columns(ct: ColumnarTrace, threads: int | None = None) -> bytes:
    """Columns -> trace document text (parses back to the same columns)."""
    c = ct.cols
    keep = []

    def arr(x, dt):
        a = np.ascontiguousarray(x, dt)
        keep.append(a)
        return a.ctypes.data if a.size else None

    d = N.TraceWriteDesc()
    d.n_events = c.n
    d.id, d.kind, d.lane = arr(c.id, np.int64), arr(c.kind, np.uint8), arr(c.lane, np.int32)
    d.start, d.duration = arr(c.start, np.int64), arr(c.duration, np.int64)
    d.correlation, d.sync_target = arr(c.correlation, np.int64), arr(c.sync_target, np.int32)
    d.name_id, d.size_bytes = arr(ct.name_id, np.int32), arr(ct.size_bytes, np.int64)
    for pre, items in (("lane", [str(ln) for ln in c.lanes]), ("name", ct.names),
                       ("layer", ct.layers)):
        raw, off = _string_table(items)
        keep += [raw, off]
        setattr(d, f"n_{pre}s", len(items))
        setattr(d, f"{pre}_bytes", raw.ctypes.data)
        setattr(d, f"{pre}_off", off.ctypes.data)
    d.n_markers = ct.n_markers
    d.m_lane, d.m_start, d.m_end = (arr(ct.m_lane, np.int32), arr(ct.m_start, np.int64),
                                    arr(ct.m_end, np.int64))
    d.m_layer, d.m_phase = arr(ct.m_layer, np.int32), arr(ct.m_phase, np.uint8)
    extra = []
    if ct.gradient_buckets is not None:
        gb = ct.gradient_buckets
        extra.append('"gradient_buckets": ' + json.dumps(
            {"bucket_of_layer": dict(gb.bucket_of_layer),
             "bucket_size_bytes": {str(k): v for k, v in gb.bucket_size_bytes.items()}}))
    if ct.metadata:
        extra.append('"metadata": ' + json.dumps(dict(ct.metadata)))
    d.extra_json = ", ".join(extra).encode() if extra else None
    out = C.c_void_p()
    ln = C.c_int64(0)
    N.check(N.lib().ks_trace_write(C.byref(d), int(threads or 0), C.byref(out), C.byref(ln)),
            "ks_trace_write")
    try:
        return C.string_at(out.value, ln.value)
    finally:
        N.lib().ks_buffer_free(out)


# ------------------------------------------------------------ config-5 chain

@dataclass
class ColumnarIngest:
    trace: ColumnarTrace
    ingest: object                 # ingest.IngestResult
    layer_tag: np.ndarray          # int32 per event: index into tags, -1 unmapped
    tags: list                     # (layer, phase.value), "*" -> "_global" at use
    frozen: object | None = None   # frozen.FrozenGraph


def ingest_document(text, *, strict: bool = False, check_overlaps: bool = False,
                    freeze: bool = True, threads: int | None = None,
                    device: int | None = None) -> ColumnarIngest:
    """parse_trace -> build_graph -> map_tasks_to_layers -> freeze, columnar:
    host parse (C++), then device kernels for the joins, layer containment and
    the CSR/topological freeze.  parse_trace already checked lane overlaps."""
    from .ingest import ingest_arrays, map_layers_arrays

    ct = load_trace_columns(text, threads=threads)
    res = ingest_arrays(ct.cols, strict=strict, check_overlaps=check_overlaps, device=device,
                        keep_device=freeze)
    tag_m, tags = ct.marker_tags()
    tag = map_layers_arrays(ct.cols, res.launcher, ct.m_lane, ct.m_start, ct.m_end, tag_m,
                            device=device)
    fz = frozen_from_ingest(ct, res, device=device) if freeze else None
    return ColumnarIngest(trace=ct, ingest=res, layer_tag=tag, tags=tags, frozen=fz)


def ingest_columns(ct: ColumnarTrace, *, strict: bool = False, check_overlaps: bool = True,
                   freeze: bool = True, device: int | None = None) -> ColumnarIngest:
    """ingest_document for columns that did not come through the validating
    reader (e.g. cupti.record()): the device ingest also checks lane overlaps
    (check_lane_overlaps, trace.py:255-265) unless told otherwise."""
    from .ingest import ingest_arrays, map_layers_arrays

    res = ingest_arrays(ct.cols, strict=strict, check_overlaps=check_overlaps, device=device,
                        keep_device=freeze)
    tag_m, tags = ct.marker_tags()
    tag = map_layers_arrays(ct.cols, res.launcher, ct.m_lane, ct.m_start, ct.m_end, tag_m,
                            device=device)
    fz = frozen_from_ingest(ct, res, device=device) if freeze else None
    return ColumnarIngest(trace=ct, ingest=res, layer_tag=tag, tags=tags, frozen=fz)


def frozen_from_ingest(ct: ColumnarTrace, res, device: int | None = None):
    """FrozenGraph straight from ingest output (no DependencyGraph objects)."""
    from .frozen import VDNN_MALLOC_PREFIX, FrozenGraph

    c = ct.cols
    n = c.n
    vdnn_name = np.array([s.startswith(VDNN_MALLOC_PREFIX) for s in ct.names] or [False], bool)
    flags = ((c.kind == KIND_CODE[TaskKind.COMM]).astype(np.uint8) * N.KS_TASK_COMM
             | (vdnn_name[ct.name_id] if n else np.zeros(0, bool)).astype(np.uint8)
             * N.KS_TASK_VDNN_MALLOC)
    dataload = c.kind == KIND_CODE[TaskKind.DATA_LOAD]
    if getattr(res, "handle", None) is not None:  # KeptIngest: freeze on the device
        return FrozenGraph.from_device_ingest(res, ids=c.id, duration=c.duration, lane=c.lane,
                                              lanes=c.lanes, flags=flags, dataload=dataload)
    return FrozenGraph(ids=c.id, duration=c.duration, gap=res.gap, ready=np.zeros(n, np.int64),
                       lane=c.lane, priority=np.zeros(n, np.int32), flags=flags,
                       group=np.zeros(n, np.uint32), edge_src=res.edge_src, edge_dst=res.edge_dst,
                       lane_order_ptr=res.lane_order_ptr, lane_order=res.lane_order,
                       lanes=c.lanes, device=N.env_device() if device is None else device,
                       dataload=dataload)


__all__ = ["ColumnarTrace", "ColumnarIngest", "load_trace_columns", "dump_trace_columns",
           "ingest_document", "ingest_columns", "frozen_from_ingest", "PHASES", "PHASE_CODE"]
