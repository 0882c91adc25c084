"""Trace collection with CUPTI: this process's CUDA activity recorded straight
into trace columns (the schema of kernsim.trace, pkg/src/kernsim/trace.py:20-90;
the reference reads it from JSON only, trace.py:281-328).

    from paper_2006_03318_b200 import cupti
    with cupti.record() as rec:
        train_step()                  # NVTX ranges "<layer>/<Forward|Backward|WeightUpdate>"
    ct = rec.trace                    # ColumnarTrace
    ci = columnar.ingest_columns(ct)  # device ingest -> layers -> frozen graph

Runtime API calls become CpuApi events on "cpu:<thread>" (Sync when CUPTI saw
them block: stream synchronise targets that stream, context / event
synchronise every GPU lane), kernels GpuKernel and copies / memsets GpuMemcpy
on "gpu:<device>:<stream>", joined by CUPTI's correlation ids (rule 3).  A
synchronous cudaMemcpy* whose copy is device-to-host is named
"memcpy_dtoh:<api>" (rule 4's dtoh link).  ``columnar.dump_trace_columns``
writes the reference's JSON document from the result.  Host C++
(csrc/cupti_trace.cu); libcupti is loaded at run time.
"""

from __future__ import annotations

import ctypes as C
from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .columnar import ColumnarTrace
from .trace import LaneId, TraceColumns


def start() -> None:
    """Begin recording (one recording per process at a time)."""
    N.check(N.lib().ks_cupti_start(), "ks_cupti_start")


def _strings(h, which: int, count: int, nbytes: int) -> list[str]:
    buf = np.empty(max(nbytes, 1), np.uint8)
    off = np.empty(count + 1, np.int64)
    N.check(N.lib().ks_cupti_strings(h, which, buf.ctypes.data, off.ctypes.data), "ks_cupti_strings")
    raw = buf.tobytes()
    return [raw[off[i]:off[i + 1]].decode("utf-8", "replace") for i in range(count)]


def stop() -> ColumnarTrace:
    """Stop recording; the activity since start() as a ColumnarTrace (times in
    ns from the first record; metadata["t0_ns"] = that record's CUPTI time)."""
    h = C.c_void_p()
    N.check(N.lib().ks_cupti_stop(C.byref(h)), "ks_cupti_stop")
    try:
        info = N.TraceInfo()
        t0, dropped = np.zeros(1, np.int64), np.zeros(1, np.int64)
        N.check(N.lib().ks_cupti_info_get(h, C.byref(info), t0.ctypes.data, dropped.ctypes.data))
        n, m = int(info.n_events), int(info.n_markers)
        a = {"id": np.empty(n, np.int64), "kind": np.empty(n, np.uint8),
             "lane": np.empty(n, np.int32), "start": np.empty(n, np.int64),
             "duration": np.empty(n, np.int64), "correlation": np.empty(n, np.int64),
             "sync_target": np.empty(n, np.int32), "is_dtoh": np.empty(n, np.uint8),
             "name_id": np.empty(n, np.int32), "size_bytes": np.empty(n, np.int64)}
        ec = N.TraceEventCols(**{k: (v.ctypes.data if n else None) for k, v in a.items()})
        N.check(N.lib().ks_cupti_events(h, C.byref(ec)))
        mk = {"lane": np.empty(m, np.int32), "start": np.empty(m, np.int64),
              "end": np.empty(m, np.int64), "layer_id": np.empty(m, np.int32),
              "phase": np.empty(m, np.uint8)}
        mc = N.TraceMarkerCols(**{k: (v.ctypes.data if m else None) for k, v in mk.items()})
        N.check(N.lib().ks_cupti_markers(h, C.byref(mc)))
        lanes = [LaneId.parse(s) for s in _strings(h, 0, int(info.n_lanes), int(info.lane_bytes))]
        names = _strings(h, 1, int(info.n_names), int(info.name_bytes))
        layers = _strings(h, 2, int(info.n_layers), int(info.layer_bytes))
    finally:
        N.lib().ks_cupti_destroy(h)
    cols = TraceColumns(id=a["id"], kind=a["kind"], lane=a["lane"], start=a["start"],
                        duration=a["duration"], correlation=a["correlation"],
                        sync_target=a["sync_target"], is_dtoh=a["is_dtoh"], lanes=lanes,
                        names=[names[i] for i in a["name_id"].tolist()] if n else [])
    return ColumnarTrace(cols=cols, name_id=a["name_id"], names=names, size_bytes=a["size_bytes"],
                         n_event_lanes=int(info.n_event_lanes), m_lane=mk["lane"],
                         m_start=mk["start"], m_end=mk["end"], m_layer=mk["layer_id"],
                         m_phase=mk["phase"], layers=layers, gradient_buckets=None,
                         metadata={"source": "cupti", "t0_ns": str(int(t0[0])),
                                   "dropped_records": str(int(dropped[0]))})


@dataclass
class Recording:
    trace: ColumnarTrace | None = None


@contextmanager
def record():
    """Record the CUDA activity of the block; ``.trace`` after it exits."""
    rec = Recording()
    start()
    try:
        yield rec
    finally:
        rec.trace = stop()


__all__ = ["start", "stop", "record", "Recording"]
