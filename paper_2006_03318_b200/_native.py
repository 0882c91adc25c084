"""ctypes binding of libddsim.so (the C-ABI in include/ddsim.h).

This is the only module that touches the native library.  There is no CPU
fallback: if the library is missing or no CUDA device is visible, every
compute entry point raises (``NoDevice`` / ``RuntimeError``) instead of
silently running something else.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from . import errors

LIB_NAME = "libddsim.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

# status codes (include/ddsim.h)
KS_OK = 0
KS_ERR_DEADLOCK = 1
KS_ERR_CYCLE = 2
KS_ERR_INVALID = 3
KS_ERR_CUDA = 4
KS_ERR_OOM = 5
KS_ERR_UNSUPPORTED = 6
KS_ERR_ORPHAN = 7
KS_ERR_AMBIGUOUS = 8
KS_ERR_OVERLAP = 9
KS_ERR_BAD_PIPELINE = 10
KS_ERR_NO_DEVICE = 11
KS_ERR_MALFORMED = 12
KS_ERR_SCHEMA = 13

KS_POLICY_DEFAULT, KS_POLICY_PRIORITY, KS_POLICY_VDNN = 0, 1, 2
KS_PATH_AUTO, KS_PATH_MAXPLUS, KS_PATH_LISTSCHED = 0, 1, 2
KS_TASK_COMM, KS_TASK_VDNN_MALLOC = 1, 2

P = C.c_void_p


class GraphDesc(C.Structure):
    _fields_ = [
        ("n_tasks", C.c_int32), ("n_lanes", C.c_int32),
        ("duration", P), ("gap", P), ("ready_time", P), ("lane", P), ("id_rank", P),
        ("priority", P), ("flags", P), ("group", P),
        ("n_edges", C.c_int64), ("edge_src", P), ("edge_dst", P),
        ("lane_order_ptr", P), ("lane_order", P),
        ("n_chains", C.c_int32), ("chain_ptr", P), ("chain_member", P),
        ("chain_head", P), ("chain_tail", P),
    ]


class GraphInfo(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "n_tasks", "n_lanes", "n_edges_unique", "chained", "n_ordered", "n_slots",
        "n_slots_smem", "n_levels", "has_lanes", "n_lane_slots_smem", "n_lane_slots_global",
        "n_lane_cuts", "seg_chain_begin", "seg_chain_end", "n_carries")]


class ScaleStep(C.Structure):
    _fields_ = [("group_lo", C.c_int32), ("group_hi", C.c_int32),
                ("num", C.c_int64), ("den", C.c_int64)]


SCALE_STEP_DTYPE = np.dtype([("group_lo", "<i4"), ("group_hi", "<i4"),
                             ("num", "<i8"), ("den", "<i8")], align=True)


class ScenariosDesc(C.Structure):
    _fields_ = [
        ("n_scenarios", C.c_int32), ("dense_kind", C.c_int32), ("dense", P), ("dense_ld", C.c_int64),
        ("n_overrides", C.c_int32), ("override_task", P), ("override", P),
        ("scale_ptr", P), ("scale", P),
        ("chain_perm", P), ("perm_ld", C.c_int32), ("chain_present", P),
        ("vdnn_rank", P),
    ]


class SimOut(C.Structure):
    _fields_ = [("start", P), ("start_ld", C.c_int64), ("makespan", P), ("lane_busy", P),
                ("schedule", P), ("dispatched", P)]


class BreakdownDesc(C.Structure):
    _fields_ = [("row_class", P), ("comm_as_gpu", C.c_int32), ("dataload_as_cpu", C.c_int32),
                ("gaps_as_cpu_busy", C.c_int32), ("row_layer", P), ("n_layers", C.c_int32),
                ("schedule", P)]


KS_BD_CPU, KS_BD_GPU, KS_BD_COMM, KS_BD_CPU_DATALOAD = 0, 1, 2, 3


class TraceCols(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("id", P), ("kind", P), ("lane", P), ("start", P), ("duration", P),
        ("correlation", P), ("sync_target", P), ("is_dtoh", P),
        ("n_lanes", C.c_int32), ("lane_class", P), ("lane_rank", P), ("strict", C.c_int32),
    ]


class IngestOut(C.Structure):
    _fields_ = [
        ("edge_cap", C.c_int64), ("n_edges", C.c_int64), ("edge_src", P), ("edge_dst", P),
        ("edge_kind", P), ("lane_order", P), ("lane_order_ptr", P), ("gap", P), ("launcher", P),
        ("bad_a", C.c_int64), ("bad_b", C.c_int64),
    ]


class MarkerCols(C.Structure):
    _fields_ = [("n", C.c_int64), ("lane", P), ("start", P), ("end", P), ("tag", P)]


class TraceInfo(C.Structure):
    _fields_ = [
        ("n_events", C.c_int64), ("n_lanes", C.c_int32), ("n_event_lanes", C.c_int32),
        ("n_names", C.c_int64), ("n_markers", C.c_int64), ("n_layers", C.c_int32),
        ("lane_bytes", C.c_int64), ("name_bytes", C.c_int64), ("layer_bytes", C.c_int64),
        ("buckets_off", C.c_int64), ("buckets_len", C.c_int64),
        ("metadata_off", C.c_int64), ("metadata_len", C.c_int64),
    ]


class TraceEventCols(C.Structure):
    _fields_ = [(n, P) for n in ("id", "kind", "lane", "start", "duration", "correlation",
                                 "sync_target", "is_dtoh", "name_id", "size_bytes")]


class TraceMarkerCols(C.Structure):
    _fields_ = [(n, P) for n in ("lane", "start", "end", "layer_id", "phase")]


class TraceWriteDesc(C.Structure):
    _fields_ = [
        ("n_events", C.c_int64), ("id", P), ("kind", P), ("lane", P), ("start", P),
        ("duration", P), ("correlation", P), ("sync_target", P), ("name_id", P),
        ("size_bytes", P),
        ("n_lanes", C.c_int32), ("lane_bytes", P), ("lane_off", P),
        ("n_names", C.c_int64), ("name_bytes", P), ("name_off", P),
        ("n_markers", C.c_int64), ("m_lane", P), ("m_start", P), ("m_end", P),
        ("m_layer", P), ("m_phase", P),
        ("n_layers", C.c_int32), ("layer_bytes", P), ("layer_off", P),
        ("extra_json", C.c_char_p),
    ]


# name, restype, argtypes
_SIGNATURES = [
    ("ks_graph_create", C.c_int, [C.POINTER(GraphDesc), C.c_int, C.POINTER(P), P]),
    ("ks_graph_get_info", C.c_int, [P, C.POINTER(GraphInfo)]),
    ("ks_ingest_keep", C.c_int, [C.POINTER(TraceCols), C.c_int, C.c_int, C.POINTER(IngestOut),
                                 C.POINTER(C.c_void_p)]),
    ("ks_ingest_dev_copy", C.c_int, [P, P, P, P, P, P]),
    ("ks_ingest_dev_free", None, [P]),
    ("ks_graph_create_from_ingest", C.c_int, [P, P, P, C.POINTER(C.c_void_p), P]),
    ("ks_graph_shape", C.c_int, [P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    ("ks_graph_levels", C.c_int, [P, P]),
    ("ks_graph_destroy", C.c_int, [P]),
    ("ks_simulate", C.c_int, [P, C.POINTER(ScenariosDesc), C.c_int, C.c_int, C.POINTER(SimOut), P]),
    ("ks_simulate_host", C.c_int, [P, C.POINTER(ScenariosDesc), C.c_int, C.c_int, C.POINTER(SimOut)]),
    ("ks_simulate_host_multi", C.c_int, [P, C.c_int, C.POINTER(ScenariosDesc), C.c_int, C.c_int,
                                         C.POINTER(SimOut)]),
    ("ks_toposort", C.c_int, [P, P, C.POINTER(C.c_int32)]),
    ("ks_breakdown", C.c_int, [P, C.POINTER(ScenariosDesc), P, C.c_int64, P,
                               C.POINTER(BreakdownDesc), P, P, P]),
    ("ks_ingest", C.c_int, [C.POINTER(TraceCols), C.c_int, C.c_int, C.POINTER(IngestOut)]),
    ("ks_map_layers", C.c_int, [C.POINTER(TraceCols), P, C.POINTER(MarkerCols), C.c_int, P, P]),
    ("ks_trace_parse", C.c_int, [C.c_char_p, C.c_int64, C.c_int, C.POINTER(P), P]),
    ("ks_trace_get_info", C.c_int, [P, C.POINTER(TraceInfo)]),
    ("ks_trace_events", C.c_int, [P, C.POINTER(TraceEventCols)]),
    ("ks_trace_markers", C.c_int, [P, C.POINTER(TraceMarkerCols)]),
    ("ks_trace_strings", C.c_int, [P, C.c_int, P, P]),
    ("ks_trace_destroy", None, [P]),
    ("ks_cupti_start", C.c_int, []),
    ("ks_cupti_stop", C.c_int, [C.POINTER(P)]),
    ("ks_cupti_info_get", C.c_int, [P, C.POINTER(TraceInfo), P, P]),
    ("ks_cupti_events", C.c_int, [P, C.POINTER(TraceEventCols)]),
    ("ks_cupti_markers", C.c_int, [P, C.POINTER(TraceMarkerCols)]),
    ("ks_cupti_strings", C.c_int, [P, C.c_int, P, P]),
    ("ks_cupti_destroy", None, [P]),
    ("ks_trace_write", C.c_int, [C.POINTER(TraceWriteDesc), C.c_int, C.POINTER(P),
                                 C.POINTER(C.c_int64)]),
    ("ks_buffer_free", None, [P]),
    ("ks_error_name", C.c_char_p, [C.c_int]),
    ("ks_last_error_detail", C.c_char_p, []),
    ("ks_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("ks_launch_count", C.c_int64, []),
    ("ks_version", C.c_char_p, []),
    ("ks_jit_log", C.c_char_p, []),
    ("ks_probe_widen", C.c_int, [P, P, C.c_int64, P]),
]
EXPORTED_SYMBOLS = [s[0] for s in _SIGNATURES]

_lib = None
_lock = threading.Lock()


def lib():
    """Load libddsim.so once; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"native library {LIB_PATH} is missing; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
            h = C.CDLL(str(LIB_PATH))
            for name, res, args in _SIGNATURES:
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def device_count() -> int:
    n = C.c_int(0)
    lib().ks_device_count(C.byref(n))
    return int(n.value)


def launch_count() -> int:
    return int(lib().ks_launch_count())


_ERROR_CLASS = {
    KS_ERR_DEADLOCK: "Deadlock",
    KS_ERR_CYCLE: "CycleDetected",
    KS_ERR_CUDA: "CudaError",
    KS_ERR_OOM: "OutOfMemory",
    KS_ERR_UNSUPPORTED: "Unsupported",
    KS_ERR_ORPHAN: "OrphanKernel",
    KS_ERR_AMBIGUOUS: "AmbiguousMarker",
    KS_ERR_BAD_PIPELINE: "BadPipeline",
    KS_ERR_NO_DEVICE: "NoDevice",
    KS_ERR_MALFORMED: "MalformedDocument",
    KS_ERR_SCHEMA: "SchemaViolation",
}


def check(rc: int, what: str = "") -> None:
    """Raise the KernsimError named by a C-ABI status code."""
    if rc == KS_OK:
        return
    detail = (lib().ks_last_error_detail() or b"").decode(errors="replace")
    msg = f"{what}: {detail}" if what else detail
    if rc == KS_ERR_INVALID:
        raise ValueError(msg)
    if rc == KS_ERR_OVERLAP:
        raise errors.OverlapViolation(msg, -1, -1)
    if rc == KS_ERR_CYCLE:
        raise errors.CycleDetected(msg, [])
    cls = getattr(errors, _ERROR_CLASS.get(rc, "KernsimError"))
    raise cls(msg)


def require_device(device: int = 0) -> None:
    n = device_count()
    if n == 0:
        raise errors.NoDevice("no CUDA device visible; the simulator has no CPU fallback")
    if device < 0 or device >= n:
        raise errors.NoDevice(f"device {device} not present ({n} visible)")


def ptr(a) -> int | None:
    """Address of a numpy array / torch tensor (None for None)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data if a.size else None
    return a.data_ptr()  # torch.Tensor


def c_i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def c_i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def env_device() -> int:
    return int(os.environ.get("DDSIM_DEVICE", "0"))
