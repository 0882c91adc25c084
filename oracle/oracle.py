"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of the C oracle (ddsim_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) import this module, always as the checker / CPU
baseline, never as part of the product path.

The oracle restates the reference algorithms (see the header of
ddsim_oracle.c for file:line citations).  It is pinned against golden vectors
produced by the reference itself (tests/golden/make_golden.py ->
tests/golden/golden.json.gz) in tests/test_oracle_pinned.py.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "ddsim_oracle.c"
LIB = HERE / "liboracle.so"

POL = {"default": 0, "priority": 1, "vdnn_prefetch": 2}
F_COMM, F_VDNN_MALLOC = 1, 2


class _OraGraph(C.Structure):
    _fields_ = [("n", C.c_int), ("L", C.c_int),
                ("dur", C.c_void_p), ("gap", C.c_void_p), ("ready", C.c_void_p),
                ("lane", C.c_void_p), ("rank", C.c_void_p), ("prio", C.c_void_p),
                ("vrank", C.c_void_p), ("flags", C.c_void_p),
                ("E", C.c_int64), ("src", C.c_void_p), ("dst", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
            subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-o", str(LIB), str(SRC),
                            "-lpthread"], check=True)
        h = C.CDLL(str(LIB))
        P = C.c_void_p
        h.ora_simulate.argtypes = [C.POINTER(_OraGraph), C.c_int, P, P, P, P]
        h.ora_simulate.restype = C.c_int
        h.ora_toposort.argtypes = [C.POINTER(_OraGraph), P]
        h.ora_toposort.restype = C.c_int
        h.ora_longest_path.argtypes = [C.POINTER(_OraGraph), P, P]
        h.ora_longest_path.restype = C.c_int
        h.ora_scale.argtypes = [C.c_int64, C.c_int64, C.c_int64]
        h.ora_scale.restype = C.c_int64
        h.ora_simulate_batch.argtypes = [C.POINTER(_OraGraph), P, C.c_int64, C.c_int, C.c_int,
                                         C.c_int, P, P]
        h.ora_simulate_batch.restype = C.c_int64
        _lib = h
    return _lib


@dataclass
class OracleGraph:
    """Dense arrays of a kernsim-shaped graph (tasks dict / edges set)."""

    ids: np.ndarray
    lanes: list
    dur: np.ndarray
    gap: np.ndarray
    ready: np.ndarray
    lane: np.ndarray
    rank: np.ndarray
    prio: np.ndarray
    flags: np.ndarray
    vrank: np.ndarray
    src: np.ndarray
    dst: np.ndarray

    @staticmethod
    def from_graph(graph, conv_order: list | None = None) -> "OracleGraph":
        tids = list(graph.tasks)
        index = {t: i for i, t in enumerate(tids)}
        lanes: list = []
        lane_ix: dict = {}
        lane = []
        for t in graph.tasks.values():
            if t.lane not in lane_ix:
                lane_ix[t.lane] = len(lanes)
                lanes.append(t.lane)
            lane.append(lane_ix[t.lane])
        ids = np.array(tids, np.int64)
        rank = np.empty(len(tids), np.int32)
        rank[np.argsort(ids, kind="stable")] = np.arange(len(tids), dtype=np.int32)
        vals = list(graph.tasks.values())
        conv = list(conv_order or [])

        def vr(t):
            if t.layer is None or t.layer[0] not in conv:
                return -1
            return conv.index(t.layer[0])

        edges = list(graph.edges)
        return OracleGraph(
            ids=ids, lanes=lanes,
            dur=np.array([t.duration for t in vals], np.int64),
            gap=np.array([t.gap for t in vals], np.int64),
            ready=np.array([t.ready_time for t in vals], np.int64),
            lane=np.array(lane, np.int32), rank=rank,
            prio=np.array([t.priority for t in vals], np.int32),
            flags=np.array([(F_COMM if t.kind.value == "Comm" else 0)
                            | (F_VDNN_MALLOC if t.name.startswith("cudaMalloc_vdnn") else 0)
                            for t in vals], np.uint8),
            vrank=np.array([vr(t) for t in vals], np.int32),
            src=np.array([index[u] for u, _, _ in edges], np.int32),
            dst=np.array([index[v] for _, v, _ in edges], np.int32),
        )

    def _c(self) -> _OraGraph:
        g = _OraGraph()
        g.n, g.L = len(self.ids), max(len(self.lanes), 1)
        for name in ("dur", "gap", "ready", "lane", "rank", "prio", "vrank", "flags", "src", "dst"):
            arr = getattr(self, name)
            setattr(g, name, arr.ctypes.data if arr.size else None)
        g.E = len(self.src)
        return g

    def simulate(self, policy: str = "default", dur: np.ndarray | None = None):
        """-> (start_of dict, makespan, lane_busy dict, trace list) or raises
        RuntimeError('Deadlock') like sim.py:132-135."""
        g = self._c()
        keep = None
        if dur is not None:
            keep = np.ascontiguousarray(dur, np.int64)
            g.dur = keep.ctypes.data
        n = len(self.ids)
        start = np.zeros(max(n, 1), np.int64)
        trace = np.zeros(max(n, 1), np.int32)
        lb = np.zeros(max(len(self.lanes), 1), np.int64)
        ms = np.zeros(1, np.int64)
        done = lib().ora_simulate(C.byref(g), POL[policy], start.ctypes.data, trace.ctypes.data,
                                  lb.ctypes.data, ms.ctypes.data)
        if done != n:
            raise RuntimeError("Deadlock")
        ids = self.ids
        start_of = {int(ids[i]): int(start[i]) for i in range(n)}
        used = set(self.lane.tolist())
        lane_busy = {self.lanes[j]: int(lb[j]) for j in range(len(self.lanes)) if j in used}
        tr = [(int(ids[i]), int(start[i])) for i in trace[:n]]
        del keep
        return start_of, int(ms[0]), lane_busy, tr

    def simulate_raw(self, policy: str = "default") -> int:
        """Alg. 1 with the results left in arrays (the CPU-baseline timing
        path: the ctypes call releases the GIL, so threads run scenarios in
        parallel).  Returns the makespan."""
        g = self._c()
        n = len(self.ids)
        start = np.zeros(max(n, 1), np.int64)
        trace = np.zeros(max(n, 1), np.int32)
        lb = np.zeros(max(len(self.lanes), 1), np.int64)
        ms = np.zeros(1, np.int64)
        if lib().ora_simulate(C.byref(g), POL[policy], start.ctypes.data, trace.ctypes.data,
                              lb.ctypes.data, ms.ctypes.data) != n:
            raise RuntimeError("Deadlock")
        return int(ms[0])

    def toposort(self) -> list[int]:
        g = self._c()
        n = len(self.ids)
        out = np.zeros(max(n, 1), np.int32)
        k = lib().ora_toposort(C.byref(g), out.ctypes.data)
        return [int(self.ids[i]) for i in out[:k]]

    def longest_path(self) -> int:
        g = self._c()
        n = len(self.ids)
        start = np.zeros(max(n, 1), np.int64)
        ms = np.zeros(1, np.int64)
        lib().ora_longest_path(C.byref(g), start.ctypes.data, ms.ctypes.data)
        return int(ms[0])

    def simulate_batch(self, dense: np.ndarray, threads: int, policy: str = "default",
                       want_start: bool = False):
        """dense: int32 [n][ld] durations (task order of this object)."""
        g = self._c()
        S = dense.shape[1]
        ms = np.zeros(S, np.int64)
        start = np.zeros(dense.shape, np.int64) if want_start else None
        upd = lib().ora_simulate_batch(C.byref(g), dense.ctypes.data, dense.shape[1], S,
                                       POL[policy], threads, ms.ctypes.data,
                                       None if start is None else start.ctypes.data)
        return ms, start, int(upd)


def scale(d: int, num: int, den: int) -> int:
    return int(lib().ora_scale(d, num, den))


class _OraTrace(C.Structure):
    _fields_ = [("n", C.c_int64), ("id", C.c_void_p), ("start", C.c_void_p), ("dur", C.c_void_p),
                ("corr", C.c_void_p), ("kind", C.c_void_p), ("is_dtoh", C.c_void_p),
                ("lane", C.c_void_p), ("sync_target", C.c_void_p), ("n_lanes", C.c_int32),
                ("lane_class", C.c_void_p)]


def _trace_struct(cols):
    keep = {
        "id": np.ascontiguousarray(cols.id, np.int64), "start": np.ascontiguousarray(cols.start, np.int64),
        "dur": np.ascontiguousarray(cols.duration, np.int64),
        "corr": np.ascontiguousarray(cols.correlation, np.int64),
        "kind": np.ascontiguousarray(cols.kind, np.uint8),
        "is_dtoh": np.ascontiguousarray(cols.is_dtoh, np.uint8),
        "lane": np.ascontiguousarray(cols.lane, np.int32),
        "sync_target": np.ascontiguousarray(cols.sync_target, np.int32),
        "lane_class": np.ascontiguousarray(cols.lane_class_codes(), np.uint8),
    }
    t = _OraTrace()
    t.n = int(cols.n)
    t.n_lanes = len(cols.lanes)
    for k, a in keep.items():
        setattr(t, k, a.ctypes.data if a.size else None)
    return t, keep


def build_graph_columns(cols):
    """-> (edge set {(src_idx, dst_idx, kind_code)}, gap[n], launcher[n])."""
    h = lib()
    h.ora_build_graph.argtypes = [C.POINTER(_OraTrace)] + [C.c_void_p] * 5
    h.ora_build_graph.restype = C.c_int64
    t, keep = _trace_struct(cols)
    n = max(int(cols.n), 1)
    cap = 3 * n + int(np.sum(cols.kind == 6)) * (len(cols.lanes) + 1) + 16
    s, d, k = np.empty(cap, np.int32), np.empty(cap, np.int32), np.empty(cap, np.uint8)
    gap, launcher = np.empty(n, np.int64), np.empty(n, np.int32)
    m = h.ora_build_graph(C.byref(t), s.ctypes.data, d.ctypes.data, k.ctypes.data,
                          gap.ctypes.data, launcher.ctypes.data)
    del keep
    return set(zip(s[:m].tolist(), d[:m].tolist(), k[:m].tolist())), gap[:cols.n], launcher[:cols.n]


def map_layers_columns(cols, launcher, m_lane, m_start, m_end, m_tag):
    h = lib()
    h.ora_map_layers.argtypes = [C.POINTER(_OraTrace), C.c_void_p, C.c_int64] + [C.c_void_p] * 5
    h.ora_map_layers.restype = C.c_int64
    t, keep = _trace_struct(cols)
    arrs = [np.ascontiguousarray(m_lane, np.int32), np.ascontiguousarray(m_start, np.int64),
            np.ascontiguousarray(m_end, np.int64), np.ascontiguousarray(m_tag, np.int32)]
    la = np.ascontiguousarray(launcher, np.int32)
    out = np.full(max(int(cols.n), 1), -1, np.int32)
    bad = h.ora_map_layers(C.byref(t), la.ctypes.data, len(arrs[0]),
                           *[a.ctypes.data if a.size else None for a in arrs], out.ctypes.data)
    del keep
    return out[:cols.n], int(bad)
