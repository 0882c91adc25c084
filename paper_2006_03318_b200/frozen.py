"""Freeze a DependencyGraph into the device-resident form (include/ddsim.h).

``FrozenGraph`` is the handle every device entry point takes: dense arrays
built from the Python object graph (pkg/src/kernsim/graph.py:75-126) and the
opaque ``ks_graph`` the native compiler returns.  Frozen row ``r`` holds task
``row_ids[r]``; rows ``0 .. n_ordered-1`` are a topological order.
"""

from __future__ import annotations

import ctypes as C
import os
import sys
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .trace import LaneId, TaskKind

VDNN_MALLOC_PREFIX = "cudaMalloc_vdnn"  # scenarios.py:619-622
_T = [0.0]


def _tick(what):
    """DDSIM_INGEST_TIMING=1: wall time of the freeze steps."""
    if not os.environ.get("DDSIM_INGEST_TIMING"):
        return
    t = time.perf_counter()
    if what is not None:
        print(f"[FrozenGraph] {what:14s} {1e3 * (t - _T[0]):8.3f} ms", file=sys.stderr)
    _T[0] = t


@dataclass
class ChainSpec:
    """A permutable chain: members (task ids) on one lane whose order varies
    per scenario; head/tail are the fixed lane neighbours (None = none)."""

    members: list
    head: int | None = None
    tail: int | None = None


class FrozenGraph:
    def __init__(self, *, ids, duration, gap, ready, lane, priority, flags, group, edge_src,
                 edge_dst, lane_order_ptr, lane_order, lanes, chains=None, device=0,
                 task_layers=None, dataload=None):
        if not os.environ.get("DDSIM_COMPILE_ONLY"):
            N.require_device(device)
        _tick(None)
        self.device = device
        self.ids = N.c_i64(ids)                      # dense input index -> external id
        self.n = int(self.ids.shape[0])
        self.lanes: list[LaneId] = list(lanes)
        self.L = len(self.lanes)
        self.duration = N.c_i64(duration)
        self.gap = N.c_i64(gap)
        self.ready = N.c_i64(ready)
        self.lane = N.c_i32(lane)
        self.priority = N.c_i32(priority)
        self.flags = np.ascontiguousarray(flags, dtype=np.uint8)
        self.group = np.ascontiguousarray(group, dtype=np.uint32)
        self.edge_src = N.c_i32(edge_src)
        self.edge_dst = N.c_i32(edge_dst)
        self.task_layers = task_layers    # per input task: layer name or None
        self.dataload = dataload          # per input task: TaskKind.DATA_LOAD
        if self.n < 2 or bool(np.all(self.ids[1:] > self.ids[:-1])):
            rank = np.arange(self.n, dtype=np.int32)  # ids already ascending (document order)
        else:
            rank = np.empty(self.n, np.int32)
            rank[np.argsort(self.ids, kind="stable")] = np.arange(self.n, dtype=np.int32)
        self.id_rank = rank
        self.chains = chains or []
        self._lane_order = (None if lane_order_ptr is None
                            else (N.c_i32(lane_order_ptr), N.c_i32(lane_order)))
        self._replicas: dict = {}
        keep = []
        d = N.GraphDesc()
        d.n_tasks, d.n_lanes = self.n, self.L
        d.duration, d.gap, d.ready_time = N.ptr(self.duration), N.ptr(self.gap), N.ptr(self.ready)
        d.lane, d.id_rank, d.priority = N.ptr(self.lane), N.ptr(self.id_rank), N.ptr(self.priority)
        d.flags, d.group = N.ptr(self.flags), N.ptr(self.group)
        d.n_edges = int(self.edge_src.shape[0])
        d.edge_src, d.edge_dst = N.ptr(self.edge_src), N.ptr(self.edge_dst)
        if lane_order_ptr is not None:
            lop, lo = N.c_i32(lane_order_ptr), N.c_i32(lane_order)
            keep += [lop, lo]
            d.lane_order_ptr = lop.ctypes.data
            d.lane_order = N.ptr(lo) if lo.size else lop.ctypes.data
        if self.chains:
            index = {int(t): i for i, t in enumerate(self.ids)}
            cptr = [0]
            mem, heads, tails = [], [], []
            for ch in self.chains:
                mem += [index[int(m)] for m in ch.members]
                cptr.append(len(mem))
                heads.append(-1 if ch.head is None else index[int(ch.head)])
                tails.append(-1 if ch.tail is None else index[int(ch.tail)])
            arrs = [N.c_i32(cptr), N.c_i32(mem), N.c_i32(heads), N.c_i32(tails)]
            keep += arrs
            d.n_chains = len(self.chains)
            d.chain_ptr, d.chain_member, d.chain_head, d.chain_tail = (a.ctypes.data for a in arrs)
        order = np.empty(self.n, np.int32)
        h = C.c_void_p()
        _tick("host prep")
        N.check(N.lib().ks_graph_create(C.byref(d), device, C.byref(h), N.ptr(order)),
                "ks_graph_create")
        _tick("ks_graph_create")
        self._h = h
        del keep
        chained, n_ordered = C.c_int32(0), C.c_int32(0)
        N.check(N.lib().ks_graph_shape(h, C.byref(chained), C.byref(n_ordered)))
        self._info = None
        self.order = order                         # frozen row -> dense input index
        self._row_ids = None
        self._row_of = None
        self.chained = bool(chained.value)
        self.n_ordered = int(n_ordered.value)
        _tick("post")

    @staticmethod
    def from_device_ingest(kept, *, ids, duration, lane, lanes, flags, dataload) -> "FrozenGraph":
        """The frozen graph of a KeptIngest, compiled on its device
        (ks_graph_create_from_ingest: unique-edge / predecessor CSR by radix
        sort, trace-time topological order verified on every edge, per-row
        arrays gathered on the device).  The host copies of the gaps and edges
        (replicas, parity checks) are fetched from the ingest on first use."""
        fz = FrozenGraph.__new__(FrozenGraph)
        fz.device = kept.device
        fz.ids = N.c_i64(ids)
        fz.n = int(fz.ids.shape[0])
        fz.lanes = list(lanes)
        fz.L = len(fz.lanes)
        fz.duration = N.c_i64(duration)
        fz.ready = np.zeros(fz.n, np.int64)
        fz.lane = N.c_i32(lane)
        fz.priority = np.zeros(fz.n, np.int32)
        fz.flags = np.ascontiguousarray(flags, dtype=np.uint8)
        fz.group = np.zeros(fz.n, np.uint32)
        fz.task_layers = None
        fz.dataload = dataload
        if fz.n < 2 or bool(np.all(fz.ids[1:] > fz.ids[:-1])):
            rank = None
            fz.id_rank = np.arange(fz.n, dtype=np.int32)
        else:
            rank = np.empty(fz.n, np.int32)
            rank[np.argsort(fz.ids, kind="stable")] = np.arange(fz.n, dtype=np.int32)
            fz.id_rank = rank
        fz.chains = []
        fz._replicas = {}
        fz._kept = kept
        order = np.empty(max(fz.n, 1), np.int32)
        h = C.c_void_p()
        _tick("host prep")
        N.check(N.lib().ks_graph_create_from_ingest(kept.handle, N.ptr(rank), N.ptr(fz.flags),
                                                    C.byref(h), N.ptr(order)),
                "ks_graph_create_from_ingest")
        _tick("ks_graph_create_from_ingest")
        fz._h = h
        chained, n_ordered = C.c_int32(0), C.c_int32(0)
        N.check(N.lib().ks_graph_shape(h, C.byref(chained), C.byref(n_ordered)))
        fz._info = None
        fz.order = order[:fz.n]
        fz._row_ids = None
        fz._row_of = None
        fz.chained = bool(chained.value)
        fz.n_ordered = int(n_ordered.value)
        return fz

    def __getattr__(self, name):
        # device-frozen graphs: host copies of the ingest's gaps / edges / lane
        # order on first use
        kept = self.__dict__.get("_kept")
        if kept is not None and name in ("gap", "edge_src", "edge_dst", "_lane_order"):
            val = {"gap": lambda: N.c_i64(kept.gap), "edge_src": lambda: N.c_i32(kept.edge_src),
                   "edge_dst": lambda: N.c_i32(kept.edge_dst),
                   "_lane_order": lambda: (N.c_i32(kept.lane_order_ptr),
                                           N.c_i32(kept.lane_order))}[name]()
            self.__dict__[name] = val
            return val
        raise AttributeError(name)

    @property
    def info(self):
        """ks_graph_info (builds the kernel programs on first use)."""
        if self._info is None:
            info = N.GraphInfo()
            N.check(N.lib().ks_graph_get_info(self._h, C.byref(info)), "ks_graph_get_info")
            self._info = info
        return self._info

    @property
    def row_ids(self) -> np.ndarray:
        """frozen row -> external id"""
        if self._row_ids is None:
            self._row_ids = self.ids[self.order]
        return self._row_ids

    @property
    def row_of(self) -> np.ndarray:
        """dense input index -> frozen row"""
        if self._row_of is None:
            r = np.empty(self.n, np.int32)
            r[self.order] = np.arange(self.n, dtype=np.int32)
            self._row_of = r
        return self._row_of

    @property
    def handle(self):
        return self._h

    def on_device(self, device: int) -> "FrozenGraph":
        """The same frozen graph (same row order) on another device, built once
        and cached -- the per-device replicas of a multi-GPU sweep."""
        if device == self.device:
            return self
        rep = self._replicas.get(device)
        if rep is None:
            lop, lo = self._lane_order if self._lane_order is not None else (None, None)
            rep = FrozenGraph(ids=self.ids, duration=self.duration, gap=self.gap, ready=self.ready,
                              lane=self.lane, priority=self.priority, flags=self.flags,
                              group=self.group, edge_src=self.edge_src, edge_dst=self.edge_dst,
                              lane_order_ptr=lop, lane_order=lo, lanes=self.lanes,
                              chains=self.chains, device=device, task_layers=self.task_layers,
                              dataload=self.dataload)
            if not np.array_equal(rep.order, self.order):
                raise RuntimeError("replica froze to a different row order")
            self._replicas[device] = rep
        return rep

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.lib().ks_graph_destroy(h)
            finally:
                self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    # ---- helpers -----------------------------------------------------------
    def row_dense(self, per_task: np.ndarray) -> np.ndarray:
        """Reorder a per-input-task array into frozen row order."""
        return np.asarray(per_task)[self.order]

    def lanes_of_rows(self) -> np.ndarray:
        return self.lane[self.order]

    def levels(self) -> np.ndarray:
        out = np.empty(self.n, np.int32)
        N.check(N.lib().ks_graph_levels(self._h, N.ptr(out)))
        return out

    def row_classes(self) -> np.ndarray:
        """KS_BD_* per frozen row (breakdown.py:57-67 lane classes; DataLoad
        tasks on CPU lanes flagged separately)."""
        lane_cls = np.array([N.KS_BD_CPU if ln.is_cpu else N.KS_BD_GPU if ln.is_gpu
                             else N.KS_BD_COMM for ln in self.lanes] or [0], np.uint8)
        cls = lane_cls[self.lane[self.order]] if self.n else np.zeros(0, np.uint8)
        if self.dataload is not None:
            dl = np.asarray(self.dataload, bool)[self.order]
            cls = np.where(dl & (cls == N.KS_BD_CPU), N.KS_BD_CPU_DATALOAD, cls).astype(np.uint8)
        return np.ascontiguousarray(cls, np.uint8)

    def unordered_ids(self) -> list[int]:
        return sorted(int(i) for i in self.row_ids[self.n_ordered:])

    # ---- construction from the object graph -----------------------------------
    @staticmethod
    def from_graph(graph, *, group_of=None, chains=None, device=None) -> "FrozenGraph":
        """Freeze a kernsim-style DependencyGraph (tasks / edges / lane_order)."""
        if device is None:
            device = N.env_device()
        tasks = graph.tasks
        ids = np.fromiter(tasks.keys(), np.int64, len(tasks))
        index = {tid: i for i, tid in enumerate(tasks.keys())}
        lane_ix: dict = {}
        lanes: list = []
        lane = np.empty(len(tasks), np.int32)
        for i, t in enumerate(tasks.values()):
            j = lane_ix.get(t.lane)
            if j is None:
                j = lane_ix[t.lane] = len(lanes)
                lanes.append(t.lane)
            lane[i] = j
        vals = list(tasks.values())
        n = len(vals)
        duration = np.fromiter((t.duration for t in vals), np.int64, n)
        gap = np.fromiter((t.gap for t in vals), np.int64, n)
        ready = np.fromiter((t.ready_time for t in vals), np.int64, n)
        prio = np.fromiter((t.priority for t in vals), np.int32, n)
        flags = np.fromiter(((N.KS_TASK_COMM if t.kind is TaskKind.COMM else 0)
                             | (N.KS_TASK_VDNN_MALLOC if t.name.startswith(VDNN_MALLOC_PREFIX)
                                else 0) for t in vals), np.uint8, n)
        group = np.zeros(n, np.uint32) if group_of is None else np.asarray(group_of, np.uint32)
        E = len(graph.edges)
        src = np.empty(E, np.int32)
        dst = np.empty(E, np.int32)
        for k, (u, v, _kind) in enumerate(graph.edges):
            src[k] = index[u]
            dst[k] = index[v]
        # lane_order -> per-lane index lists; anything inconsistent => unchained
        chain_members = set()
        for ch in chains or []:
            chain_members.update(ch.members)
        lop = None
        lo: list = []
        ok = True
        per_lane: list[list[int]] = [[] for _ in lanes]
        for ln, ids_on in graph.lane_order.items():
            j = lane_ix.get(ln)
            if j is None:
                if ids_on:
                    ok = False
                continue
            for tid in ids_on:
                i = index.get(tid)
                if i is None:
                    ok = False
                    break
                per_lane[j].append(i)
        if ok:
            lop = [0]
            for j in range(len(lanes)):
                lo += per_lane[j]
                lop.append(len(lo))
        layers = [t.layer[0] if t.layer is not None else None for t in vals]
        dataload = np.fromiter((t.kind is TaskKind.DATA_LOAD for t in vals), bool, n)
        return FrozenGraph(ids=ids, duration=duration, gap=gap, ready=ready, lane=lane,
                           priority=prio, flags=flags, group=group, edge_src=src, edge_dst=dst,
                           lane_order_ptr=lop, lane_order=lo, lanes=lanes, chains=chains,
                           device=device, task_layers=layers, dataload=dataload)

    def toposort(self) -> tuple[list[int], bool]:
        """verify_acyclic order (smallest-id Kahn) computed on the device."""
        out = np.empty(max(self.n, 1), np.int32)
        nout = C.c_int32(0)
        rc = N.lib().ks_toposort(self._h, N.ptr(out), C.byref(nout))
        if rc not in (N.KS_OK, N.KS_ERR_CYCLE):
            N.check(rc, "ks_toposort")
        k = int(nout.value)
        return [int(x) for x in self.ids[out[:k]]], rc == N.KS_OK
