"""Batched simulation: many what-if scenarios of one frozen graph at once.

This is the additive API that replaces the reference's per-scenario loop
(``kernsim sweep``: copy -> apply_pipeline -> simulate per point,
pkg/src/kernsim/cli.py:185-193).  A scenario is a row of a table:

* dense durations   dur[r][s] for every frozen row r (Monte-Carlo jitter),
* overrides         per-scenario durations of a few tasks (set_duration),
* scale programs    sequential half-up Shrink steps on task groups
                    (scale_durations, transform.py:174-183); a step whose
                    factor is ``REMOVE`` removes the group's tasks instead
                    (remove_task, transform.py:249-265),
* chains            per-scenario order / presence of inserted tasks on one
                    lane (sequenced insert_task, transform.py:204-246).

Compilers below turn the reference's sweeps (AMP, per-layer Shrink,
data-parallel bandwidth x workers x bucket order) into such tables; the
device evaluates all scenarios in one launch (maxplus_sim).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _native as N
from .comm import COLLECTIVE_LANE, NetworkConfig, allreduce_duration, earliest_weight_update_task
from .comm import last_backward_gpu_task
from .errors import BadPipeline, Deadlock, MissingLayer, NoWeightUpdate, Unsupported
from .frozen import ChainSpec, FrozenGraph
from .graph import DependencyGraph, EdgeKind, Task
from .trace import GradientBucketMap, TaskKind
from .transform import Selector, TransformPipeline

REMOVE = "remove"  # a compile_scale_sweep factor: remove the selected tasks

POLICY_IDS = {"default": N.KS_POLICY_DEFAULT, "priority": N.KS_POLICY_PRIORITY,
              "vdnn_prefetch": N.KS_POLICY_VDNN}


@dataclass
class BatchResult:
    frozen: FrozenGraph
    makespan: np.ndarray                 # [S] int64
    lane_busy: np.ndarray | None         # [S][L] int64
    start: np.ndarray | None             # [rows][S] int64 (frozen rows), -1 = absent
    schedule: np.ndarray | None = None   # [S][N] frozen rows in dispatch order
    parts: np.ndarray | None = None      # [S][4] cpu_only, gpu_only, parallel, idle
    layer_busy: np.ndarray | None = None # [n_layers][2][S] per-layer cpu / gpu ns
    layer_names: list | None = None

    def start_of(self, s: int) -> dict[int, int]:
        col = self.start[:, s]
        ids = self.frozen.row_ids
        keep = col >= 0
        return dict(zip(ids[keep].tolist(), col[keep].tolist()))

    def lane_busy_of(self, s: int, present_lanes=None) -> dict:
        """lane_busy dict of scenario s keyed like sim.py:124 (lanes that still
        hold a task: absent chains and removed tasks drop out)."""
        fz = self.frozen
        used = np.zeros(fz.L, bool)
        if present_lanes is None and self.start is not None:
            used[fz.lane[fz.order][self.start[:, s] >= 0]] = True
        elif present_lanes is None:
            used[fz.lane] = True
        else:
            used[list(present_lanes)] = True
        return {fz.lanes[j]: int(self.lane_busy[s, j]) for j in range(fz.L) if used[j]}


    def breakdown_of(self, s: int):
        """compute_breakdown (breakdown.py:42-98) of scenario s as the
        reference's BreakdownReport, from the device-computed parts."""
        from .breakdown import BreakdownReport
        if self.parts is None:
            raise ValueError("simulate_batch(..., breakdown=True) computes the breakdown")
        c, g, par, idle = (int(x) for x in self.parts[s])
        if c < 0:
            raise Unsupported(f"scenario {s}: lane intervals not in lane order (negative durations)")
        per_layer = {}
        if self.layer_busy is not None:
            fz = self.frozen
            rc = fz.row_classes()
            rows = rc != N.KS_BD_COMM
            if self.start is not None:
                rows &= self.start[:, s] >= 0
            present = np.unique(_row_layer_ids(fz)[rows])
            per_layer = {self.layer_names[k]: (int(self.layer_busy[k, 0, s]),
                                               int(self.layer_busy[k, 1, s])) for k in present}
        return BreakdownReport(cpu_only=c, gpu_only=g, parallel=par, idle=idle,
                               total=int(self.makespan[s]), per_layer=per_layer)


def _row_layer_ids(fz: FrozenGraph) -> np.ndarray:
    """Layer index per frozen row (names sorted; None -> UNMAPPED_LAYER)."""
    cached = getattr(fz, "_row_layer_cache", None)
    if cached is not None:
        return cached[0]
    from .layers import UNMAPPED_LAYER
    names = [UNMAPPED_LAYER if x is None else x
             for x in (fz.task_layers or [None] * fz.n)]
    uniq = sorted(set(names))
    ix = {k: i for i, k in enumerate(uniq)}
    per_task = np.fromiter((ix[k] for k in names), np.int32, len(names))
    row = np.ascontiguousarray(per_task[fz.order] if fz.n else per_task, np.int32)
    fz._row_layer_cache = (row, uniq)
    return row


def layer_names_of(fz: FrozenGraph) -> list:
    _row_layer_ids(fz)
    return fz._row_layer_cache[1]


@dataclass
class ScenarioTable:
    n_scenarios: int
    dense: object = None                 # np.ndarray / torch.Tensor [rows][ld] int32|int64
    overrides: dict = field(default_factory=dict)   # frozen row -> int64[S]
    scale_ptr: np.ndarray | None = None  # int32[S+1]
    scale: np.ndarray | None = None      # SCALE_STEP_DTYPE[...]
    chain_perm: np.ndarray | None = None # int16[S][sum B]
    chain_present: np.ndarray | None = None  # uint8[S][n_chains]
    vdnn_rank: np.ndarray | None = None  # int32[rows]
    # schedule policy (name, params) the compiled pipelines ask for
    # (TransformPipeline.schedule_policy / policy_params); not part of the C descriptor
    policy: tuple = ("default", None)

    def desc(self, keep: list, rows: int | None = None) -> N.ScenariosDesc:
        """C descriptor of the table.  ``rows`` (the frozen graph's row
        count) is checked against a dense table: the kernels read
        dense[r * ld + s] for every frozen row r and scenario s."""
        sc = N.ScenariosDesc()
        S = self.n_scenarios
        sc.n_scenarios = S
        if self.dense is not None:
            d = self.dense
            dt = str(d.dtype)
            sc.dense_kind = 1 if dt.endswith("int32") else 2
            if not dt.endswith(("int32", "int64")):
                raise ValueError("dense durations must be int32 or int64")
            if d.ndim != 2:
                raise ValueError("dense durations must be a [rows][scenarios] matrix")
            if hasattr(d, "stride") and callable(d.stride):
                ld, inner = int(d.stride(0)), int(d.stride(1))
            else:
                ld, inner = d.strides[0] // d.itemsize, d.strides[1] // d.itemsize
            if inner != 1 or d.shape[1] < S or ld < S:
                raise ValueError("dense durations need unit inner stride and at least "
                                 "n_scenarios columns")
            if rows is not None and d.shape[0] < rows:
                raise ValueError(f"dense durations have {d.shape[0]} rows, the graph {rows}")
            sc.dense = N.ptr(d)
            sc.dense_ld = ld
        if self.overrides:
            rows = np.array(sorted(self.overrides), np.int32)
            vals = np.ascontiguousarray(np.stack([np.asarray(self.overrides[r], np.int64)
                                                  for r in rows.tolist()]))
            if vals.shape[1] != S:
                raise ValueError("override rows must have n_scenarios entries")
            keep += [rows, vals]
            sc.n_overrides = len(rows)
            sc.override_task, sc.override = rows.ctypes.data, vals.ctypes.data
        if self.scale_ptr is not None:
            sp = N.c_i32(self.scale_ptr)
            st = np.ascontiguousarray(self.scale, N.SCALE_STEP_DTYPE)
            if st.size == 0:
                st = np.zeros(1, N.SCALE_STEP_DTYPE)
            keep += [sp, st]
            sc.scale_ptr, sc.scale = sp.ctypes.data, st.ctypes.data
        if self.chain_perm is not None:
            pm = np.ascontiguousarray(self.chain_perm, np.int16)
            keep.append(pm)
            sc.chain_perm, sc.perm_ld = pm.ctypes.data, pm.shape[1]
        if self.chain_present is not None:
            pr = np.ascontiguousarray(self.chain_present, np.uint8)
            keep.append(pr)
            sc.chain_present = pr.ctypes.data
        if self.vdnn_rank is not None:
            vr = N.c_i32(self.vdnn_rank)
            keep.append(vr)
            sc.vdnn_rank = vr.ctypes.data
        return sc


def _host_empty(shape) -> np.ndarray:
    """int64 host array; page-locked when large, so that ks_simulate_host's
    chunked device->host copies run asynchronously (a copy into pageable
    memory blocks the issuing thread and serialises the chunk pipeline)."""
    n = int(np.prod(shape))
    if n * 8 >= (64 << 20):
        import torch

        return torch.empty(shape, dtype=torch.int64, pin_memory=True).numpy()
    return np.empty(shape, np.int64)


def simulate_batch(frozen: FrozenGraph, table: ScenarioTable, policy: str = "default",
                   want_start: bool = True, want_schedule: bool = False,
                   path: int = N.KS_PATH_AUTO, breakdown: bool = False,
                   comm_as_gpu: bool = True, dataload_as_cpu: bool = True,
                   gaps_as_cpu_busy: bool = True, devices=None) -> BatchResult:
    """Host buffers in/out (ks_simulate_host): the reference-facing call.
    breakdown=True also runs compute_breakdown / per_layer_breakdown for
    every scenario on the device (ks_breakdown; max-plus graphs).
    devices=[d0, d1, ...]: scenarios split into contiguous shards simulated
    concurrently on those devices of this process (ks_simulate_host_multi;
    the graph is replicated per device once)."""
    if breakdown:
        return _simulate_batch_with_breakdown(frozen, table, policy, want_start, comm_as_gpu,
                                              dataload_as_cpu, gaps_as_cpu_busy)
    S = table.n_scenarios
    if frozen.n_ordered < frozen.n:
        missing = frozen.unordered_ids()
        raise Deadlock(f"{len(missing)} tasks never became ready (first ids: {missing[:10]})")
    keep: list = []
    sc = table.desc(keep, frozen.n)
    rows, L = frozen.n, frozen.L
    ms = np.zeros(S, np.int64)
    lb = np.zeros((S, max(L, 1)), np.int64)
    start = _host_empty((max(rows, 1), S)) if want_start else None
    sched = np.empty((S, max(rows, 1)), np.int32) if want_schedule else None
    out = N.SimOut()
    out.makespan, out.lane_busy = ms.ctypes.data, lb.ctypes.data
    if start is not None:
        out.start, out.start_ld = start.ctypes.data, S
    if sched is not None:
        out.schedule = sched.ctypes.data
        path = N.KS_PATH_LISTSCHED
    if devices is not None and len(devices) > 1:
        if breakdown:
            raise Unsupported("breakdown=True runs on one device")
        graphs = [frozen.on_device(int(d)) for d in devices]
        arr = (C.c_void_p * len(graphs))(*[gr.handle.value for gr in graphs])
        N.check(N.lib().ks_simulate_host_multi(arr, len(graphs), C.byref(sc), POLICY_IDS[policy],
                                               path, C.byref(out)), "simulate_batch")
    else:
        N.check(N.lib().ks_simulate_host(frozen.handle, C.byref(sc), POLICY_IDS[policy], path,
                                         C.byref(out)), "simulate_batch")
    return BatchResult(frozen=frozen, makespan=ms, lane_busy=lb[:, :L],
                       start=None if start is None else start[:rows], schedule=sched)


def _simulate_batch_with_breakdown(frozen, table, policy, want_start, comm_as_gpu, dataload_as_cpu,
                                   gaps_as_cpu_busy) -> BatchResult:
    import torch

    if frozen.n_ordered < frozen.n:
        missing = frozen.unordered_ids()
        raise Deadlock(f"{len(missing)} tasks never became ready (first ids: {missing[:10]})")
    listsched = not frozen.chained
    if listsched and frozen.chains:
        raise Unsupported("permutable chains need a lane-chained graph for the batched breakdown")
    dev = torch.device("cuda", frozen.device)
    S, rows, L = table.n_scenarios, frozen.n, frozen.L
    dtab = table
    if table.dense is not None and not (hasattr(table.dense, "is_cuda") and table.dense.is_cuda):
        dtab = ScenarioTable(**{**table.__dict__, "dense": torch.as_tensor(
            np.ascontiguousarray(table.dense)).to(dev)})
    ms = torch.empty(S, dtype=torch.int64, device=dev)
    lb = torch.empty((S, max(L, 1)), dtype=torch.int64, device=dev)
    st = torch.empty((max(rows, 1), S), dtype=torch.int64, device=dev)
    parts = torch.empty((S, 4), dtype=torch.int64, device=dev)
    row_layer = _row_layer_ids(frozen)
    names = layer_names_of(frozen)
    lbz = torch.empty((max(len(names), 1), 2, S), dtype=torch.int64, device=dev)
    sched = (torch.empty((S, max(rows, 1)), dtype=torch.int32, device=dev) if listsched
             else None)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream().cuda_stream
        simulate_batch_device(frozen, dtab, makespan=ms, lane_busy=lb, start=st, start_ld=S,
                              stream=stream, policy=policy, schedule=sched)
        breakdown_batch_device(frozen, dtab, start=st, makespan=ms, parts=parts, layer_busy=lbz,
                               stream=stream, comm_as_gpu=comm_as_gpu,
                               dataload_as_cpu=dataload_as_cpu, gaps_as_cpu_busy=gaps_as_cpu_busy,
                               row_layer=row_layer, n_layers=len(names), schedule=sched)
        torch.cuda.current_stream().synchronize()
    return BatchResult(frozen=frozen, makespan=ms.cpu().numpy(), lane_busy=lb.cpu().numpy()[:, :L],
                       start=st.cpu().numpy()[:rows] if want_start else None,
                       parts=parts.cpu().numpy(), layer_busy=lbz.cpu().numpy(), layer_names=names)


def breakdown_batch_device(frozen: FrozenGraph, table: ScenarioTable, *, start, makespan, parts,
                           layer_busy=None, stream: int = 0, comm_as_gpu: bool = True,
                           dataload_as_cpu: bool = True, gaps_as_cpu_busy: bool = True,
                           row_layer=None, n_layers: int = 0, start_ld: int | None = None,
                           schedule=None) -> None:
    """ks_breakdown on device tensors (start / makespan from
    simulate_batch_device on the same table); asynchronous on ``stream``.
    A list-scheduled (not lane-chained) batch passes its dispatch order
    ``schedule`` [S][rows] int32 from the same simulate_batch_device call."""
    keep: list = []
    sc = table.desc(keep, frozen.n)
    bd = N.BreakdownDesc()
    rc = frozen.row_classes()
    keep.append(rc)
    bd.row_class = rc.ctypes.data if rc.size else None
    bd.comm_as_gpu, bd.dataload_as_cpu = int(comm_as_gpu), int(dataload_as_cpu)
    bd.gaps_as_cpu_busy = int(gaps_as_cpu_busy)
    if layer_busy is not None:
        rl = N.c_i32(row_layer if row_layer is not None else _row_layer_ids(frozen))
        keep.append(rl)
        bd.row_layer = rl.ctypes.data if rl.size else None
        bd.n_layers = n_layers or len(layer_names_of(frozen))
    bd.schedule = N.ptr(schedule)
    ld = start_ld if start_ld is not None else int(start.stride(0))
    N.check(N.lib().ks_breakdown(frozen.handle, C.byref(sc), N.ptr(start), ld, N.ptr(makespan),
                                 C.byref(bd), N.ptr(parts), N.ptr(layer_busy), C.c_void_p(stream)),
            "ks_breakdown")


def simulate_batch_device(frozen: FrozenGraph, table: ScenarioTable, *, makespan, lane_busy=None,
                          start=None, start_ld: int | None = None, stream: int = 0,
                          policy: str = "default", path: int = N.KS_PATH_AUTO,
                          schedule=None) -> None:
    """Device tensors in/out (ks_simulate): asynchronous on ``stream``
    (a cudaStream_t as int, e.g. torch.cuda.current_stream().cuda_stream).
    ``schedule`` [S][rows] int32 receives the dispatch order (list scheduler)."""
    keep: list = []
    sc = table.desc(keep, frozen.n)
    out = N.SimOut()
    out.makespan = N.ptr(makespan)
    out.lane_busy = N.ptr(lane_busy)
    if start is not None:
        out.start = N.ptr(start)
        out.start_ld = start_ld if start_ld is not None else int(start.stride(0))
    if schedule is not None:
        out.schedule = N.ptr(schedule)
        path = N.KS_PATH_LISTSCHED
    N.check(N.lib().ks_simulate(frozen.handle, C.byref(sc), POLICY_IDS[policy], path,
                                C.byref(out), C.c_void_p(stream)), "simulate_batch_device")


# ------------------------------------------------------------------ compilers

def compile_scale_sweep(graph: DependencyGraph, scenarios: list[list[tuple[Selector, object]]]):
    """Per-scenario lists of (selector, factor) Shrink steps -> (group_of per
    task in graph.tasks order, scale_ptr, scale steps).

    Tasks are grouped by their membership signature over every distinct
    selector; a step then touches the groups whose signature contains its
    selector (one ks_scale_step per group)."""
    sels: dict[object, int] = {}
    for steps in scenarios:
        for sel, _f in steps:
            key = repr(sel.to_object())
            if key not in sels:
                sels[key] = (len(sels), sel)
    tasks = list(graph.tasks.values())
    sig_of_task = []
    sel_list = sorted(sels.values(), key=lambda x: x[0])
    for t in tasks:
        sig_of_task.append(tuple(i for i, s in sel_list if s.matches(t)))
    group_id: dict[tuple, int] = {(): 0}
    group_of = np.zeros(len(tasks), np.uint32)
    for i, sig in enumerate(sig_of_task):
        if sig not in group_id:
            group_id[sig] = len(group_id)
        group_of[i] = group_id[sig]
    groups_with: dict[int, list[int]] = {i: [] for i, _ in sel_list}
    for sig, gid in group_id.items():
        for i in sig:
            groups_with[i].append(gid)
    ptr = [0]
    steps_out = []
    for steps in scenarios:
        for sel, factor in steps:
            if isinstance(factor, str) and factor == REMOVE:
                for gid in sorted(groups_with[sels[repr(sel.to_object())][0]]):
                    steps_out.append((gid, gid, 0, 0))  # KS_STEP_REMOVE
                continue
            f = Fraction(str(factor)) if not isinstance(factor, Fraction) else factor
            if f <= 0:
                raise BadPipeline(f"scale factor must be positive, got {f}")
            for gid in sorted(groups_with[sels[repr(sel.to_object())][0]]):
                steps_out.append((gid, gid, f.numerator, f.denominator))
        ptr.append(len(steps_out))
    arr = np.zeros(len(steps_out), N.SCALE_STEP_DTYPE)
    for k, (lo, hi, num, den) in enumerate(steps_out):
        arr[k] = (lo, hi, num, den)
    return group_of, np.array(ptr, np.int32), arr


BATCHABLE_OPS = frozenset({"scale", "set_duration", "set_priority", "remove"})


def compile_pipelines(graph: DependencyGraph, pipelines: list, device: int | None = None):
    """Compile what-if pipelines (TransformPipeline, apply_pipeline semantics,
    transform.py:285-399) into one scenario table over a frozen copy of
    ``graph``: scale -> scale steps, set_duration -> per-scenario overrides,
    remove -> KS_STEP_REMOVE steps, set_priority -> nothing (a lane-chained
    graph's schedule does not depend on the policy or priorities; on other
    graphs priorities are structure: see _compile_structural).

    Selections are evaluated on ``graph`` itself: scale / set_duration /
    set_priority do not change the attributes selectors read, and removal is
    final, so each step touches the same tasks as on the progressively
    transformed graph.  Pipelines with inserts (or with set_priority steps
    and one common structure) compile through _compile_structural.
    Returns (FrozenGraph, ScenarioTable); raises Unsupported when no table
    expresses the pipelines."""
    from .errors import UnknownTask
    from .transform import select

    pipes = [p if isinstance(p, TransformPipeline) else TransformPipeline.from_object(p)
             for p in pipelines]
    all_ops = {step.get("op") for p in pipes for step in p.steps}
    if all_ops & INSERT_OPS or ("set_priority" in all_ops and len({structure_key(p) for p in pipes}) == 1):
        return _compile_structural(graph, pipes, device)
    # 1. distinct selections
    sel_ix: dict = {}
    sel_sets: list[frozenset] = []
    plan = []  # per pipeline: [(op, sel index, payload)]

    def sel_of(step) -> int:
        if "task_id" in step:
            tid = step["task_id"]
            if tid not in graph.tasks:
                raise UnknownTask(f"task {tid} does not exist")
            key = ("id", tid)
            ids = frozenset([tid])
        else:
            key = ("sel", repr(step["selector"]))
            if key in sel_ix:
                return sel_ix[key]
            ids = frozenset(select(graph, Selector.from_object(step["selector"])))
        if key not in sel_ix:
            sel_ix[key] = len(sel_sets)
            sel_sets.append(ids)
        return sel_ix[key]

    for pipe in pipes:
        ops = []
        for step in pipe.steps:
            op = step.get("op")
            if op not in BATCHABLE_OPS:
                raise Unsupported(f"pipeline op {op!r} has no scenario-table form "
                                  "(run it through apply_pipeline + simulate)")
            if op == "set_priority":
                continue
            if op == "scale":
                f = Fraction(str(step["factor"]))
                if f <= 0:
                    raise BadPipeline(f"scale factor must be positive, got {f}")
                ops.append(("scale", sel_of(step), f))
            elif op == "set_duration":
                ops.append(("set", sel_of(step), int(step["duration_ns"])))
            else:
                ops.append(("remove", sel_of(step), None))
        plan.append(ops)
    # 2. groups = membership signatures over the selections
    member: dict[int, list[int]] = {}
    for k, ids in enumerate(sel_sets):
        for tid in ids:
            member.setdefault(tid, []).append(k)
    tasks = list(graph.tasks)
    group_id: dict[tuple, int] = {(): 0}
    group_of = np.zeros(len(tasks), np.uint32)
    for i, tid in enumerate(tasks):
        sig = tuple(member.get(tid, ()))
        gid = group_id.setdefault(sig, len(group_id))
        group_of[i] = gid
    groups_of_sel: dict[int, list[int]] = {k: [] for k in range(len(sel_sets))}
    for sig, gid in group_id.items():
        for k in sig:
            groups_of_sel[k].append(gid)
    fz = FrozenGraph.from_graph(graph, group_of=group_of, device=device)
    if not fz.chained and "set_priority" in all_ops:
        raise Unsupported("set_priority steps of different structure on a list-scheduled graph")
    if not fz.chained and any(op == "remove" for pl in plan for op, _k, _p in pl):
        raise Unsupported("remove steps on a graph that is not lane-chained are structural "
                          "(run them through apply_pipeline + simulate)")
    # 3. per-scenario programs
    S = len(pipes)
    ptr = [0]
    steps_out: list = []
    ovr: dict[int, np.ndarray] = {}
    index = {int(t): i for i, t in enumerate(fz.ids)}
    base_rows = fz.duration
    for s, ops in enumerate(plan):
        prog: list = []          # [gid, num, den] in order
        removed: set[int] = set()
        for op, k, payload in ops:
            gids = groups_of_sel[k]
            if op == "scale":
                prog += [[g, payload.numerator, payload.denominator] for g in gids if g not in removed]
            elif op == "remove":
                removed.update(gids)
            else:  # set_duration of one task: earlier scales of its group are void
                (tid,) = sel_sets[k]
                g = gids[0]
                if g in removed:
                    raise UnknownTask(f"task {tid} does not exist")
                prog = [e for e in prog if e[0] != g]
                row = int(fz.row_of[index[tid]])
                if row not in ovr:
                    ovr[row] = np.full(S, base_rows[index[tid]], np.int64)
                ovr[row][s] = payload
        steps_out += [(g, g, num, den) for g, num, den in prog if g not in removed]
        steps_out += [(g, g, 0, 0) for g in sorted(removed)]
        ptr.append(len(steps_out))
    arr = np.zeros(len(steps_out), N.SCALE_STEP_DTYPE)
    for i, st in enumerate(steps_out):
        arr[i] = st
    table = ScenarioTable(n_scenarios=S, overrides=ovr,
                          scale_ptr=np.array(ptr, np.int32) if steps_out else None,
                          scale=arr if steps_out else None)
    _set_policy(table, graph, fz, pipes)
    return fz, table


def _set_policy(table: ScenarioTable, graph: DependencyGraph, fz: FrozenGraph, pipes: list) -> None:
    """The pipelines' schedule policy (one per table) and its device
    parameters (vdnn_prefetch: per-row conv rank, scenarios.py:593-630)."""
    names = {(p.schedule_policy, repr(p.policy_params)) for p in pipes}
    if len(names) > 1:
        raise Unsupported("pipelines of one table must share a schedule policy")
    p0 = pipes[0]
    table.policy = (p0.schedule_policy, dict(p0.policy_params or {}))
    if p0.schedule_policy == "vdnn_prefetch":
        from .sim import make_policy
        pol = make_policy(p0.schedule_policy, **(p0.policy_params or {}))
        vr = pol.device_params(graph, fz).get("vdnn_rank")
        table.vdnn_rank = np.ascontiguousarray(np.asarray(vr, np.int32)[fz.order])


INSERT_OPS = frozenset({"insert", "insert_gpu_with_launch"})


def structure_key(pipeline) -> str:
    """A pipeline with every duration / factor blanked (plus its schedule
    policy): pipelines with equal keys transform a graph into the same task
    set, edges, lane orders and priorities, and differ only in durations.
    A zero launch cost changes the structure (the launch is elided,
    transform.py:347-353), so only its zero-ness stays in the key."""
    import json

    p = pipeline if isinstance(pipeline, TransformPipeline) else TransformPipeline.from_object(pipeline)
    steps = []
    for step in p.steps:
        st = dict(step)
        op = st.get("op")
        if op == "scale":
            st["factor"] = None
        elif op == "set_duration":
            st["duration_ns"] = None
        elif op == "insert":
            st["task"] = {**st["task"], "duration_ns": None}
        elif op == "insert_gpu_with_launch":
            st["kernel"] = {**st["kernel"], "duration_ns": None}
            if st.get("launch_cost_ns") is not None:
                st["launch_cost_ns"] = int(st["launch_cost_ns"]) > 0
        steps.append(st)
    return json.dumps([steps, p.schedule_policy, p.policy_params], sort_keys=True, default=str)


def _compile_structural(graph: DependencyGraph, pipes: list, device):
    """Pipelines with inserts (distributed, p3, blueconnect, vdnn, gist, dgc,
    scenarios.py:191-470) that share one structure_key: the first pipeline is
    applied structurally once (apply_pipeline, transform.py:370-396, with its
    errors), and every pipeline's durations become table columns over that
    transformed graph:

    * an inserted task's (or launch's) duration and a set_duration value ->
      a per-scenario override row when it varies across the pipelines;
    * scale steps -> per-scenario half-up scale programs on groups of tasks
      with the same sequence of selecting steps after their last base-setting
      step (a selector is evaluated on the graph as it is at its step, so
      tasks inserted later are not selected, exactly as in apply_step).

    Unchained results (unsequenced inserts) run on the list scheduler with the
    pipelines' policy; lane-chained ones on the max-plus kernels."""
    from .transform import apply_pipeline, apply_step, insert_gpu_with_launch_step, select
    from . import transform as TR

    keys = {structure_key(p) for p in pipes}
    if len(keys) != 1:
        raise Unsupported("pipelines with inserts differ in structure (one table per "
                          "structure_key; Analysis.whatif_batch groups them)")
    p0 = pipes[0]
    for p in pipes:  # every scale factor must be valid (scale_durations raises otherwise)
        for step in p.steps:
            if step.get("op") == "scale" and Fraction(str(step["factor"])) <= 0:
                raise BadPipeline(f"scale factor must be positive, got {step['factor']}")
    final = apply_pipeline(graph, p0)  # the reference's own errors, in step order
    # replay pipeline 0 recording what each step touches
    h = graph.copy()
    events: dict[int, list] = {}   # task id -> [(step index, "base" | "scale")]
    base_src: dict[int, tuple] = {}  # task id -> (step index, field) of its per-scenario base
    numeric_seen = False
    TR._DEFER["on"] = True
    try:
        for i, step in enumerate(p0.steps):
            op = step.get("op")
            if op == "scale":
                for tid in select(h, Selector.from_object(step["selector"])):
                    events.setdefault(tid, []).append((i, "scale"))
                numeric_seen = True
            elif op == "set_duration":
                events.setdefault(step["task_id"], []).append((i, "base"))
                base_src[step["task_id"]] = (i, "set")
                numeric_seen = True
            elif op == "insert":
                before = set(h.tasks)
                apply_step(h, step)
                (tid,) = set(h.tasks) - before
                events[tid] = [(i, "base")]
                base_src[tid] = (i, "insert")
                continue
            elif op == "insert_gpu_with_launch":
                if step.get("launch_cost_ns") is None and numeric_seen:
                    raise Unsupported("insert_gpu_with_launch without launch_cost_ns after a "
                                      "duration-changing step (its default cost varies)")
                launch, kernel = insert_gpu_with_launch_step(h, step)
                events[kernel] = [(i, "base")]
                base_src[kernel] = (i, "kernel")
                if launch in h.tasks and h.tasks[launch].kind is TaskKind.CPU_API and \
                        launch != kernel:
                    events[launch] = [(i, "base")]
                    base_src[launch] = (i, "launch")
                continue
            elif op == "remove":
                before = set(h.tasks)
                apply_step(h, step)
                for tid in before - set(h.tasks):
                    events.pop(tid, None)
                    base_src.pop(tid, None)
                continue
            apply_step(h, step)
    finally:
        TR._DEFER["on"] = False
    assert set(h.tasks) == set(final.tasks)
    g = final
    S = len(pipes)

    def value(p, i, field):
        step = p.steps[i]
        if field == "set":
            return int(step["duration_ns"])
        if field == "insert":
            return int(step["task"]["duration_ns"])
        if field == "kernel":
            return int(step["kernel"]["duration_ns"])
        cost = step.get("launch_cost_ns")
        return int(cost) if cost is not None else int(g.tasks[launch_of[i]].duration)

    launch_of = {i: tid for tid, (i, f) in base_src.items() if f == "launch"}
    # per task: the scale steps after its last base-setting step
    sig_of: dict[int, tuple] = {}
    for tid, ev in events.items():
        last_base = max((i for i, k in ev if k == "base"), default=-1)
        sig_of[tid] = tuple(i for i, k in ev if k == "scale" and i > last_base)
    tasks = list(g.tasks)
    group_id: dict[tuple, int] = {(): 0}
    group_of = np.zeros(len(tasks), np.uint32)
    for j, tid in enumerate(tasks):
        group_of[j] = group_id.setdefault(sig_of.get(tid, ()), len(group_id))
    # base durations: the original duration, or pipeline 0's base-setting value
    base_vals: dict[int, np.ndarray] = {}
    for tid in tasks:
        ev = events.get(tid, [])
        last_base = max((i for i, k in ev if k == "base"), default=-1)
        if last_base >= 0:
            field = "set" if p0.steps[last_base]["op"] == "set_duration" else base_src[tid][1]
            vals = np.array([value(p, last_base, field) for p in pipes], np.int64)
            g.tasks[tid].duration = int(vals[0])
            if np.any(vals != vals[0]):
                base_vals[tid] = vals
        else:
            g.tasks[tid].duration = int(graph.tasks[tid].duration)
    fz = FrozenGraph.from_graph(g, group_of=group_of, device=device)
    index = {int(t): k for k, t in enumerate(fz.ids)}
    ovr = {int(fz.row_of[index[tid]]): v for tid, v in base_vals.items()}
    groups_with: dict[int, list[int]] = {}
    for sig, gid in group_id.items():
        for i in sig:
            groups_with.setdefault(i, []).append(gid)
    ptr, steps_out = [0], []
    scale_steps = [i for i, st in enumerate(p0.steps) if st.get("op") == "scale"]
    for p in pipes:
        for i in scale_steps:
            f = Fraction(str(p.steps[i]["factor"]))
            steps_out += [(gid, gid, f.numerator, f.denominator) for gid in groups_with.get(i, ())]
        ptr.append(len(steps_out))
    arr = np.zeros(len(steps_out), N.SCALE_STEP_DTYPE)
    for k, st in enumerate(steps_out):
        arr[k] = st
    table = ScenarioTable(n_scenarios=S, overrides=ovr,
                          scale_ptr=np.array(ptr, np.int32) if steps_out else None,
                          scale=arr if steps_out else None)
    _set_policy(table, g, fz, pipes)
    fz.source_graph = g
    return fz, table


@dataclass
class DistributedSweep:
    frozen: FrozenGraph
    table: ScenarioTable
    member_ids: list[int]
    configs: list[dict]
    perms: np.ndarray


def distributed_sweep(graph: DependencyGraph, buckets: GradientBucketMap, configs: list[dict],
                      perms: np.ndarray | None = None, device: int | None = None) -> DistributedSweep:
    """Data-parallel what-if table: one allReduce per non-empty bucket on
    comm:collective (whatif_distributed, scenarios.py:194-241) with a
    per-scenario network config (bandwidth x workers ...) and bucket order.

    Scenario s equals the reference pipeline whose sequenced inserts are
    applied in order perms[s] (the lane order of sequenced inserts is their
    insertion order); workers == 1 drops the inserts (empty pipeline)."""
    wu = earliest_weight_update_task(graph)
    if wu is None:
        raise NoWeightUpdate("no weight-update tasks in the graph")
    g = graph.copy()
    head_order = g.lane_order.get(COLLECTIVE_LANE, [])
    head = head_order[-1] if head_order else None
    nid = g.next_id()
    members, sizes = [], []
    for b in buckets.buckets():
        layers = buckets.layers_of_bucket(b)
        if not layers:
            continue
        size = buckets.bucket_size_bytes[b]
        tid = nid + len(members)
        g.tasks[tid] = Task(id=tid, kind=TaskKind.COMM, name=f"allreduce_bucket_{b}",
                            lane=COLLECTIVE_LANE, duration=0, size_bytes=size)
        for layer in layers:
            src = last_backward_gpu_task(graph, layer)
            if src is None:
                raise MissingLayer(f"bucket {b}: layer {layer!r} has no backward GPU tasks")
            g.edges.add((src.id, tid, EdgeKind.INJECTED))
        g.edges.add((tid, wu.id, EdgeKind.INJECTED))
        members.append(tid)
        sizes.append(size)
    B = len(members)
    S = len(configs)
    fz = FrozenGraph.from_graph(g, chains=[ChainSpec(members=members, head=head)] if B else None,
                                device=device)
    if perms is None:
        perms = np.tile(np.arange(B, dtype=np.int16), (S, 1))
    perms = np.asarray(perms, np.int16).reshape(S, B)
    present = np.ones((S, 1), np.uint8)
    ovr = {}
    if B:
        dur = np.zeros((B, S), np.int64)
        for s, cfg_obj in enumerate(configs):
            cfg = NetworkConfig.from_object(cfg_obj)
            if cfg.n_workers == 1:
                present[s, 0] = 0
                continue
            for k, size in enumerate(sizes):
                dur[k, s] = allreduce_duration(size, cfg)
        idx = {int(t): i for i, t in enumerate(fz.ids)}
        for k, tid in enumerate(members):
            ovr[int(fz.row_of[idx[tid]])] = dur[k]
    table = ScenarioTable(n_scenarios=S, overrides=ovr, chain_perm=perms if B else None,
                          chain_present=present if B else None)
    return DistributedSweep(frozen=fz, table=table, member_ids=members, configs=configs,
                            perms=perms)
