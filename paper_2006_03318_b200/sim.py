"""simulate(): the device-resident schedule simulator (drop-in for kernsim.sim).

Reference: pkg/src/kernsim/sim.py.  ``simulate(graph, policy)`` freezes the
graph (frozen.py) and runs one of two sm_100a kernels through the C-ABI:

* maxplus_sim  -- every task lane-chained: start(v) = max(ready, max over
  preds of start+dur+gap), exact for all three built-in policies because
  lane progress never binds (sim.py:113-130);
* listsched_sim -- otherwise: the exact Alg. 1 event loop with the policy's
  tie rules (sim.py:55-86, scenarios.py:618-630).

The dispatch order (``schedule_trace``) of a chained graph is produced lazily
by the list-scheduling kernel the first time it is read.

Schedule policies are identified, not executed: a policy object selects the
device rule.  A user subclass that overrides ``choose`` cannot run on the
device and is rejected with ``UnsupportedPolicy`` (there is no CPU fallback).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import Deadlock, UnsupportedPolicy, ZeroBaseline
from .graph import DependencyGraph, Task
from .trace import LaneId


@dataclass
class SimulationState:
    """Alg. 1 state as exposed to ``SchedulePolicy.choose`` (sim.py:19-28)."""

    lane_progress: dict[LaneId, int]
    ready_time: dict[int, int]
    remaining_parents: dict[int, int]
    tasks: dict[int, Task]

    def effective_start(self, task_id: int) -> int:
        t = self.tasks[task_id]
        return max(self.lane_progress.get(t.lane, 0), self.ready_time[task_id])


class SimulationResult:
    """start_of / makespan / lane_busy / schedule_trace of one run."""

    __slots__ = ("start_of", "makespan", "lane_busy", "_trace", "_trace_fn")

    def __init__(self, start_of, makespan, lane_busy, schedule_trace=None, trace_fn=None):
        self.start_of: dict[int, int] = start_of
        self.makespan: int = makespan
        self.lane_busy: dict[LaneId, int] = lane_busy
        self._trace = None if schedule_trace is None else tuple(schedule_trace)
        self._trace_fn = trace_fn

    @property
    def schedule_trace(self) -> tuple[tuple[int, int], ...]:
        if self._trace is None:
            self._trace = tuple(self._trace_fn()) if self._trace_fn else ()
            self._trace_fn = None
        return self._trace

    def __eq__(self, other):
        if not isinstance(other, SimulationResult):
            return NotImplemented
        return (self.start_of == other.start_of and self.makespan == other.makespan
                and self.lane_busy == other.lane_busy
                and self.schedule_trace == other.schedule_trace)

    def __repr__(self):
        return (f"SimulationResult(makespan={self.makespan}, tasks={len(self.start_of)}, "
                f"lanes={len(self.lane_busy)})")

    def to_object(self) -> dict:
        return {
            "makespan_ns": self.makespan,
            "starts_ns": {str(t): s for t, s in sorted(self.start_of.items())},
            "lane_busy_ns": {str(ln): b for ln, b in
                             sorted(self.lane_busy.items(), key=lambda kv: str(kv[0]))},
        }


class SchedulePolicy:
    """Frontier choice rule; the device kernels implement the built-in ones.

    ``choose`` is the reference's rule (sim.py:55-63) kept for introspection
    of a single decision; simulate() never calls it."""

    name = "default"
    device_policy = N.KS_POLICY_DEFAULT

    def begin(self, graph: DependencyGraph) -> None:
        """Reset per-run state (no-op for the built-in rules)."""

    def choose(self, state: SimulationState, frontier: set[int]) -> int:
        return min(frontier, key=lambda t: (state.effective_start(t), t))

    def device_params(self, graph: DependencyGraph, frozen) -> dict:
        return {}


class DefaultSchedule(SchedulePolicy):
    """Earliest effective start, ties to the smallest task id."""

    name = "default"


class PrioritySchedule(SchedulePolicy):
    """Earliest effective start; among tied comm tasks the strictly higher
    priority wins, other ties go to the smallest id (sim.py:72-86)."""

    name = "priority"
    device_policy = N.KS_POLICY_PRIORITY

    def choose(self, state: SimulationState, frontier: set[int]) -> int:
        eff = {t: state.effective_start(t) for t in frontier}
        low = min(eff.values())
        tied = sorted(t for t, e in eff.items() if e == low)
        if not state.tasks[tied[0]].is_comm:
            return tied[0]
        comm = [t for t in tied if state.tasks[t].is_comm]
        return max(comm, key=lambda t: (state.tasks[t].priority, -t))


_BUILTIN_CHOOSERS = {SchedulePolicy.choose, PrioritySchedule.choose}


def _device_policy(policy: SchedulePolicy) -> int:
    choose = type(policy).choose
    if choose not in _BUILTIN_CHOOSERS and getattr(choose, "__device_rule__", None) is None:
        raise UnsupportedPolicy(
            f"policy {type(policy).__name__!r} overrides choose(); only the built-in rules "
            "(default, priority, vdnn_prefetch) run on the device")
    return int(policy.device_policy)


def _run(fz, policy_id: int, scen: N.ScenariosDesc, want_schedule: bool, path: int):
    n, L = fz.n, fz.L
    start = np.empty(max(n, 1), np.int64)
    ms = np.zeros(1, np.int64)
    lb = np.zeros(max(L, 1), np.int64)
    disp = np.zeros(1, np.int32)
    sched = np.empty(max(n, 1), np.int32) if want_schedule else None
    out = N.SimOut()
    out.start, out.start_ld = start.ctypes.data, 1
    out.makespan, out.lane_busy = ms.ctypes.data, lb.ctypes.data
    out.dispatched = disp.ctypes.data
    out.schedule = N.ptr(sched)
    rc = N.lib().ks_simulate_host(fz.handle, scen, policy_id, path, out)
    return rc, start, int(ms[0]), lb, sched


def _deadlock(fz) -> Deadlock:
    missing = fz.unordered_ids()
    return Deadlock(f"{len(missing)} tasks never became ready (first ids: {missing[:10]})")


def _scenarios_for(fz, policy: SchedulePolicy, graph: DependencyGraph):
    sc = N.ScenariosDesc()
    sc.n_scenarios = 1
    keep = []
    params = policy.device_params(graph, fz)
    vr = params.get("vdnn_rank")
    if vr is not None:
        vr = N.c_i32(np.asarray(vr)[fz.order])  # per dense input -> per frozen row
        keep.append(vr)
        sc.vdnn_rank = vr.ctypes.data
    return sc, keep


def simulate(graph: DependencyGraph, policy: SchedulePolicy | None = None) -> SimulationResult:
    """Assign a start time to every task; ``graph`` is not mutated."""
    from .frozen import FrozenGraph

    if policy is None:
        policy = DefaultSchedule()
    pid = _device_policy(policy)
    policy.begin(graph)
    if not graph.tasks:
        return SimulationResult({}, 0, {}, ())
    fz = FrozenGraph.from_graph(graph)
    if fz.n_ordered < fz.n:
        fz.close()
        raise _deadlock(fz)
    sc, keep = _scenarios_for(fz, policy, graph)
    chained = fz.chained
    rc, start, makespan, lb, sched = _run(fz, pid, sc, want_schedule=not chained,
                                          path=N.KS_PATH_AUTO)
    if rc == N.KS_ERR_DEADLOCK:
        raise _deadlock(fz)
    N.check(rc, "simulate")
    row_ids = fz.row_ids
    start_of = dict(zip(row_ids.tolist(), start[:fz.n].tolist()))
    used = np.zeros(fz.L, bool)
    used[fz.lane] = True
    lane_busy = {fz.lanes[j]: int(lb[j]) for j in range(fz.L) if used[j]}

    def trace_from(sched_rows):
        rows = sched_rows[:fz.n]
        return list(zip(row_ids[rows].tolist(), start[rows].tolist()))

    if chained:
        def lazy():
            rc2, _s, _m, _l, sched2 = _run(fz, pid, sc, True, N.KS_PATH_LISTSCHED)
            N.check(rc2, "schedule_trace")
            out = trace_from(sched2)
            fz.close()
            return out

        _keep = keep  # noqa: F841 - vdnn ranks must outlive the lazy call
        return SimulationResult(start_of, makespan, lane_busy, trace_fn=lazy)
    out = SimulationResult(start_of, makespan, lane_busy, schedule_trace=trace_from(sched))
    fz.close()
    return out


def speedup(baseline: SimulationResult, variant: SimulationResult) -> float:
    """Signed fractional improvement of ``variant`` over ``baseline``."""
    if baseline.makespan == 0:
        raise ZeroBaseline("baseline makespan is zero")
    return (baseline.makespan - variant.makespan) / baseline.makespan


POLICIES: dict[str, type[SchedulePolicy]] = {"default": DefaultSchedule,
                                             "priority": PrioritySchedule}


def make_policy(name: str, **params) -> SchedulePolicy:
    from .scenarios import EXTRA_POLICIES

    if name in POLICIES:
        return POLICIES[name]()
    if name in EXTRA_POLICIES:
        return EXTRA_POLICIES[name](**params)
    raise ValueError(f"unknown schedule policy {name!r}")
