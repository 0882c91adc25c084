"""Kernel-granularity dependency graph: object model, construction, checks.

Drop-in for kernsim.graph (pkg/src/kernsim/graph.py).  The object model
(Task / DependencyGraph with tasks, edges, lane_order) is kept verbatim in
shape because callers mutate it directly.  The work is on the device:

* ``build_graph`` -> ks_ingest (lane sort, correlation join, sync linking,
  gaps; graph.py:198-312), see ingest.py;
* ``verify_acyclic`` -> ks_toposort (Kahn, smallest-id first;
  graph.py:129-148).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from enum import Enum

from .errors import CycleDetected
from .trace import LaneId, Phase, TaskKind, TraceDocument

DTOH_NAME_PREFIX = "memcpy_dtoh"


class EdgeKind(str, Enum):
    LANE_SEQ_CPU = "LaneSeqCpu"
    LANE_SEQ_GPU = "LaneSeqGpu"
    LAUNCH_CORRELATION = "LaunchCorrelation"
    SYNC_BLOCK = "SyncBlock"
    COMM_ORDER = "CommOrder"
    INJECTED = "Injected"


# device edge-kind codes (include/ddsim.h KS_EDGE_*)
EDGE_KIND_OF_CODE = [EdgeKind.LANE_SEQ_CPU, EdgeKind.LANE_SEQ_GPU, EdgeKind.LAUNCH_CORRELATION,
                     EdgeKind.SYNC_BLOCK, EdgeKind.COMM_ORDER, EdgeKind.INJECTED]


@dataclass
class Task:
    """A node.  ``trace_start`` is construction metadata only; simulation
    starts every task at ``ready_time`` (0 unless set)."""

    id: int
    kind: TaskKind
    name: str
    lane: LaneId
    duration: int
    gap: int = 0
    ready_time: int = 0
    correlation: int | None = None
    layer: tuple[str, Phase] | None = None
    priority: int = 0
    size_bytes: int | None = None
    trace_start: int | None = None

    @property
    def is_comm(self) -> bool:
        return self.kind is TaskKind.COMM


Edge = tuple[int, int, EdgeKind]


def lane_seq_kind(lane: LaneId) -> EdgeKind:
    if lane.is_cpu:
        return EdgeKind.LANE_SEQ_CPU
    return EdgeKind.LANE_SEQ_GPU if lane.is_gpu else EdgeKind.COMM_ORDER


@dataclass
class DependencyGraph:
    tasks: dict[int, Task] = field(default_factory=dict)
    edges: set[Edge] = field(default_factory=set)
    # Tasks whose on-lane order is fixed; tasks missing from their lane's list
    # are placed by the scheduler alone (graph.py:79-81).
    lane_order: dict[LaneId, list[int]] = field(default_factory=dict)

    def copy(self) -> "DependencyGraph":
        return DependencyGraph(tasks={k: replace(t) for k, t in self.tasks.items()},
                               edges=set(self.edges),
                               lane_order={ln: list(v) for ln, v in self.lane_order.items()})

    def next_id(self) -> int:
        return max(self.tasks, default=-1) + 1

    def parents_of(self) -> dict[int, list[int]]:
        out: dict[int, list[int]] = {t: [] for t in self.tasks}
        for u, v, _ in self.edges:
            out[v].append(u)
        return out

    def children_of(self) -> dict[int, list[int]]:
        out: dict[int, list[int]] = {t: [] for t in self.tasks}
        for u, v, _ in self.edges:
            out[u].append(v)
        return out

    def to_object(self) -> dict:
        rows = []
        for t in sorted(self.tasks.values(), key=lambda t: t.id):
            rows.append({
                "id": t.id, "kind": t.kind.value, "name": t.name, "lane": str(t.lane),
                "duration_ns": t.duration, "gap_ns": t.gap, "correlation": t.correlation,
                "layer": t.layer[0] if t.layer else None,
                "phase": t.layer[1].value if t.layer else None,
                "priority": t.priority, "size_bytes": t.size_bytes,
            })
        return {
            "tasks": rows,
            "edges": sorted([u, v, k.value] for u, v, k in self.edges),
            "lane_order": {str(ln): list(ids) for ln, ids in
                           sorted(self.lane_order.items(), key=lambda kv: str(kv[0]))},
        }


def _cycle_among(graph: DependencyGraph, stuck: set[int]) -> list[int]:
    """A concrete cycle inside the tasks Kahn could not order (error report
    only; graph.py:151-186 semantics: a closed walk, first node repeated)."""
    succ: dict[int, list[int]] = {t: [] for t in stuck}
    for u, v, _ in graph.edges:
        if u in stuck and v in stuck:
            succ[u].append(v)
    for lst in succ.values():
        lst.sort()
    state: dict[int, int] = {}
    for root in sorted(stuck):
        if root in state:
            continue
        path = [root]
        state[root] = 1
        iters = [iter(succ[root])]
        while iters:
            nxt = next(iters[-1], None)
            if nxt is None:
                state[path.pop()] = 2
                iters.pop()
                continue
            st = state.get(nxt)
            if st == 1:
                return path[path.index(nxt):] + [nxt]
            if st is None:
                state[nxt] = 1
                path.append(nxt)
                iters.append(iter(succ[nxt]))
    return sorted(stuck)


def is_acyclic(graph: DependencyGraph) -> bool:
    """Acyclicity without the ordered list: the frozen graph's topological
    pass (ks_graph_create) orders every task iff there is no cycle, so the
    lexicographically-first order (verify_acyclic, the device's sequential
    Kahn walk) is only computed when a caller wants the list or the cycle."""
    if not graph.tasks:
        return True
    from .frozen import FrozenGraph

    fz = FrozenGraph.from_graph(graph)
    try:
        return fz.n_ordered == fz.n
    finally:
        fz.close()


def verify_acyclic(graph: DependencyGraph) -> list[int]:
    """Topological order with smallest-id tie-break; CycleDetected otherwise.
    The order is computed on the device (ks_toposort)."""
    if not graph.tasks:
        return []
    from .frozen import FrozenGraph

    fz = FrozenGraph.from_graph(graph)
    try:
        order, ok = fz.toposort()
    finally:
        fz.close()
    if not ok:
        done = set(order)
        cycle = _cycle_among(graph, {t for t in graph.tasks if t not in done})
        raise CycleDetected(f"dependency cycle: {cycle}", cycle)
    return order


def build_graph(trace: TraceDocument, strict: bool = False) -> DependencyGraph:
    """Build the dependency graph of a validated trace (graph.py:198-245):
    lane sequencing (rules 1, 2, 5), launch correlation (rule 3, last CPU
    launch of a correlation wins), synchronisation (rule 4) and CPU gaps --
    all derived on the device by the ingest kernels."""
    from .ingest import build_graph_device

    return build_graph_device(trace, strict=strict)


def link_syncs(trace: TraceDocument, graph: DependencyGraph) -> DependencyGraph:
    """Rule 4 only (graph.py:248-298); adds SyncBlock edges to ``graph``."""
    from .ingest import ingest_columns

    res = ingest_columns(trace, strict=False)
    for u, v, k in res.edge_triples():
        if k is EdgeKind.SYNC_BLOCK:
            graph.edges.add((u, v, k))
    return graph


def compute_gaps(trace: TraceDocument, graph: DependencyGraph) -> DependencyGraph:
    """CPU-lane gaps (graph.py:301-312) from the device ingest result."""
    from .ingest import ingest_columns

    res = ingest_columns(trace, strict=False)
    for tid, gap in res.gaps_by_id().items():
        if tid in graph.tasks:
            graph.tasks[tid].gap = gap
    return graph
