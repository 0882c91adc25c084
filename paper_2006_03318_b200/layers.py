"""Synchronisation-free task -> (layer, phase) mapping (kernsim.layers).

Reference: pkg/src/kernsim/layers.py:30-93.  A CPU-kind task belongs to the
innermost marker on its lane that contains its trace interval (ties broken
by (length, layer, phase) with an ambiguity check of the best two); a GPU-kind
task inherits its launcher's tag.  The containment search runs on the device
(ks_map_layers: per-lane sorted markers + max-end sparse table, so each task
costs O(depth * log M) instead of the reference's O(M) scan).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .graph import DependencyGraph
from .trace import LayerMarker, Phase

GLOBAL_LAYER = "_global"
UNMAPPED_LAYER = "_unmapped"


@dataclass
class LayerAssignment:
    mapped: dict[int, tuple[str, Phase]] = field(default_factory=dict)
    unmapped: set[int] = field(default_factory=set)

    def layer_of(self, task_id: int) -> tuple[str, Phase] | None:
        return self.mapped.get(task_id)


def map_tasks_to_layers(graph: DependencyGraph, markers: list[LayerMarker]) -> LayerAssignment:
    """Assign (layer, phase) tags on the device; also written onto the tasks
    (the reference mutates Task.layer, layers.py:79-80)."""
    from .ingest import map_layers_device

    mapped = map_layers_device(graph, list(markers))
    out = LayerAssignment(mapped=mapped, unmapped={t for t in graph.tasks if t not in mapped})
    for tid, tag in mapped.items():
        graph.tasks[tid].layer = tag
    return out


def select_by_layer(graph: DependencyGraph, layer: str, phase: Phase | None = None) -> set[int]:
    return {t.id for t in graph.tasks.values()
            if t.layer is not None and t.layer[0] == layer
            and (phase is None or t.layer[1] == phase)}
