"""The device's half-up Shrink arithmetic (round_half_up, transform.py:174-183:
d <- floor((2*d*num + den) / (2*den)), a 128-bit intermediate on the device)
on every golden units.scale vector the reference produced, through each
kernel path that applies scale programs.

Vectors go four at a time into a graph of four independent tasks, one per
CPU lane, each task in its own group; one scenario scales group j by vector
j's factor, so lane j's busy time is exactly that vector's scaled duration.
Vectors whose exact result leaves int64 are outside the simulated domain (the
reference uses unbounded ints) and skipped, as in test_oracle_pinned."""

import numpy as np
import pytest

from paper_2006_03318_b200 import _native as N
from paper_2006_03318_b200.batch import ScenarioTable, simulate_batch
from paper_2006_03318_b200.frozen import FrozenGraph
from paper_2006_03318_b200.graph import DependencyGraph, Task
from paper_2006_03318_b200.trace import LaneId, TaskKind

pytestmark = pytest.mark.gpu

PATHS = {
    "derived-lanes": ({"DDSIM_FORCE_DERIVED": "1"}, N.KS_PATH_AUTO),
    "expand+lanes": ({"DDSIM_NO_DERIVED": "1"}, N.KS_PATH_AUTO),  # int32 matrix where it fits
    "expand64+lanes": ({"DDSIM_NO_DERIVED": "1", "DDSIM_EXPAND64": "1"}, N.KS_PATH_AUTO),
    "lanes-general": ({"DDSIM_NO_EXPAND": "1"}, N.KS_PATH_AUTO),
    "general": ({"DDSIM_NO_EXPAND": "1", "DDSIM_NO_LANES": "1"}, N.KS_PATH_AUTO),
    "listsched": ({}, N.KS_PATH_LISTSCHED),
}


@pytest.mark.parametrize("mode", list(PATHS))
def test_device_scale_on_every_golden_vector(golden, mode, monkeypatch):
    env, path = PATHS[mode]
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    vec = [(d, num, den, want) for d, num, den, want in golden["units"]["scale"]
           if want < 2**63 and d < 2**63]
    assert len(vec) > 300
    got, want = [], []
    for c in range(0, len(vec), 4):
        chunk = vec[c:c + 4]
        g = DependencyGraph()
        for j, (d, _n, _dn, _w) in enumerate(chunk):
            lane = LaneId.parse(f"cpu:{j}")
            g.tasks[j] = Task(id=j, kind=TaskKind.CPU_API, name=f"t{j}", lane=lane, duration=int(d))
            g.lane_order[lane] = [j]
        fz = FrozenGraph.from_graph(g, group_of=np.arange(1, len(chunk) + 1, dtype=np.uint32))
        steps = np.zeros(len(chunk), N.SCALE_STEP_DTYPE)
        for j, (_d, num, den, _w) in enumerate(chunk):
            steps[j] = (j + 1, j + 1, num, den)
        res = simulate_batch(fz, ScenarioTable(n_scenarios=1, scale_ptr=np.array([0, len(chunk)],
                                                                                 np.int32),
                                               scale=steps), path=path)
        for j, (_d, _n, _dn, w) in enumerate(chunk):
            got.append(int(res.lane_busy[0, fz.lanes.index(LaneId.parse(f"cpu:{j}"))]))
            want.append(int(w))
        assert int(res.makespan[0]) == max(int(w) for *_x, w in chunk)
    assert got == want
