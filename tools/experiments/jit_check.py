import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2006_03318_b200 import _native as N
from paper_2006_03318_b200.frozen import FrozenGraph
from paper_2006_03318_b200.batch import ScenarioTable, simulate_batch
from paper_2006_03318_b200.workloads import resnet_like_graph
g = resnet_like_graph(400, 1)
fz = FrozenGraph.from_graph(g)
dense = np.ascontiguousarray(np.repeat(fz.duration[fz.order][:, None], 64, 1).astype(np.int32))
r = simulate_batch(fz, ScenarioTable(n_scenarios=64, dense=dense))
print("makespan", r.makespan[:2])
print(N.lib().ks_jit_log().decode())
from paper_2006_03318_b200.workloads import gpt_trace
w = gpt_trace(n_tasks=100000)
fz = FrozenGraph.from_graph(w.graph)
dense = np.ascontiguousarray(np.repeat(fz.duration[fz.order][:, None], 64, 1).astype(np.int32))
r = simulate_batch(fz, ScenarioTable(n_scenarios=64, dense=dense))
print("gpt makespan", r.makespan[:2])
print(N.lib().ks_jit_log().decode())
