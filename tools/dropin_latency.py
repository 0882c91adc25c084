"""Latency of the drop-in calls on config 1 (ResNet-50-like, ~10k tasks):
simulate(graph), simulate_batch of 2 scenarios (host buffers), whatif("amp"),
Analysis.from_trace -- medians of repeated calls after a warm-up."""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_03318_b200 import Analysis, simulate  # noqa: E402
from paper_2006_03318_b200 import workloads as W  # noqa: E402
from paper_2006_03318_b200.batch import ScenarioTable, compile_scale_sweep, simulate_batch  # noqa: E402
from paper_2006_03318_b200.frozen import FrozenGraph  # noqa: E402
from paper_2006_03318_b200.scenarios import whatif_amp  # noqa: E402
from paper_2006_03318_b200.transform import Selector  # noqa: E402


def med(fn, k=15):
    fn()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return round(statistics.median(ts) * 1e3, 3)


w = W.resnet50_trace()
a = Analysis.from_trace(w.trace)
g = a.graph
amp = whatif_amp(g)
scen = [[], [(Selector.from_object(x["selector"]), x["factor"]) for x in amp.steps]]
group_of, ptr, steps = compile_scale_sweep(g, scen)
fz = FrozenGraph.from_graph(g, group_of=group_of)
table = ScenarioTable(n_scenarios=2, scale_ptr=ptr, scale=steps)
out = {
    "tasks": len(g.tasks),
    "simulate_ms": med(lambda: simulate(g)),
    "freeze_ms": med(lambda: FrozenGraph.from_graph(g, group_of=group_of).close()),
    "simulate_batch_2_ms": med(lambda: simulate_batch(fz, table)),
    "whatif_amp_ms": med(lambda: a.whatif("amp"), k=7),
    "from_trace_ms": med(lambda: Analysis.from_trace(w.trace), k=5),
}
print(json.dumps(out))
