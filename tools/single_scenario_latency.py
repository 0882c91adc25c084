"""Single-scenario device latency of simulate (the drop-in simulate(graph) /
Analysis.whatif path) on the config-1 and config-4 graphs, and where the
drop-in simulate(graph) call spends its time."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2006_03318_b200 import simulate  # noqa: E402
from paper_2006_03318_b200 import workloads as W  # noqa: E402
from paper_2006_03318_b200.batch import ScenarioTable, simulate_batch_device  # noqa: E402
from paper_2006_03318_b200.frozen import FrozenGraph  # noqa: E402


def med(fn, k=12):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts[2:]) * 1e3


for name, g in (("resnet50 (config 1)", W.resnet50_trace().graph),
                ("gpt 100k (config 4)", W.gpt_trace(seed=0, n_tasks=100_000).graph)):
    fz = FrozenGraph.from_graph(g, device=0)
    tab = ScenarioTable(n_scenarios=1)
    st = torch.empty((fz.n, 1), dtype=torch.int64, device="cuda")
    ms = torch.empty(1, dtype=torch.int64, device="cuda")
    simulate_batch_device(fz, tab, makespan=ms, start=st)  # programs built on first use
    t_dev = med(lambda: simulate_batch_device(fz, tab, makespan=ms, start=st))
    simulate(g)
    t_freeze = med(lambda: FrozenGraph.from_graph(g, device=0), 7)
    t_drop = med(lambda: simulate(g), 7)
    print(f"{name}: device simulate {t_dev:.3f} ms, freeze of the Python graph {t_freeze:.2f} ms, "
          f"drop-in simulate(graph) {t_drop:.2f} ms")
