"""cProfile of the drop-in API on config 1 (Analysis.from_trace + whatif("amp"))."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_03318_b200 import Analysis  # noqa: E402
from paper_2006_03318_b200 import workloads as W  # noqa: E402

w = W.resnet50_trace()
Analysis.from_trace(w.trace).whatif("amp")  # warm-up (CUDA context, JIT, CUB)
t0 = time.perf_counter()
Analysis.from_trace(w.trace).whatif("amp")
print("wall", time.perf_counter() - t0)
pr = cProfile.Profile()
pr.enable()
Analysis.from_trace(w.trace).whatif("amp")
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
