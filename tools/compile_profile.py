"""Host graph-compiler timings without a device (DDSIM_COMPILE_ONLY): a synthetic
config-5-shaped graph (CPU lanes launching kernels onto stream lanes; lane-order
edges + launch->kernel edges), section times from DDSIM_INGEST_TIMING."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("DDSIM_COMPILE_ONLY", "1")
os.environ.setdefault("DDSIM_INGEST_TIMING", "1")
import numpy as np  # noqa: E402

from paper_2006_03318_b200.frozen import FrozenGraph  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
rng = np.random.default_rng(0)
CPU, STREAMS = 4, 20
L = CPU + STREAMS
half = n // 2                            # launches 0..half-1, kernels half..n-1
lane = np.empty(n, np.int32)
lane[:half] = np.arange(half) % CPU
lane[half:] = CPU + rng.integers(0, STREAMS, n - half)
# document order interleaves: launch i, kernel i
perm = np.empty(n, np.int64)
perm[0::2] = np.arange(half)
perm[1::2] = half + np.arange(n - half)
pos = np.empty(n, np.int64)
pos[perm] = np.arange(n)
order = np.lexsort((pos, lane)).astype(np.int32)
cnt = np.bincount(lane, minlength=L)
lop = np.zeros(L + 1, np.int32)
lop[1:] = np.cumsum(cnt)
same = lane[order[1:]] == lane[order[:-1]]
es = np.concatenate([order[:-1][same], np.arange(half, dtype=np.int32)])
ed = np.concatenate([order[1:][same], (half + np.arange(half)).astype(np.int32)])
dur = rng.integers(1000, 20000, n)
for rep in range(2):
    t = time.perf_counter()
    fz = FrozenGraph(ids=np.arange(n), duration=dur, gap=np.zeros(n, np.int64),
                     ready=np.zeros(n, np.int64), lane=lane, priority=np.zeros(n, np.int32),
                     flags=np.zeros(n, np.uint8), group=np.zeros(n, np.uint32),
                     edge_src=es, edge_dst=ed, lane_order_ptr=lop, lane_order=order,
                     lanes=list(range(L)))
    print(f"rep {rep}: freeze {time.perf_counter()-t:.3f} s ({n} tasks, {es.size} edges, "
          f"{os.cpu_count()} cpus, chained={fz.chained})", flush=True)
    del fz
