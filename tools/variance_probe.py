"""Config-4 timing stability: several timed rounds per allocation, several
allocations per process, plus the int32->int64 copy of the same matrices."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2006_03318_b200.batch import ScenarioTable, simulate_batch_device  # noqa: E402

torch.cuda.set_device(0)
w, fz = bench.build_workload(0)
S = bench.S_PER_GPU
rows, L = fz.n, fz.L
base = torch.from_numpy(fz.duration[fz.order].copy()).cuda()


def alloc(seed):
    dense = torch.empty((rows, S), dtype=torch.int32, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    step = max(1, (1 << 28) // S)
    for r0 in range(0, rows, step):
        r1 = min(rows, r0 + step)
        k = torch.randint(900, 1101, (r1 - r0, S), generator=g, device="cuda", dtype=torch.int64)
        dense[r0:r1] = ((2 * base[r0:r1, None] * k + 1000) // 2000).to(torch.int32)
    start = torch.empty((rows, S), dtype=torch.int64, device="cuda")
    return dense, start


def timed(fn, n):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    dense, start = alloc(1000 + rep)
    ms = torch.empty(S, dtype=torch.int64, device="cuda")
    lb = torch.empty((S, L), dtype=torch.int64, device="cuda")
    table = ScenarioTable(n_scenarios=S, dense=dense)
    st = torch.cuda.current_stream().cuda_stream

    def step():
        simulate_batch_device(fz, table, makespan=ms, lane_busy=lb, start=start, stream=st)
    step()
    res = [timed(step, 5) for _ in range(3)]
    cp = timed(lambda: start.copy_(dense), 3)
    print(f"alloc {rep}: dense@{dense.data_ptr():#x} start@{start.data_ptr():#x} "
          f"sim ms {['%.2f' % x for x in res]} copy {cp:.2f} ms", flush=True)
    del dense, start, table
    torch.cuda.empty_cache()
    time.sleep(1)
