"""Config-4 timing stability: several timed rounds per allocation, several
allocations per process, plus the int32->int64 copy of the same matrices."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
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


ENQ = []


def timed(fn, n):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    ENQ.append((time.perf_counter() - t0) * 1e3 / n)  # host ms per enqueued step
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
    from paper_2006_03318_b200 import _native as N
    cp = timed(lambda: N.lib().ks_probe_widen(dense.data_ptr(), start.data_ptr(), rows * S, st), 3)
    print(f"alloc {rep}: sim ms {['%.2f' % x for x in res]} probe-copy {cp:.2f} ms "
          f"host enqueue ms/step {['%.3f' % x for x in ENQ[-4:-1]]}", flush=True)
    del dense, start, table
    torch.cuda.empty_cache()
    time.sleep(1)
