"""Config 4 as one launch vs the scenarios split into k launches on k streams
(same results; checks whether concurrent launches at different record
positions draw more HBM bandwidth)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2006_03318_b200.batch import ScenarioTable, simulate_batch_device  # noqa: E402

S = 65536
w, fz = bench.build_workload(0)
rows, L = fz.n, fz.L
base = torch.from_numpy(fz.duration[fz.order].copy()).cuda()
dense = torch.empty((rows, S), dtype=torch.int32, device="cuda")
g = torch.Generator(device="cuda")
g.manual_seed(1)
step = max(1, (1 << 28) // S)
for r0 in range(0, rows, step):
    r1 = min(rows, r0 + step)
    k = torch.randint(900, 1101, (r1 - r0, S), generator=g, device="cuda", dtype=torch.int64)
    dense[r0:r1] = ((2 * base[r0:r1, None] * k + 1000) // 2000).to(torch.int32)
start = torch.empty((rows, S), dtype=torch.int64, device="cuda")
ms = torch.empty(S, dtype=torch.int64, device="cuda")
lb = torch.empty((S, L), dtype=torch.int64, device="cuda")
ref_ms = None
for k in [1, 2, 4, 1, 2, 4]:
    streams = [torch.cuda.Stream() for _ in range(k)]
    w_ = S // k
    parts = [(ScenarioTable(n_scenarios=w_, dense=dense[:, i * w_:(i + 1) * w_]), i) for i in range(k)]

    def step_():
        ev = torch.cuda.current_stream().record_event()
        for (tab, i), st in zip(parts, streams):
            st.wait_event(ev)
            simulate_batch_device(fz, tab, makespan=ms[i * w_:(i + 1) * w_], lane_busy=lb[i * w_:(i + 1) * w_],
                                  start=start[:, i * w_:], start_ld=S, stream=st.cuda_stream)
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
    for _ in range(3):
        step_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        step_()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 5
    if ref_ms is None:
        ref_ms = ms.clone()
    same = bool(torch.equal(ms, ref_ms))
    print(f"k={k}: {t:.3f} ms/step  {rows * S * 12 / t / 1e6:.0f} GB/s  same={same}", flush=True)
