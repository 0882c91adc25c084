import sys, os
sys.path[:0]=['.','oracle']
import torch, bench
from paper_2006_03318_b200.batch import simulate_batch_device
c = int(os.environ.get("CFG", "2"))
fz, table, _g, _i = bench.build_config(c, 0)
S=table.n_scenarios
st = torch.empty((fz.n, S), dtype=torch.int64, device="cuda:0")
ms = torch.empty(S, dtype=torch.int64, device="cuda:0")
lb = torch.empty((S, fz.L), dtype=torch.int64, device="cuda:0")
for _ in range(3):
    simulate_batch_device(fz, table, makespan=ms, lane_busy=lb, start=st, stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("done")
