"""Traffic-pattern probe variants (DDSIM_PROBE_VARIANT) at the config-4 size:
int32 [100k x 65,536] -> int64, GB/s of compulsory traffic (CUDA events)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2006_03318_b200 import _native as N  # noqa: E402

n = 100_000 * 65_536
src = torch.randint(0, 1 << 20, (n,), dtype=torch.int32, device="cuda")
dst = torch.empty(n, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
for var in sys.argv[1:] or ["0", "1", "2", "3", "4", "5", "0"]:
    os.environ["DDSIM_PROBE_VARIANT"] = var
    for _ in range(2):
        N.check(N.lib().ks_probe_widen(src.data_ptr(), dst.data_ptr(), n, st.cuda_stream))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        N.check(N.lib().ks_probe_widen(src.data_ptr(), dst.data_ptr(), n, st.cuda_stream))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    ok = bool(torch.equal(dst[:: 1 << 20], src[:: 1 << 20].long()))
    print(f"variant {var}: {ms:.3f} ms  {12 * n / ms / 1e6:.0f} GB/s  correct={ok}", flush=True)
