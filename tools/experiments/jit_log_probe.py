"""Print the NVRTC log after one derived-duration launch (diagnostics)."""
import sys
sys.path[:0] = ['.', 'oracle']
import bench
from paper_2006_03318_b200 import _native as N
from paper_2006_03318_b200.batch import simulate_batch
fz, table, _g, _i = bench.build_config(2, 0)
try:
    simulate_batch(fz, table)
except Exception as e:  # noqa: BLE001
    print("ERR", e)
print((N.lib().ks_jit_log() or b"").decode()[-6000:])
