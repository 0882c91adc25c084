"""Config-1 latency probe: which kernel path and how long per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tools"))
import bench_configs as B
import torch
from paper_2006_03318_b200 import _native as N
r = B.config1()
print(os.environ.get("TAG", ""), "device_ms", r["device_s"] * 1e3, "launches", N.lib().ks_launch_count())
print(N.lib().ks_jit_log().decode()[-600:])
