#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_seg_gpu.py -q -x > gpurun_out/seg_tests.log 2>&1; tail -15 gpurun_out/seg_tests.log
timeout 600 python tools/seg_probe.py config2 > gpurun_out/seg_c2.log 2>&1; cat gpurun_out/seg_c2.log | tail -4
timeout 900 python tools/seg_probe.py config4 8192 16384 32768 > gpurun_out/seg_c4.log 2>&1; cat gpurun_out/seg_c4.log | tail -12
grep -i "seg\|fail" <(python -c "
import sys; sys.path.insert(0,'.')
from paper_2006_03318_b200 import _native as N
print((N.lib().ks_jit_log() or b'').decode())") | head
