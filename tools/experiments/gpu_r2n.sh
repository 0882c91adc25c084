#!/bin/bash
# derived durations in the lanes kernels (DK 0): correctness + configs 2/3 timing
mkdir -p gpurun_out
timeout 600 python tools/seg_probe.py config3 2>&1 | tail -3
timeout 600 python tools/seg_probe.py config2 2>&1 | tail -3
DDSIM_NO_DERIVED=1 timeout 600 python tools/seg_probe.py config3 2>&1 | tail -3
timeout 1700 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
python -c "
import sys; sys.path.insert(0,'.')
from paper_2006_03318_b200 import _native as N
print((N.lib().ks_jit_log() or b'').decode()[-3000:])" | grep -iE "fail|error" | head
