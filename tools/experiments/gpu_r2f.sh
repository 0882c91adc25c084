#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_seg_gpu.py -q -x 2>&1 | tail -3
timeout 600 python tools/seg_probe.py config4 4096 8192 16384 32768 2>&1
timeout 600 python tools/seg_probe.py config2 2>&1
for tps in 1024 2048 8192; do timeout 600 python tools/seg_probe.py config4 8192 32768 DDSIM_SEG_TPS=$tps 2>&1 | grep '"seg"'; done
