#!/bin/bash
# chain segment with carries (config 3 on the segment path)
mkdir -p gpurun_out
timeout 600 python tools/seg_probe.py config3 2>&1 | tail -4
timeout 600 python tools/seg_probe.py config2 2>&1 | tail -3
timeout 900 python -m pytest tests/test_fullsize_gpu.py tests/test_seg_gpu.py tests/test_sweeps_gpu.py -q -x 2>&1 | tail -5
