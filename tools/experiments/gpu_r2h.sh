#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_seg_gpu.py -q -x 2>&1 | tail -2
timeout 600 python tools/seg_probe.py config4 8192 32768 2>&1 | grep -v single
timeout 600 python tools/seg_probe.py config2 2>&1 | grep -v single
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/tests_h.log 2>&1; tail -2 gpurun_out/tests_h.log
