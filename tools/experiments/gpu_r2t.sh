#!/bin/bash
mkdir -p gpurun_out
NVTX_INJECTION64_PATH=/usr/local/cuda/lib64/libcupti.so timeout 600 python tools/cupti_capture.py --out gpurun_out/cupti_trace.json 2>&1 | tail -20
timeout 600 python -m pytest tests/test_cupti_gpu.py -q -x 2>&1 | tail -15
