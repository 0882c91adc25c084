#!/bin/bash
# lean breakdown merge with L2 prefetch distance sweep at 65,536 x 100k
mkdir -p gpurun_out
DDSIM_BD_PF=8 timeout 900 python -m pytest tests/test_breakdown_gpu.py -x -q > gpurun_out/bdpf_tests.log 2>&1; tail -1 gpurun_out/bdpf_tests.log
for d in 0 2 4 8 16 32; do echo pf=$d; DDSIM_BD_PF=$d timeout 600 python tools/bench_breakdown.py 2>&1 | tail -1 | cut -c80-200; done
