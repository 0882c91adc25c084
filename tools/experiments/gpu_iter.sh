#!/bin/bash
# Fast iteration: GPU tests + bench (device arm only) + ncu of the hot kernel.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; tail -2 gpurun_out/tests.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
DDSIM_NO_LANES=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/bench_nolanes.log 2>&1; tail -1 gpurun_out/bench_nolanes.log | cut -c1-300
S=${NCU_S:-65536}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-lanes} -s 1 -c 1 -o gpurun_out/prof_hot python bench.py --scenarios $S --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
