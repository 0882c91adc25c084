#!/bin/bash
# ncu --set full of config 3's segment kernels
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ddsim_seg_transfer" -s 1 -c 1 -o gpurun_out/prof_c3_t python tools/experiments/c3one.py > gpurun_out/ncu_c3_t.log 2>&1; tail -1 gpurun_out/ncu_c3_t.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ddsim_seg_replay" -s 3 -c 1 -o gpurun_out/prof_c3_r python tools/experiments/c3one.py > gpurun_out/ncu_c3_r.log 2>&1; tail -1 gpurun_out/ncu_c3_r.log
ls -la gpurun_out/*.ncu-rep
