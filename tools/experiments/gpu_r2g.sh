#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_transfer" -s 2 -c 1 -o gpurun_out/prof_seg_t python tools/seg_probe.py config4 8192 > gpurun_out/ncu_seg_t.log 2>&1; tail -2 gpurun_out/ncu_seg_t.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_replay" -s 2 -c 1 -o gpurun_out/prof_seg_r python tools/seg_probe.py config4 8192 > gpurun_out/ncu_seg_r.log 2>&1; tail -2 gpurun_out/ncu_seg_r.log
