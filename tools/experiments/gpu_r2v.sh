#!/bin/bash
# segment kernels: unroll / min blocks per SM
mkdir -p gpurun_out
for env in "X=1" "DDSIM_SEG_UNROLL=1" "DDSIM_SEG_MINB=6" "DDSIM_SEG_MINB=8" "DDSIM_SEG_UNROLL=1 DDSIM_SEG_MINB=6" "DDSIM_SEG_TPS=8192" "DDSIM_SEG_MIN_LEN=160"; do
  echo "== $env"
  env $env timeout 300 python tools/seg_probe.py config3 2>&1 | grep '"seg"' 
  env $env timeout 300 python tools/seg_probe.py config2 2>&1 | grep '"seg"'
done
