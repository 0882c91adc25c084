#!/bin/bash
for env in "X=1" "DDSIM_SEG_STAGES=2" "DDSIM_SEG_STAGES=3" "DDSIM_SEG_STAGES=6" "DDSIM_SEG_TPS=2048" "DDSIM_SEG_TPS=8192"; do
  echo "== $env"
  env $env timeout 300 python tools/seg_probe.py config4 8192 2>&1 | grep '"seg"'
  env $env timeout 300 python tools/seg_probe.py config3 2>&1 | grep '"seg"'
done
