#!/bin/bash
# segment length / derived-mode sweep on the small-S configs (warp-parallel scan)
for w in config2 config3; do
  for m in 128 192 256 320 448; do timeout 300 python tools/seg_probe.py $w DDSIM_SEG_MIN_LEN=$m 2>&1 | grep '"seg"'; done
  timeout 300 python tools/seg_probe.py $w DDSIM_FORCE_DERIVED=1 2>&1 | grep '"seg"'
  timeout 300 python tools/seg_probe.py $w DDSIM_SEG_TPS=8192 2>&1 | grep '"seg"'
  timeout 300 python tools/seg_probe.py $w DDSIM_SEG_TPS=8192 DDSIM_SEG_MIN_LEN=192 2>&1 | grep '"seg"'
done
timeout 300 python tools/seg_probe.py config4 2048 DDSIM_SEG_MIN_LEN=192 2>&1 | grep '"seg"'
timeout 300 python tools/seg_probe.py config4 2048 DDSIM_SEG_TPS=8192 2>&1 | grep '"seg"'
