#!/bin/bash
for S in 8192 16384 32768; do for K in 2 3 4 8 16; do
  DDSIM_SEG_K=$K timeout 300 python tools/seg_probe.py config4 $S 2>&1 | grep '"seg"' | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print($S, $K, l['ms'])"
done; done
