#!/bin/bash
timeout 900 python -m pytest tests/test_seg_gpu.py tests/test_fullsize_gpu.py -q -x 2>&1 | tail -1
for e in X=1 DDSIM_SEG_T1=1; do for S in 8192 16384 32768; do
  env $e timeout 300 python tools/seg_probe.py config4 $S 2>&1 | grep -E '"seg"|identical' | python -c "
import json,sys
ls=[json.loads(x) for x in sys.stdin.read().strip().splitlines()]
print('$e', $S, ls[0]['ms'], ls[-1].get('identical'))"
done; done
for e in X=1 DDSIM_SEG_T1=1; do env $e timeout 300 python tools/seg_probe.py config2 2>&1 | grep '"seg"'; done
