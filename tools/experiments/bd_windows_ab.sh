#!/bin/bash
# ks_breakdown time windows per scenario (config-4 shape)
mkdir -p gpurun_out
for k in default 2 10 20 40; do
  if [ $k = default ]; then e=X=1; else e=DDSIM_BD_WINDOWS=$k; fi
  env $e timeout 900 python tools/bench_breakdown.py > gpurun_out/bdw.log 2>&1
  echo "$k: $(tail -1 gpurun_out/bdw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['parts']['s']*1e3,1), 'ms', round(d['parts+layers']['s']*1e3,1), 'ms')" 2>&1 | tail -1)"
done
