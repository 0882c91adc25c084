#!/bin/bash
# configs 2/3 (latency-bound lanes kernel) under pipeline-depth / block-size variants
mkdir -p gpurun_out
for cfg in "X=1" "DDSIM_LANES_STAGES=2" "DDSIM_LANES_STAGES=3" "DDSIM_LANES_STAGES=6" "DDSIM_LANES_STAGES=8" "DDSIM_LANES_BD=64" "DDSIM_JIT_UNROLL=3" "X=1"; do
  env $cfg timeout 600 python tools/bench_configs.py --only 2,3 --out gpurun_out/ab_cfg.json > gpurun_out/ab_cfg.log 2>&1
  echo "$cfg: $(python -c "import json; d=json.load(open('gpurun_out/ab_cfg.json')); print({k: round(v['device_s']*1e3, 3) for k, v in d.items()})" 2>&1 | tail -1)"
done
