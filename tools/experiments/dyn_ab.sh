#!/bin/bash
# Branch-free lanes handler (latency-bound launches) vs the specialised if-chain:
# parity, config 2 kernel times (ncu launch list), config 4 both ways.
mkdir -p gpurun_out
summ() { python - "$1" <<'PY'
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
agg = collections.defaultdict(list)
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows[1:]:
    try: agg[r[ki][:40]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    except ValueError: pass
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:4]:
    print(f"   {k:40s} n={len(v):3d} median={sorted(v)[len(v)//2]:10.1f} us")
PY
}
timeout 900 python -m pytest tests/test_sweeps_gpu.py tests/test_sim_gpu.py tests/test_whatif_batch_gpu.py tests/test_breakdown_gpu.py -q -x 2>&1 | tail -1
DDSIM_LANES_DYN=1 timeout 900 python -m pytest tests/test_sim_gpu.py -q -x -k "dense" 2>&1 | tail -1
for dyn in 1 0; do
  DDSIM_LANES_DYN=$dyn timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_dyn$dyn.csv python tools/bench_configs.py --only 2,3 --out gpurun_out/c23.json > gpurun_out/c23.log 2>&1
  echo "DYN=$dyn configs 2+3 kernels:"; summ gpurun_out/c2_dyn$dyn.csv
done
timeout 600 python tools/bench_configs.py --only 1,2,3 --out gpurun_out/c123.json > gpurun_out/c123.log 2>&1; grep -o '"device_s": [0-9.e-]*' gpurun_out/c123.log
for cfg in "DDSIM_LANES_DYN=0" "DDSIM_LANES_DYN=1" "DDSIM_LANES_DYN=0"; do
  env $cfg timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/v.log 2>&1
  echo "$cfg config4: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/v.log) $(grep -o '"pattern_copy_gbs": [0-9.]*' gpurun_out/v.log)"
done
