#!/bin/bash
mkdir -p gpurun_out
for tps in 256 1024 2048 4096; do
  timeout 600 python tools/seg_probe.py config4 8192 32768 DDSIM_SEG_TPS=$tps DDSIM_SEG_MAX_S=65536 2>&1 | grep '"seg"'
done > gpurun_out/seg_tps_c4.log
cat gpurun_out/seg_tps_c4.log
for tps in 256 1024 2048 4096; do
  timeout 600 python tools/seg_probe.py config2 DDSIM_SEG_TPS=$tps 2>&1 | grep '"seg"'
done > gpurun_out/seg_tps_c2.log
cat gpurun_out/seg_tps_c2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"seg|lanes|expand|maxplus" --csv --log-file gpurun_out/seg_launches.csv python tools/seg_probe.py config4 8192 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/seg_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:40]: print(r[ki][:40], r[vi])
PY
