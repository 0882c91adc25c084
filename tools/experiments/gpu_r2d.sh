#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_seg_gpu.py -q -x 2>&1 | tail -2
for tps in 256 512 2048 4096; do
  timeout 600 python tools/seg_probe.py config4 8192 32768 DDSIM_SEG_TPS=$tps DDSIM_SEG_MAX_S=65536 2>&1 | grep '"seg"'
  timeout 600 python tools/seg_probe.py config2 DDSIM_SEG_TPS=$tps 2>&1 | grep '"seg"'
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"seg" --csv --log-file gpurun_out/seg_launches2.csv python tools/seg_probe.py config4 8192 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/seg_launches2.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:7]: print(r[ki][:40], r[vi])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"seg" --csv --log-file gpurun_out/seg_launches3.csv python tools/seg_probe.py config2 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/seg_launches3.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:7]: print(r[ki][:40], r[vi])
PY
