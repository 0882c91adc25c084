#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_seg_gpu.py -q -x 2>&1 | tail -1
timeout 600 python tools/seg_probe.py config4 4096 8192 16384 32768 2>&1 | grep -v '"single"'
timeout 600 python tools/seg_probe.py config2 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"seg" -c 6 --csv --log-file gpurun_out/seg_launches4.csv python tools/seg_probe.py config4 8192 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/seg_launches4.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:7]: print(r[ki][:40], r[vi])
PY
