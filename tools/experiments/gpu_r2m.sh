#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/experiments/c3one.py > gpurun_out/c3.log 2>&1
tail -2 gpurun_out/c3.log
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c3_launches.csv')))
hdr=None
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        print(d['ID'], d['Kernel Name'][:60], d['Grid Size'], d['Block Size'], d['Metric Value'])
PY
