#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/seg_probe.py config4 8192 2>&1 | grep -v single | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,launch__registers_per_thread --clock-control none -k regex:"seg|lanes" -c 6 --csv --log-file gpurun_out/c4_8192.csv python tools/seg_probe.py config4 8192 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c4_8192.csv')))
hdr=None
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); print(d['ID'], d['Kernel Name'][:40], d['Grid Size'], d['Metric Name'], d['Metric Value'])
PY
