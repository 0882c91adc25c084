#!/bin/bash
# round-2 final validation: GPU suite, smoke, bench for every config, reference arms,
# launch lists of the small configs (ncu, cold per-launch times), ncu of the breakdown sweep
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/fin5_smi.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/fin5_tests.log 2>&1; tail -2 gpurun_out/fin5_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/fin5_c4.jsonl 2> gpurun_out/fin5_c4.err; tail -c 400 gpurun_out/fin5_c4.jsonl
for c in 1 2 3 5; do timeout 1200 python bench.py --config $c > gpurun_out/fin5_c$c.jsonl 2> gpurun_out/fin5_c$c.err; echo "config $c rc=$?"; done
timeout 600 python bench.py --impl reference > gpurun_out/fin5_ref_c4.jsonl 2>&1
for c in 1 2 3 5; do timeout 900 python bench.py --impl reference --config $c > gpurun_out/fin5_ref_c$c.jsonl 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"breakdown|bd_" --csv --log-file gpurun_out/fin5_bd_launches.csv python tools/bench_breakdown.py > /dev/null 2>&1
timeout 900 ncu --set full --import-source on -k regex:breakdown_stream -c 1 -o gpurun_out/fin5_bd_stream python tools/bench_breakdown.py > gpurun_out/fin5_bd_ncu.log 2>&1
python - <<'PY'
import json
for c in (4, 1, 2, 3, 5):
    l = json.loads(open(f'gpurun_out/fin5_c{c}.jsonl').read().strip().splitlines()[-1])
    r = json.loads(open(f'gpurun_out/fin5_ref_c{c}.jsonl').read().strip().splitlines()[-1])
    print(c, round(l['ms_per_step'], 3), round(l['roofline']['frac'], 4), "%.4g" % l['value'], "e2e %.4g" % l['e2e']['value'], "ref %.4g" % r['value'], "e2e/ref %.1f" % (l['e2e']['value'] / r['value']), l['clocks'].get('sm_mhz'))
PY
