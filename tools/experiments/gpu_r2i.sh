#!/bin/bash
# Round-2 validation of the restored checkpoint: full GPU suite, smoke, bench (all configs), reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_i.txt
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/tests_i.log 2>&1; tail -3 gpurun_out/tests_i.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_i_c4.jsonl 2> gpurun_out/bench_i_c4.err; tail -c 3000 gpurun_out/bench_i_c4.jsonl
for c in 1 2 3 5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_i_c$c.jsonl 2> gpurun_out/bench_i_c$c.err; echo "config $c rc=$?"; tail -c 1500 gpurun_out/bench_i_c$c.jsonl
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_i_ref.jsonl 2>&1; tail -c 800 gpurun_out/bench_i_ref.jsonl
