mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v1_smi.txt
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/v1_tests.log 2>&1; tail -3 gpurun_out/v1_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/v1_c4.jsonl 2> gpurun_out/v1_c4.err; tail -c 600 gpurun_out/v1_c4.jsonl
timeout 600 python tools/bench_breakdown.py > gpurun_out/v1_bd.log 2>&1; tail -20 gpurun_out/v1_bd.log
