#!/bin/bash
# Round-2 first GPU session: new parity tests, full GPU suite, bench, self-spawned 2-rank bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py tests/test_shard_gloo.py "tests/test_sim_gpu.py::test_every_maxplus_kernel_path_matches_oracle" -q -x > gpurun_out/tests_new.log 2>&1; tail -3 gpurun_out/tests_new.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/tests.log 2>&1; tail -3 gpurun_out/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-600
DDSIM_BENCH_SAME_DEVICE=1 DDSIM_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --scenarios 16384 --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/bench_g2.log 2>&1; tail -1 gpurun_out/bench_g2.log | cut -c1-400
