#!/bin/bash
# memcheck over the segment-path suites (warp scan, int32 expansion) + config-3 chain segment info
mkdir -p gpurun_out
for t in "tests/test_seg_gpu.py" "tests/test_scale_vectors_gpu.py" "tests/test_sim_gpu.py"; do
  timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest $t -m gpu -x -q -p no:cacheprovider > gpurun_out/memcheck_seg.log 2>&1
  echo "memcheck $t rc=$? $(grep -E 'passed|failed' gpurun_out/memcheck_seg.log | tail -1) $(grep -c 'Invalid\|ERROR SUMMARY: [1-9]' gpurun_out/memcheck_seg.log)"
done
timeout 300 python - <<'PY'
import bench
fz, table, _g, _i = bench.build_config(3, 0)
i = fz.info
print("config3 rows", fz.n, "chain seg", i.seg_chain_begin, i.seg_chain_end, "carries", i.n_carries, "cuts", i.n_lane_cuts)
PY
