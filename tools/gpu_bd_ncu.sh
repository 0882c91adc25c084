# ncu of the breakdown streaming sweep at 65,536 x 100k (first launch: parts only)
mkdir -p gpurun_out
S=65536 timeout 900 ncu --set full --import-source on -k regex:breakdown_stream -c 1 -o gpurun_out/bd_stream65k python tools/bench_breakdown.py > gpurun_out/bd_ncu.log 2>&1
tail -2 gpurun_out/bd_ncu.log
