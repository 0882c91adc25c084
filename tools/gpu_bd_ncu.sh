mkdir -p gpurun_out
S=16384 DDSIM_BD_SWEEP=1 timeout 900 ncu --set full --import-source on -k regex:breakdown_stream -c 1 -o gpurun_out/bd_stream python tools/bench_breakdown.py > gpurun_out/bd_ncu.log 2>&1
S=16384 DDSIM_BD_SWEEP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"breakdown|bd_" --csv --log-file gpurun_out/bd_launches.csv python tools/bench_breakdown.py > /dev/null 2>&1
tail -3 gpurun_out/bd_ncu.log
