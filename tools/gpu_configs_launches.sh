bash tools/gpu_configs.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lanes|maxplus|listsched|probe" -c 16 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log | cut -c1-200
