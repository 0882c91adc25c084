# breakdown sweep: parity suite + throughput (sweep auto / windowed merge; NOBULK=1: per-thread cp.async staging)
mkdir -p gpurun_out
[ -n "$NOTEST" ] || timeout 900 python -m pytest tests/test_breakdown_gpu.py tests/test_whatif_batch_gpu.py -q -x > gpurun_out/bd_tests.log 2>&1; tail -3 gpurun_out/bd_tests.log
for S in ${SIZES:-65536 32768 16384}; do
  for m in ${MODES:-1 -1}; do
    echo "S=$S sweep=$m nobulk=${NOBULK:-}" | tee -a gpurun_out/bd_timing.log
    S=$S DDSIM_BD_SWEEP=$m timeout 600 python tools/bench_breakdown.py 2>&1 | tail -1 | cut -c1-330 | tee -a gpurun_out/bd_timing.log
  done
done
