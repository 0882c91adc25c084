mkdir -p gpurun_out
for p in 1 2 3; do
  echo "--- no nvidia-smi"; timeout 400 python tools/variance_probe.py 2 2>&1 | grep alloc
  echo "--- with nvidia-smi -lms 200"
  nvidia-smi -i 0 --query-gpu=index,clocks.sm,clocks.mem,power.draw --format=csv,noheader,nounits -lms 200 > gpurun_out/smi.csv 2>&1 &
  SMI=$!
  timeout 400 python tools/variance_probe.py 2 2>&1 | grep alloc
  kill $SMI
done
