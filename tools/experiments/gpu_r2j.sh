#!/bin/bash
# new parity tests (scale vectors, config 1 full, insert generators as tables)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_scale_vectors_gpu.py tests/test_whatif_batch_gpu.py "tests/test_fullsize_gpu.py::test_config1_full_baseline_and_amp" tests/test_breakdown_gpu.py tests/test_acceptance_gpu.py -q -x 2>&1 | tail -30
