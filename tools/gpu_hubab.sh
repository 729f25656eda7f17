#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_fuzz_gpu.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
VARIANTS="A B A B" ./tools/gpu_hubvar.sh
