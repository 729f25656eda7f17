#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_shim_gpu.py -x -q > gpurun_out/pytest_shim.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_shim.log
for r in 1 2; do
  PARAC_SHIM_TIMING=1 ./tools/_build/dropin_time 128 5 2 2>&1 | tail -3 >> gpurun_out/dropin3.txt
done
