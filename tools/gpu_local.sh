#!/bin/bash
# CTA-local ready stack: parity with it on, K3 time per capacity
mkdir -p gpurun_out
PARAC_LOCAL_STACK=32 timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_fuzz_gpu.py -x -q > gpurun_out/pytest_local.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_local.log
for e in 0 16 32 64 0; do
  for w in poisson3d_128 poisson27_96 poisson2d_256; do
    echo "== local=$e $(PARAC_LOCAL_STACK=$e timeout 300 python tools/k3_time.py --workload $w --reps 5 2>&1 | tail -1 | cut -c1-140)" >> gpurun_out/local.txt
  done
done
PARAC_LOCAL_STACK=32 timeout 300 python tools/profile_factor.py --n 128 --json gpurun_out/prof128_local32.json > /dev/null 2>&1
