#!/bin/bash
# K3 iteration: parity tests, microbench, timing per PARAC_KEEP_EXTRA setting, critical-path profile
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_fullsize_gpu.py tests/test_fuzz_gpu.py -x -q > gpurun_out/pytest_k3b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k3b.log
./tools/microbench/k3parts > gpurun_out/k3parts_b.txt 2>&1
for e in ${KEEPS:-3,16384}; do
  for w in poisson3d_128 poisson27_96 poisson2d_256; do
    echo "== keep_extra=$e $(PARAC_KEEP_EXTRA=$e timeout 300 python tools/k3_time.py --workload $w --reps 5 2>&1 | tail -1)" >> gpurun_out/k3b.txt
  done
done
timeout 300 python tools/profile_factor.py --n 128 --json gpurun_out/prof128b.json > gpurun_out/prof128b.txt 2>&1
