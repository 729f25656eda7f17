#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_factor_gpu.py tests/test_fullsize_gpu.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for c0 in 64 128 256; do
  timeout 300 python tools/profile_factor.py --n 128 --c0 $c0 --json gpurun_out/prof128_c0_$c0.json > /dev/null 2>&1
done
timeout 600 python bench.py --no-cpu-baseline --no-pcg > gpurun_out/bench.json 2> gpurun_out/bench.err
