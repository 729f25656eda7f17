#!/bin/bash
mkdir -p gpurun_out
./tools/microbench/k3parts > gpurun_out/k3parts.txt 2>&1
timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_fullsize_gpu.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_factor.py --n 128 --json gpurun_out/prof128.json > /dev/null 2>&1
timeout 300 python tools/profile_factor.py --n 96 --workload poisson27 --json gpurun_out/prof27.json > /dev/null 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-pcg > gpurun_out/bench.json 2> gpurun_out/bench.err
