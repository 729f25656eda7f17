#!/bin/bash
mkdir -p gpurun_out
./tools/microbench/tailbench > gpurun_out/tailbench.txt 2>&1
timeout 600 python -m pytest tests/test_solve_gpu.py tests/test_fullsize_gpu.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/sweep_profile.py 128 > gpurun_out/sweep_profile.txt 2>&1
timeout 300 python tools/pcg_time.py > gpurun_out/pcg_time.jsonl 2>&1
timeout 300 python tools/profile_factor.py --n 128 --json gpurun_out/prof128.json > /dev/null 2>&1
