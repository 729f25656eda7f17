#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_solve_gpu.py tests/test_factor_gpu.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
PARAC_QUEUE=prio timeout 600 python -m pytest tests/test_factor_gpu.py -x -q > gpurun_out/pytest_prio.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_prio.log
timeout 300 python tools/sweep_profile.py 128 > gpurun_out/sweep_profile.txt 2>&1
timeout 300 python tools/pcg_time.py > gpurun_out/pcg_time.jsonl 2>&1
timeout 300 python tools/profile_factor.py --n 128 --json gpurun_out/prof128_fifo.json > /dev/null 2>&1
PARAC_QUEUE=prio timeout 300 python tools/profile_factor.py --n 128 --json gpurun_out/prof128_prio.json > /dev/null 2>&1
PARAC_QUEUE=prio timeout 300 python tools/profile_factor.py --n 96 --workload poisson27 --json gpurun_out/prof27_prio.json > /dev/null 2>&1
timeout 300 python tools/profile_factor.py --n 96 --workload poisson27 --json gpurun_out/prof27_fifo.json > /dev/null 2>&1
