#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_solve_gpu.py tests/test_factor_gpu.py tests/test_shim_gpu.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/sweep_profile.py 128 > gpurun_out/sweep_profile.txt 2>&1
rm -f gpurun_out/pcg_time.jsonl
for w in 32 64; do PARAC_TAIL_WIDTH=$w timeout 300 python tools/pcg_time.py >> gpurun_out/pcg_time.jsonl 2>&1; done
PARAC_WIDE_WEIGHT=0 timeout 300 python tools/pcg_time.py >> gpurun_out/pcg_time.jsonl 2>&1
timeout 300 python tools/pcg_time.py --workload poisson27 --n 96 >> gpurun_out/pcg_time.jsonl 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py -x -q > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
