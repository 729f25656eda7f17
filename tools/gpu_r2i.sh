#!/bin/bash
# Radix sort v2 (per-digit row scans): ordering / solve / hub GPU tests, nnz-sort timing, launch list of the nnz-sort
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ordering_gpu.py tests/test_solve_gpu.py tests/test_hub_gpu.py -q -x > gpurun_out/pytest_sort.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sort.log
timeout 300 python tools/ordering_time.py > gpurun_out/ordering_time.txt 2>&1
timeout 300 python tools/pcg_first_call.py > gpurun_out/pcg_first_call.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_ord.csv python tools/ordering_time.py > gpurun_out/ncu_ord.log 2>&1
