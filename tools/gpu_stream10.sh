#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_solve_gpu.py -x -q > gpurun_out/pytest_stream.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stream.log
for rep in 1 2; do for c in 4 6 8; do PARAC_STREAM_CTAS=$c timeout 300 python tools/factor_time.py >> gpurun_out/stream_sweep.txt 2>&1; done; done
for c in 4 8; do PARAC_STREAM_CTAS=$c timeout 300 python tools/factor_time.py --workload poisson27 --n 96 >> gpurun_out/stream_sweep.txt 2>&1; done
