#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_shim_gpu.py tests/test_factor_gpu.py tests/test_solve_gpu.py -x -q > gpurun_out/pytest_stream.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stream.log
PARAC_SHIM_TIMING=1 timeout 300 ./tools/_build/dropin_time 128 4 2 > gpurun_out/dropin.txt 2>&1
timeout 900 python bench.py --no-batch > gpurun_out/bench.json 2> gpurun_out/bench.err
