#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_factor_gpu.py tests/test_multirank_gpu.py -x -q > gpurun_out/pytest_stream.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stream.log
timeout 900 python bench.py --workload batch_64x64 --no-cpu-baseline > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err
