#!/bin/bash
mkdir -p gpurun_out
PARAC_STREAM_BATCH=1 timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_factor_gpu.py tests/test_multirank_gpu.py -x -q > gpurun_out/pytest_stream.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stream.log
for c in 8 16 32; do PARAC_STREAM_BATCH=1 PARAC_STREAM_CTAS=$c timeout 900 python bench.py --workload batch_64x64 --no-cpu-baseline > gpurun_out/bench_batch_c$c.json 2> gpurun_out/bench_batch_c$c.err; done
