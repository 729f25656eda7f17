#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_factor_gpu.py tests/test_multirank_gpu.py tests/test_shim_gpu.py -x -q > gpurun_out/pytest_stream.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stream.log
for s in 1 0; do PARAC_STREAM=$s timeout 900 python bench.py --workload batch_64x64 --no-cpu-baseline > gpurun_out/bench_batch_s$s.json 2> gpurun_out/bench_batch_s$s.err; done
for c in 16 32; do PARAC_STREAM_CTAS=$c timeout 900 python bench.py --workload batch_64x64 --no-cpu-baseline > gpurun_out/bench_batch_c$c.json 2> gpurun_out/bench_batch_c$c.err; done
PARAC_STREAM=3 timeout 300 python tools/factor_time.py --reps 3 >> gpurun_out/stream_sweep.txt 2>&1
timeout 300 python tools/factor_time.py >> gpurun_out/stream_sweep.txt 2>&1
timeout 900 python bench.py --no-batch --no-pcg --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
