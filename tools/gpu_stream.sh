#!/bin/bash
# Streamed assembly + download: tests, then A/B (PARAC_STREAM=1/0) on the default bench and the drop-in call.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_stream_gpu.py tests/test_factor_gpu.py -x -q > gpurun_out/pytest_stream.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stream.log
for s in 1 0 1 0; do
  PARAC_STREAM=$s timeout 600 python bench.py --no-pcg --no-batch --no-cpu-baseline > gpurun_out/bench_s$s.json 2>> gpurun_out/bench_s.err
  cat gpurun_out/bench_s$s.json >> gpurun_out/bench_s_all.txt
  echo "== PARAC_STREAM=$s" >> gpurun_out/dropin_s.txt
  PARAC_STREAM=$s PARAC_SHIM_TIMING=1 timeout 300 ./tools/_build/dropin_time 128 4 2 >> gpurun_out/dropin_s.txt 2>&1
done
