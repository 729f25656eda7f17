#!/bin/bash
# Streamed assembly evidence: compute-sanitizer over the sanitizer workload, fuzz sweeps through the streamed path.
mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 --launch-timeout 0 python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$t.log
done
timeout 1500 python tools/fuzz_sweep.py 0 3000 > gpurun_out/fuzz_sweep_0_3000.log 2>&1
timeout 900 python tools/fuzz_sweep.py 0 400 --batch > gpurun_out/fuzz_batch_0_400.log 2>&1
timeout 900 python tools/fuzz_sweep.py 0 300 --rmat > gpurun_out/fuzz_rmat_0_300.log 2>&1
