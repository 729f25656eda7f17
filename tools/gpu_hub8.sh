#!/bin/bash
mkdir -p gpurun_out
./tools/microbench/chains_iso > gpurun_out/chains_iso.txt 2>&1
timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_fuzz_gpu.py tests/test_fullsize_gpu.py -x -q -k "rmat or hub or trace or fuzz or batch" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for w in poisson3d_128; do
  echo "== $w $(timeout 300 python tools/k3_time.py --workload $w --reps 5 2>&1 | tail -1)" >> gpurun_out/variants.txt
done
echo "== rmat20 $(timeout 300 python tools/rmat_time.py --scale 20 --reps 3 2>&1 | tail -1)" >> gpurun_out/variants.txt
timeout 300 python tools/hub_trace.py --scale 20 --json gpurun_out/hub_trace20.json > /dev/null 2>&1
