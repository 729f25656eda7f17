#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_factor_gpu.py -x -q > gpurun_out/pytest_hub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_hub.log
for w in poisson3d_128 poisson27_96; do
  echo "== $w $(timeout 300 python tools/k3_time.py --workload $w --reps 5 2>&1 | tail -1)" >> gpurun_out/variants.txt
done
echo "== rmat20 $(timeout 300 python tools/rmat_time.py --scale 20 --reps 3 2>&1 | tail -1)" >> gpurun_out/variants.txt
timeout 300 python tools/hub_trace.py --scale 20 --json gpurun_out/hub_trace20.json > /dev/null 2>&1
