#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_fuzz_gpu.py tests/test_hub_gpu.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for e in 1 0 1; do
  echo "== pipe=$e $(PARAC_HUB_PIPE=$e timeout 300 python tools/rmat_time.py --scale 20 --reps 2 2>&1 | tail -1 | cut -c1-110)" >> gpurun_out/variants.txt
done
timeout 300 python tools/hub_trace.py --scale 20 --json gpurun_out/hub_trace20.json > /dev/null 2>&1
