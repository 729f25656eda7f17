#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_fuzz_gpu.py -x -q -k "rmat or hub or trace or fuzz" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
echo "== mode1 rmat20 $(timeout 300 python tools/rmat_time.py --scale 20 --reps 2 2>&1 | tail -1)" >> gpurun_out/variants.txt
echo "== mode0 rmat20 $(PARAC_HUB_MODE=0 timeout 300 python tools/rmat_time.py --scale 20 --reps 2 2>&1 | tail -1)" >> gpurun_out/variants.txt
timeout 300 python tools/hub_trace.py --scale 20 --json gpurun_out/hub_trace20.json > /dev/null 2>&1
