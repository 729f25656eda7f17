#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_factor_gpu.py -x -q > gpurun_out/pytest_hub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_hub.log
VARIANTS="A3 Q" ./tools/gpu_variants.sh
L=paper_2505_02977_b200/lib
for X in A3 Q; do
  cp $L/variants/$X/libparac_gpu.so $L/libparac_gpu.so
  timeout 300 python tools/hub_trace.py --scale 20 --json gpurun_out/hub_trace20_$X.json > /dev/null 2>&1
done
