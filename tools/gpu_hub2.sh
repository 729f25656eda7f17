#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_factor_gpu.py -x -q > gpurun_out/pytest_hub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_hub.log
VARIANTS="A B C" ./tools/gpu_variants.sh
timeout 300 python tools/hub_trace.py --scale 20 --json gpurun_out/hub_trace20.json > gpurun_out/hub_trace20.txt 2>&1
