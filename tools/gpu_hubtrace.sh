#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_factor_gpu.py -x -q -k "rmat or hub or trace" > gpurun_out/pytest_hubt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_hubt.log
timeout 300 python tools/hub_trace.py --scale 20 --json gpurun_out/hub_trace20.json > gpurun_out/hub_trace20.txt 2>&1
