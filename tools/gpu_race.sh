#!/bin/bash
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 --launch-timeout 0 python tools/sanitize_run.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
timeout 900 python -m pytest tests/test_factor_gpu.py -x -q > gpurun_out/pytest_factor.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_factor.log
