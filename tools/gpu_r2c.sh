#!/bin/bash
# Round 2 (c): new GPU tests (multi-rank batch on one device, on_phase trace,
# CLI metrics), K3 building-block microbench, fill-slot sweep, critical-path
# profile, and the default bench with the batch sub-record.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multirank_gpu.py tests/test_factor_gpu.py tests/test_cli_gpu.py -x -q > gpurun_out/pytest_r2c.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2c.log
./tools/microbench/k3parts > gpurun_out/k3parts.txt 2>&1
timeout 300 python tools/k3_time.py --c0 0,32,64,128,256 > gpurun_out/k3_c0.txt 2>&1
timeout 300 python tools/profile_factor.py --n 128 --json gpurun_out/prof128.json > gpurun_out/prof128.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err
