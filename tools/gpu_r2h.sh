#!/bin/bash
# Hand-written radix sort build: GPU tests, smoke, default bench, launch list,
# PCG setup (transpose + level order) and device nnz-sort timings.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/pcg_first_call.py > gpurun_out/pcg_first_call.txt 2>&1
timeout 300 python tools/ordering_time.py > gpurun_out/ordering_time.txt 2>&1
PARAC_STREAM=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python tools/ncu_factor.py --pcg > gpurun_out/ncu_launch.log 2>&1
