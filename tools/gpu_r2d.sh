#!/bin/bash
# Re-entry validation: GPU tests, smoke, default bench, R-MAT 22 device time.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --workload rmat_22 --no-cpu-baseline --no-pcg --no-dropin --no-batch --steps 1 --warmup 1 > gpurun_out/bench_rmat.json 2> gpurun_out/bench_rmat.err
timeout 300 python tools/profile_factor.py --workload rmat --n 20 --json gpurun_out/prof_rmat20.json > gpurun_out/prof_rmat20.txt 2>&1
