#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --workload rmat_22 --no-pcg --no-dropin --no-batch --steps 2 --warmup 3 > gpurun_out/bench_rmat.json 2> gpurun_out/bench_rmat.err
timeout 600 python bench.py --workload poisson27_96 > gpurun_out/bench_27.json 2> gpurun_out/bench_27.err
timeout 600 python bench.py --workload poisson2d_256 > gpurun_out/bench_2d.json 2> gpurun_out/bench_2d.err
