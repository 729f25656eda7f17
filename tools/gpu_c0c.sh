#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/batch_time.py >> gpurun_out/c0_batch.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --workload batch_64x64 > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err
timeout 900 python bench.py --workload rmat_22 --no-pcg --no-dropin --no-batch --steps 2 --warmup 3 > gpurun_out/bench_rmat.json 2> gpurun_out/bench_rmat.err
