#!/bin/bash
# Hub-path iteration: factor parity tests (R-MAT wide columns, traces), R-MAT
# 20/22 timing + critical-path profile, 128^3 / 27-point K3 timing (no regression).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_factor_gpu.py -x -q > gpurun_out/pytest_hub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_hub.log
timeout 300 python tools/profile_factor.py --workload rmat --n 20 --json gpurun_out/prof_rmat20.json > gpurun_out/prof_rmat20.txt 2>&1
for w in ${WLS:-poisson3d_128 poisson27_96}; do
  echo "== $w $(timeout 300 python tools/k3_time.py --workload $w --reps 5 2>&1 | tail -1)" >> gpurun_out/k3hub.txt
done
timeout 600 python bench.py --workload rmat_22 --no-cpu-baseline --no-pcg --no-dropin --no-batch --steps 2 --warmup 3 > gpurun_out/bench_rmat.json 2> gpurun_out/bench_rmat.err
timeout 900 python -m pytest tests/test_fullsize_gpu.py tests/test_hub_gpu.py tests/test_fuzz_gpu.py -x -q > gpurun_out/pytest_hub2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_hub2.log
