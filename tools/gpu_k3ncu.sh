#!/bin/bash
# K3 A/B timing per env (ENVS) + one ncu --set full capture of K3 (default env)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_fullsize_gpu.py tests/test_fuzz_gpu.py -x -q > gpurun_out/pytest_k3env.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k3env.log
for e in ${ENVS:-NONE=0}; do
  for w in ${WLS:-poisson3d_128 poisson27_96 poisson2d_256}; do
    echo "== $e $(env ${e//,/ } timeout 300 python tools/k3_time.py --workload $w --reps 5 2>&1 | tail -1)" >> gpurun_out/k3env.txt
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eliminate_kernel -c 1 -o gpurun_out/k3_full -f python tools/ncu_factor.py > gpurun_out/ncu_full.log 2>&1
