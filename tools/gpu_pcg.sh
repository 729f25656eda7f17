#!/bin/bash
# PCG iteration script: solve tests + device timing per env setting + per-level sweep profile
# PCG_ENVS="A=1,B=2 C=3" runs pcg_time once per space-separated setting (comma = several vars)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_solve_gpu.py tests/test_fullsize_gpu.py -x -q -k "not batch" > gpurun_out/pytest_pcg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pcg.log
for e in ${PCG_ENVS:-NONE=0}; do
  echo "== $e" >> gpurun_out/pcg_time.txt
  env ${e//,/ } timeout 300 python tools/pcg_time.py --reps 2 >> gpurun_out/pcg_time.txt 2>&1
  env ${e//,/ } timeout 300 python tools/pcg_time.py --workload poisson27 --n 96 --reps 2 >> gpurun_out/pcg_time.txt 2>&1
  env ${e//,/ } timeout 300 python tools/pcg_time.py --workload poisson2d --n 256 --reps 2 >> gpurun_out/pcg_time.txt 2>&1
done
for e in ${PCG_ENVS:-NONE=0}; do echo "== $e" >> gpurun_out/sweep_profile.txt; env ${e//,/ } timeout 300 python tools/sweep_profile.py >> gpurun_out/sweep_profile.txt 2>&1; done
[ -n "$PCG_NCU" ] && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pcg_launches.csv \
  python tools/pcg_time.py --reps 1 > /dev/null 2>&1
true
