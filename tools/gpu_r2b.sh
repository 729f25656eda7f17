#!/bin/bash
# PCG dense-tail iteration: solve tests, timing per PARAC_TAIL_ROWS, verbose setup stages, sweep profile
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_solve_gpu.py tests/test_pcg_exact_gpu.py tests/test_hub_gpu.py tests/test_fullsize_gpu.py -x -q > gpurun_out/pytest_r2b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2b.log
for t in ${TAILS:-auto}; do
  if [ "$t" = auto ]; then unset PARAC_TAIL_ROWS; else export PARAC_TAIL_ROWS=$t; fi
  PARAC_VERBOSE=1 timeout 300 python tools/pcg_time.py --reps 2 >> gpurun_out/pcg_r2b.txt 2>&1
done
unset PARAC_TAIL_ROWS
timeout 300 python tools/pcg_time.py --workload poisson27 --n 96 --reps 2 >> gpurun_out/pcg_r2b.txt 2>&1
timeout 300 python tools/pcg_time.py --workload poisson2d --n 256 --reps 2 >> gpurun_out/pcg_r2b.txt 2>&1
timeout 300 python tools/sweep_profile.py > gpurun_out/sweep_profile_r2b.txt 2>&1
