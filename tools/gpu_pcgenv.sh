#!/bin/bash
# PCG A/B by environment (ENVS): solve time and iterations at 128^3 (+ 27-point)
mkdir -p gpurun_out
for e in ${ENVS:-NONE=0}; do
  echo "== $e $(env ${e//,/ } timeout 300 python tools/pcg_time.py --reps 2 2>&1 | tail -1 | cut -c1-200)" >> gpurun_out/pcgenv.txt
done
