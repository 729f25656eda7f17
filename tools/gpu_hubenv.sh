#!/bin/bash
# hub path A/B by environment (ENVS="A=1,B=2 C=3"): R-MAT 20 K3 time
mkdir -p gpurun_out
for e in ${ENVS:-NONE=0}; do
  echo "== $e $(env ${e//,/ } timeout 300 python tools/rmat_time.py --scale 20 --reps 2 2>&1 | tail -1 | cut -c1-60)" >> gpurun_out/hubenv.txt
done
