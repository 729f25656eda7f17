#!/bin/bash
# Drop-in call timing breakdown per staging setting (PARAC_STAGE_THREADS, PARAC_STAGE_CHUNK_MB)
mkdir -p gpurun_out
nproc > gpurun_out/dropin_sweep.txt
for t in 8 12 16; do for c in 8 32; do
  echo "== threads=$t chunk=$c" >> gpurun_out/dropin_sweep.txt
  PARAC_SHIM_TIMING=1 PARAC_STAGE_THREADS=$t PARAC_STAGE_CHUNK_MB=$c ./tools/_build/dropin_time 128 4 2 2>&1 | tail -3 >> gpurun_out/dropin_sweep.txt
done; done
