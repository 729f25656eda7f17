#!/bin/bash
mkdir -p gpurun_out
for r in 0 1 0 1; do
  echo "== register=$r" >> gpurun_out/dropin_reg.txt
  PARAC_SHIM_TIMING=1 PARAC_STAGE_REGISTER=$r ./tools/_build/dropin_time 128 4 2 2>&1 | tail -3 >> gpurun_out/dropin_reg.txt
done
cat /sys/kernel/mm/transparent_hugepage/enabled >> gpurun_out/dropin_reg.txt 2>&1
