#!/bin/bash
mkdir -p gpurun_out
for e in PARAC_KEEP_LIMIT=1 PARAC_KEEP_LIMIT=2 PARAC_KEEP_DELAY_US=100000 PARAC_KEEP_DELAY_US=5000; do
  for w in poisson27_96 poisson3d_128 poisson2d_256; do
    echo "== $e $w $(env $e timeout 300 python tools/k3_time.py --workload $w --reps 2 2>&1 | tail -1 | cut -c1-160)" >> gpurun_out/repro.txt
  done
done
