#!/bin/bash
mkdir -p gpurun_out
for w in poisson3d_128 poisson2d_256; do
  for e in "NONE=0" "PARAC_KEEP=width" "PARAC_KEEP_LIMIT=8" "PARAC_KEEP_LIMIT=64" "PARAC_CLAIM_SLEEP=96,768,3072"; do
    echo "== $w $e" >> gpurun_out/k3sweep.txt
    env $e timeout 300 python bench.py --workload $w --no-cpu-baseline --no-pcg --steps 6 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" >> gpurun_out/k3sweep.txt
  done
done
