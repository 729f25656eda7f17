#!/bin/bash
# K3 claim back-off tiers on several workloads (device factor ms)
mkdir -p gpurun_out
for w in poisson27_96 batch_64x64 poisson2d_256; do
  for e in "NONE=0" "PARAC_CLAIM_SLEEP=128,1024,4096"; do
    echo "== $w $e" >> gpurun_out/k3sweep.txt
    env $e timeout 300 python bench.py --workload $w --no-cpu-baseline --no-pcg --steps 6 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" >> gpurun_out/k3sweep.txt
  done
done
