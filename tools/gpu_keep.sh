#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for k in low high width; do PARAC_KEEP=$k timeout 300 python tools/factor_time.py >> gpurun_out/keep.txt 2>&1; done
done
for k in low high; do PARAC_KEEP=$k timeout 300 python tools/factor_time.py --workload poisson27 --n 96 >> gpurun_out/keep.txt 2>&1; PARAC_KEEP=$k timeout 300 python tools/factor_time.py --workload poisson2d --n 256 >> gpurun_out/keep.txt 2>&1; done
