#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do for c in 256 384 512 1024; do timeout 300 python tools/factor_time.py --c0 $c >> gpurun_out/c0.txt 2>&1; done; done
for c in 256 512; do timeout 300 python tools/factor_time.py --c0 $c --workload poisson27 --n 96 >> gpurun_out/c0.txt 2>&1; timeout 300 python tools/factor_time.py --c0 $c --workload poisson2d --n 256 >> gpurun_out/c0.txt 2>&1; done
