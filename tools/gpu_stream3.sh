#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for f in 0 0.5 0.8 0.9 0.95; do PARAC_STREAM_START=$f timeout 300 python tools/factor_time.py >> gpurun_out/stream_sweep.txt 2>&1; done
PARAC_STREAM=0 timeout 300 python tools/factor_time.py >> gpurun_out/stream_sweep.txt 2>&1
done
for f in 0 0.9; do PARAC_STREAM_START=$f timeout 300 python tools/factor_time.py --workload poisson27 --n 96 >> gpurun_out/stream_sweep.txt 2>&1; done
