#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for c in 2 8; do PARAC_STREAM_CTAS=$c timeout 300 python tools/factor_time.py >> gpurun_out/stream_sweep.txt 2>&1; done
PARAC_STREAM=0 timeout 300 python tools/factor_time.py >> gpurun_out/stream_sweep.txt 2>&1
PARAC_STREAM=0 timeout 300 python tools/factor_time.py --grid 584 >> gpurun_out/stream_sweep.txt 2>&1
PARAC_STREAM=2 timeout 300 python tools/factor_time.py --grid 584 >> gpurun_out/stream_sweep.txt 2>&1
done
