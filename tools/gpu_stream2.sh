#!/bin/bash
# Streamed assembly: streamer CTA count sweep (device + K3 time), on/off A/B on the other configs.
mkdir -p gpurun_out
for rep in 1 2; do
for c in 2 4 8 16; do PARAC_STREAM_CTAS=$c timeout 300 python tools/factor_time.py >> gpurun_out/stream_sweep.txt 2>&1; done
PARAC_STREAM=0 timeout 300 python tools/factor_time.py >> gpurun_out/stream_sweep.txt 2>&1
done
for s in 1 0; do
  PARAC_STREAM=$s timeout 300 python tools/factor_time.py --workload poisson27 --n 96 >> gpurun_out/stream_sweep.txt 2>&1
  PARAC_STREAM=$s timeout 300 python tools/factor_time.py --workload poisson2d --n 256 >> gpurun_out/stream_sweep.txt 2>&1
  PARAC_STREAM=$s timeout 300 python tools/factor_time.py --workload rmat --n 20 --reps 3 >> gpurun_out/stream_sweep.txt 2>&1
done
