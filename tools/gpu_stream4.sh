#!/bin/bash
mkdir -p gpurun_out
PARAC_STREAM=3 PARAC_STREAM_CTAS=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_assemble -c 1 -o gpurun_out/stream_full -f python tools/factor_time.py --reps 0 > gpurun_out/ncu_stream.log 2>&1
