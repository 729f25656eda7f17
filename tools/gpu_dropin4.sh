#!/bin/bash
mkdir -p gpurun_out
for i in 1 2 3; do PARAC_SHIM_TIMING=1 timeout 300 ./tools/_build/dropin_time 128 5 2 >> gpurun_out/dropin.txt 2>&1; done
timeout 900 python bench.py --no-batch --no-cpu-baseline --no-pcg > gpurun_out/bench.json 2> gpurun_out/bench.err
