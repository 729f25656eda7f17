#!/bin/bash
mkdir -p gpurun_out
./tools/microbench/tailbench > gpurun_out/tailbench.txt 2>&1
timeout 300 python tools/profile_factor.py --n 128 --json gpurun_out/prof128.json > gpurun_out/prof128.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:eliminate_kernel -c 1 -o gpurun_out/k3_full2 -f python tools/ncu_factor.py > gpurun_out/ncu_k3.log 2>&1
