#!/bin/bash
mkdir -p gpurun_out
./tools/microbench/chain > gpurun_out/chain.txt 2>&1
./tools/gpu_hub10.sh
