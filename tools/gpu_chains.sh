#!/bin/bash
mkdir -p gpurun_out
./tools/microbench/chains_iso > gpurun_out/chains_iso.txt 2>&1
./tools/microbench/chains_iso64 > gpurun_out/chains_iso64.txt 2>&1
