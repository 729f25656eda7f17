#!/bin/bash
# Round-2 fuzz sweeps over the hub path: random graphs (hubs included), batches, R-MAT
mkdir -p gpurun_out/fuzz_r02
timeout 1500 python tools/fuzz_sweep.py 0 3000 > gpurun_out/fuzz_r02/fuzz_sweep_0_3000.log 2>&1
timeout 900 python tools/fuzz_sweep.py 0 400 --batch > gpurun_out/fuzz_r02/fuzz_batch_0_400.log 2>&1
timeout 1500 python tools/fuzz_sweep.py 0 300 --rmat > gpurun_out/fuzz_r02/fuzz_rmat_0_300.log 2>&1
