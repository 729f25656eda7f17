#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for sc in 48 64 80 96; do PARAC_SMALL_CAP=$sc timeout 300 python tools/factor_time.py >> gpurun_out/k3sweep.txt 2>&1; done
for cs in 64,512,4096 128,1024,4096 256,2048,8192 128,1024,2048; do PARAC_CLAIM_SLEEP=$cs timeout 300 python tools/factor_time.py >> gpurun_out/k3sweep.txt 2>&1; done
for hw in 1024 4096; do PARAC_HUB_WAIT_NS=$hw timeout 300 python tools/factor_time.py >> gpurun_out/k3sweep.txt 2>&1; done
done
