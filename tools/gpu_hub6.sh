#!/bin/bash
mkdir -p gpurun_out
L=paper_2505_02977_b200/lib
cp $L/libparac_gpu.so /tmp/main.so
./tools/microbench/chain > gpurun_out/chain.txt 2>&1
timeout 600 python -m pytest tests/test_factor_gpu.py -x -q > gpurun_out/pytest_hub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_hub.log
for X in C N1 N2 C N1 N2; do
  cp $L/variants/$X/libparac_gpu.so $L/libparac_gpu.so
  echo "== $X 128 $(timeout 300 python tools/k3_time.py --workload poisson3d_128 --reps 5 2>&1 | tail -1)" >> gpurun_out/variants.txt
done
for X in C N1; do
  cp $L/variants/$X/libparac_gpu.so $L/libparac_gpu.so
  echo "== $X 27 $(timeout 300 python tools/k3_time.py --workload poisson27_96 --reps 5 2>&1 | tail -1)" >> gpurun_out/variants.txt
done
cp /tmp/main.so $L/libparac_gpu.so
echo "== main rmat20 $(timeout 300 python tools/rmat_time.py --scale 20 --reps 3 2>&1 | tail -1)" >> gpurun_out/variants.txt
