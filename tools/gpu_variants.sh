#!/bin/bash
# A/B of prebuilt library variants (lib/variants/<X>/libparac_gpu.so): K3 time on
# the mesh workloads and R-MAT 20. Restores the main library at the end.
mkdir -p gpurun_out
L=paper_2505_02977_b200/lib
cp $L/libparac_gpu.so /tmp/main.so
for X in ${VARIANTS:-A B C}; do
  cp $L/variants/$X/libparac_gpu.so $L/libparac_gpu.so
  for w in poisson3d_128 poisson27_96; do
    echo "== $X $w $(timeout 300 python tools/k3_time.py --workload $w --reps 5 2>&1 | tail -1)" >> gpurun_out/variants.txt
  done
  echo "== $X rmat20 $(timeout 300 python tools/rmat_time.py --scale 20 --reps 3 2>&1 | tail -1)" >> gpurun_out/variants.txt
done
cp /tmp/main.so $L/libparac_gpu.so
