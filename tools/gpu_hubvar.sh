#!/bin/bash
# A/B of prebuilt hub-path library variants on R-MAT 20 (VARIANTS)
mkdir -p gpurun_out
L=paper_2505_02977_b200/lib
cp $L/libparac_gpu.so /tmp/main.so
for X in ${VARIANTS:-S8 S16 S8 S16}; do
  cp $L/variants/$X/libparac_gpu.so $L/libparac_gpu.so
  echo "== $X rmat20 $(timeout 300 python tools/rmat_time.py --scale 20 --reps 2 2>&1 | tail -1 | cut -c1-70)" >> gpurun_out/hubvar.txt
done
cp /tmp/main.so $L/libparac_gpu.so
