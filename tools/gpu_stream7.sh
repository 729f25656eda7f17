#!/bin/bash
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
for s in 1 0; do
PARAC_STREAM=$s PARAC_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --workload batch_64x64 > gpurun_out/b2_s$s.out 2> gpurun_out/b2_s$s.err
done
for c in 8 16 32 64; do PARAC_STREAM_CTAS=$c timeout 900 python bench.py --workload batch_64x64 --no-cpu-baseline > gpurun_out/bench_batch_c$c.json 2> gpurun_out/bench_batch_c$c.err; done
