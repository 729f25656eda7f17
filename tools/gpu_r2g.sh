#!/bin/bash
# Round-2 final evidence (streamed assembly build): GPU tests, smoke, default bench (+ reference arm),
# the other configs, R-MAT 22 + hub trace, launch list, K3 ncu capture, K3 timeline.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --workload batch_64x64 > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err
timeout 600 python bench.py --workload poisson27_96 > gpurun_out/bench_27.json 2> gpurun_out/bench_27.err
timeout 600 python bench.py --workload poisson2d_256 > gpurun_out/bench_2d.json 2> gpurun_out/bench_2d.err
timeout 900 python bench.py --workload rmat_22 --no-pcg --no-dropin --no-batch --steps 2 --warmup 3 > gpurun_out/bench_rmat.json 2> gpurun_out/bench_rmat.err
timeout 300 python tools/hub_trace.py --scale 22 --json gpurun_out/hub_trace22.json > /dev/null 2>&1
PARAC_STREAM=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python tools/ncu_factor.py --pcg > gpurun_out/ncu_launch.log 2>&1
PARAC_STREAM=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:eliminate_kernel -c 1 -o gpurun_out/k3_full -f python tools/ncu_factor.py > gpurun_out/ncu_full.log 2>&1
timeout 300 python tools/profile_factor.py --n 128 --json gpurun_out/prof128.json > gpurun_out/prof128.txt 2>&1
PARAC_STREAM=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_assemble -c 1 -o gpurun_out/stream_full -f python tools/ncu_factor.py > gpurun_out/ncu_stream.log 2>&1
timeout 300 python tools/watermark.py --n 128 > gpurun_out/watermark128.json 2>&1
