#!/bin/bash
# Full validation + evidence pass: GPU tests, smoke, default bench (with the
# CPU baseline and PCG), the reference arm, batch and other workloads, and the
# ncu launch list + full captures of the top kernels. Output in gpurun_out/.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --workload batch_64x64 > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err
timeout 600 python bench.py --workload poisson27_96 --no-cpu-baseline > gpurun_out/bench_27.json 2> gpurun_out/bench_27.err
timeout 600 python bench.py --workload poisson2d_256 --no-cpu-baseline > gpurun_out/bench_2d.json 2> gpurun_out/bench_2d.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python tools/ncu_factor.py --pcg > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eliminate_kernel -c 1 -o gpurun_out/k3_full -f python tools/ncu_factor.py > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"head_sweep|tw_gemv|wide_level" -s 20 -c 6 -o gpurun_out/sweeps_full -f python tools/ncu_factor.py --pcg > gpurun_out/ncu_sweeps.log 2>&1
timeout 300 python tools/sweep_profile.py > gpurun_out/sweep_profile.txt 2>&1
timeout 300 python tools/profile_factor.py --n 128 --json gpurun_out/prof128.json > gpurun_out/prof128.txt 2>&1
