mkdir -p gpurun_out
timeout 300 python tools/profile_factor.py --n 128 --json gpurun_out/prof128.json > gpurun_out/prof128.log 2>&1
for w in poisson2d_256 poisson27_96; do
timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 900 python bench.py --workload rmat_22 --no-cpu-baseline --no-pcg --steps 3 > gpurun_out/bench_rmat_22.json 2> gpurun_out/bench_rmat_22.err
echo done
