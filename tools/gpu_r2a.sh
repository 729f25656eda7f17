mkdir -p gpurun_out
./tools/microbench/dadd > gpurun_out/dadd.txt 2>&1
timeout 900 python -m pytest tests/test_pcg_exact_gpu.py tests/test_errors_gpu.py tests/test_solve_gpu.py tests/test_fuzz_gpu.py -x -q > gpurun_out/pytest_r2a.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2a.log
for n in 32 64 128; do timeout 300 python tools/pcg_time.py --n $n --mode exact --reps 1 >> gpurun_out/pcg_exact.txt 2>&1; done
timeout 300 python tools/pcg_time.py --n 128 --reps 2 >> gpurun_out/pcg_exact.txt 2>&1
