#!/bin/bash
# Final round-2 validation of the radix sort build: GPU tests, smoke, default bench + reference arm,
# racecheck / memcheck of the radix sort kernels through the ordering tests.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_ordering_gpu.py -q -k "random_connected_ragged or rmat_16 or tiny" > gpurun_out/racecheck_sort.log 2>&1; echo "rc=$?" >> gpurun_out/racecheck_sort.log
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_ordering_gpu.py -q -k "random_connected_ragged or rmat_16 or tiny" > gpurun_out/memcheck_sort.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck_sort.log
