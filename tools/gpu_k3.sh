#!/bin/bash
# K3 iteration: factor parity tests, K3 timing per env setting, critical-path profile
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_factor_gpu.py tests/test_fullsize_gpu.py tests/test_fuzz_gpu.py -x -q > gpurun_out/pytest_k3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k3.log
for e in ${K3_ENVS:-NONE=0}; do
  for w in poisson3d_128 poisson27_96 poisson2d_256; do
    echo "== $e $w $(env ${e//,/ } timeout 300 python bench.py --workload $w --no-cpu-baseline --no-pcg --no-dropin --steps 5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["factor_ms"]["eliminate_k3"],3), d["e2e"]["ms_per_step"])')" >> gpurun_out/k3.txt
  done
done
[ -n "$K3_PROF" ] && timeout 300 python tools/profile_factor.py --n 128 --json gpurun_out/prof128.json > /dev/null 2> gpurun_out/prof.err
true
