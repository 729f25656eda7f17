#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 300 python - > gpurun_out/pyfactor.txt 2>&1 <<'PY'
import time, paper_2505_02977_b200 as P
g = P.gen_poisson3d(128); o = P.ordering_random(g.n, 0); ctx = P.GpuContext(0)
for i in range(4):
    t = time.perf_counter(); f = P.factor_gpu(g, o, 0, ctx=ctx); print("factor_gpu s", time.perf_counter() - t, f"{f.checksum():016x}")
PY
