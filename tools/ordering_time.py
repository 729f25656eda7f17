#!/usr/bin/env python3
"""Wall time of ordering_nnz_sort: host restatement (std::sort, like the
reference) vs the device path (H2D of the row pointer + keys + radix sort +
D2H of perm), same perm. Prints one JSON line per graph."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2505_02977_b200 as P

ctx = P.GpuContext(0)
for name, build in (("poisson3d_128", lambda: P.gen_poisson3d(128)), ("rmat_20", lambda: P.gen_rmat(20, 16, 0))):
    g = build()
    P.ordering_nnz_sort_gpu(g, 0, ctx=ctx)  # warm-up
    t = time.perf_counter(); h = P.ordering_nnz_sort(g, 0).perm; th = time.perf_counter() - t
    ts = []
    for _ in range(5):
        t = time.perf_counter(); d = P.ordering_nnz_sort_gpu(g, 0, ctx=ctx).perm; ts.append(time.perf_counter() - t)
    print(json.dumps({"graph": name, "n": g.n, "host_ms": th * 1e3, "device_ms": min(ts) * 1e3,
                      "equal": bool(np.array_equal(h, d))}))
