"""Long run of tests/test_fuzz_gpu.py's generator: python tools/fuzz_sweep.py START COUNT.
Prints one line per failing case and a summary (GPU; the oracle is the checker)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle  # noqa: E402
import paper_2505_02977_b200 as P  # noqa: E402
from corpus import factor_from_port  # noqa: E402
from test_fuzz_gpu import random_graph  # noqa: E402

start, count = int(sys.argv[1]), int(sys.argv[2])
port, ctx = oracle.Port(), P.GpuContext(0)
bad, t0 = 0, time.time()
for cs in range(start, start + count):
    rng = np.random.default_rng(1000 + cs)
    g, kind = random_graph(rng)
    seed = int(rng.integers(0, 1 << 31))
    perm = P.ordering_random(g.n, seed).perm if rng.random() < 0.7 else P.ordering_nnz_sort(g, seed).perm
    opts = dict(grid_ctas=int(rng.choice([0, 1, 7, 300])), verify=True)
    try:
        f = P.factor_gpu(g, P.Ordering(perm), seed, P.GpuOptions(**opts), ctx=ctx)
        ok = f.same_values(factor_from_port(port.factor(g, perm, seed)))
    except P.Error as e:
        ok = False
        print("error", cs, kind, g.n, e, flush=True)
    if not ok:
        bad += 1
        print("MISMATCH", cs, kind, g.n, opts, flush=True)
print(f"cases {count} mismatches {bad} seconds {time.time() - t0:.1f}")
