#!/usr/bin/env python3
"""How early is each part of the factor final? For a streamed download the
columns below the lowest not-yet-eliminated position (the watermark) have
known output offsets. Prints, over the eliminate kernel's span, the share of
the factor's entries whose column is below the watermark.

  python tools/watermark.py [--n 128] [--workload poisson3d]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_02977_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--workload", default="poisson3d")
    args = ap.parse_args()
    if args.workload == "poisson3d":
        g = P.gen_poisson3d(args.n)
    elif args.workload == "poisson27":
        g = P.gen_poisson27(args.n, 1)
    else:
        g = P.gen_poisson2d(args.n)
    o = P.ordering_random(g.n, 0)
    ctx = P.GpuContext(0)
    opts = P.GpuOptions(record_times=True)
    st = P.FactorStats()
    for _ in range(2):
        f = P.factor_gpu(g, o, 0, opts, st, ctx=ctx)
    tt = ctx.vertex_times().astype(np.int64)
    t0 = tt[:, 0].min()
    end = (tt[:, 7] - t0) / 1e3
    span = float(end.max())
    wm = np.maximum.accumulate(end)          # column k final once all columns <= k are
    sizes = np.diff(f.col_ptr).astype(np.int64)
    cum = np.cumsum(sizes) / sizes.sum()
    out = {"n": g.n, "eliminate_ms": st.eliminate_ms, "span_us": span, "nnz": int(sizes.sum()), "curve": []}
    for frac in (0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 0.95, 0.99, 1.0):
        t = frac * span
        k = int(np.searchsorted(wm, t, side="right"))
        out["curve"].append({"t_frac": frac, "t_us": round(t, 1), "cols_final": k / g.n,
                             "nnz_final": float(cum[k - 1]) if k else 0.0})
    # end-time share of nnz per position decile
    dec = []
    for i in range(10):
        a, b = i * g.n // 10, (i + 1) * g.n // 10
        dec.append({"decile": i, "nnz_share": float(sizes[a:b].sum() / sizes.sum()),
                    "end_max_us": float(end[a:b].max()), "end_p50_us": float(np.median(end[a:b]))})
    out["deciles"] = dec
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
