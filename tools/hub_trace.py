#!/usr/bin/env python3
"""Per-phase timing of the cooperative hub path (record_times run): for every
wide column (raw > 1024) the owner's post time, the first chunk start, the
last chunk end and who ran the chunks, per phase; printed as means over the
columns (all, and the widest quartile).

  python tools/hub_trace.py [--scale 20] [--json out.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_02977_b200 as P  # noqa: E402

WORDS = 64
STEPS = ["gather+tile", "cross rank", "merge", "weight tiles", "weight rank", "sample+column", "release",
         "lkk chain", "suffix chain"]
# each phase is posted by the CTA that completed the previous one's last chunk
# (the owner posts gather and sample): span = post -> last chunk end


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--star", type=int, default=0, help="a star with this many leaves instead (one hub column)")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    if args.star:  # centre 0 eliminated first, every leaf waits on it
        n = args.star + 1
        g = P.LaplacianGraph.from_edges(n, [(0, v, 1.0 + (v % 7) * 0.25) for v in range(1, n)])
    else:
        g = P.gen_rmat(args.scale, 16, 0)
    o = P.Ordering.identity(g.n) if args.star else P.ordering_random(g.n, 0)
    ctx = P.GpuContext(0)
    st = P.FactorStats()
    for _ in range(2):
        P.factor_gpu(g, o, 0, P.GpuOptions(record_times=True), st, ctx=ctx)
    lib = P.rchol.lib
    cnt = np.zeros(1, np.int32)
    P.rchol._check(lib.parac_gpu_download_hub_trace(ctx.handle, None, 0, cnt.ctypes.data))
    n = int(cnt[0])
    rec = np.zeros(n * WORDS, np.uint64)
    P.rchol._check(lib.parac_gpu_download_hub_trace(ctx.handle, rec.ctypes.data, n, cnt.ctypes.data))
    rec = rec.reshape(n, WORDS).astype(np.float64)
    R = rec[:, 1]
    m = rec[:, 2]
    total = (rec[:, 4] - rec[:, 3]) / 1e3
    out = {"scale": args.scale, "eliminate_ms": st.eliminate_ms, "wide_columns": n}

    def summarise(sel):
        d = {"count": int(sel.sum()), "R_mean": float(R[sel].mean()), "m_mean": float(m[sel].mean()),
             "total_us": float(total[sel].mean()), "steps": {}}
        for p, name in enumerate(STEPS, start=1):
            b = 8 + 4 * (p - 1)
            post, first, last, ch = rec[sel, b], rec[sel, b + 1], rec[sel, b + 2], rec[sel, b + 3].astype(np.uint64)
            ok = post > 0
            if not ok.any():
                continue
            e = {"span_us": float(((last - post)[ok]).mean() / 1e3)}
            if p >= 8:  # chain thread: cycles in the chain << 32 | cycles at its group barrier
                e["chain_busy_cycles"] = float((ch[ok] >> np.uint64(32)).astype(np.float64).mean())
                e["barrier_wait_cycles"] = float((ch[ok] & np.uint64(0xffffffff)).astype(np.float64).mean())
                per = (ch[ok] >> np.uint64(32)).astype(np.float64) / np.maximum(m[sel][ok], 1)
                e["cycles_per_element_p10_p50_p90"] = [float(np.percentile(per, q)) for q in (10, 50, 90)]
            if p <= 7:
                okf = ok & (first < 2 ** 63)
                e["join_us"] = float(((first - post)[okf]).mean() / 1e3) if okf.any() else None
                e["owner_chunks"] = float((ch[ok] >> np.uint64(32)).astype(np.float64).mean())
                e["helper_chunks"] = float((ch[ok] & np.uint64(0xffffffff)).astype(np.float64).mean())
                nchunks = (ch[ok] >> np.uint64(32)) + (ch[ok] & np.uint64(0xffffffff))
                e["chunk_us"] = float((rec[sel, 48 + p][ok] / np.maximum(nchunks.astype(np.float64), 1)).mean() / 1e3)
            d["steps"][name] = e
        # gaps: owner time between steps (post of p+1 - last end of p)
        return d

    out["all"] = summarise(np.ones(n, bool))
    q = np.quantile(R, 0.75) if n else 0
    out["widest_quartile"] = summarise(R >= q)
    print(json.dumps(out, indent=1))
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
