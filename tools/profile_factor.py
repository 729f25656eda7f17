#!/usr/bin/env python3
"""Timeline analysis of one factorization (record_times): where does the
eliminate kernel's time go? Prints the elimination-rate profile, per-vertex
service time vs column size, and the realised critical path split into
service time (inside eliminate_vertex) and hand-off latency (ready -> claimed).

  python tools/profile_factor.py [--n 128] [--workload poisson3d] [--json out.json]
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
    ap.add_argument("--json", default=None)
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--c0", type=int, default=0, help="preallocated fill slots per vertex (0: library default)")
    args = ap.parse_args()
    if args.workload == "poisson3d":
        g = P.gen_poisson3d(args.n)
    elif args.workload == "poisson27":
        g = P.gen_poisson27(args.n, 1)
    elif args.workload == "poisson2d":
        g = P.gen_poisson2d(args.n)
    else:
        g = P.gen_rmat(args.n, 16, 0)
    o = P.ordering_random(g.n, 0)
    ctx = P.GpuContext(0)
    opts = P.GpuOptions(record_times=True, grid_ctas=args.grid, first_chunk=args.c0)
    st = P.FactorStats()
    for _ in range(2):
        f = P.factor_gpu(g, o, 0, opts, st, ctx=ctx)
    tt = ctx.vertex_times().astype(np.int64)
    sub_all = np.zeros(12 * g.n, np.uint64)
    P.rchol._check(P.rchol.lib.parac_gpu_download_subtimes(ctx.handle, sub_all.ctypes.data))
    sub = sub_all[:8 * g.n].reshape(g.n, 8).astype(np.int64)
    cyc = sub_all[8 * g.n:].reshape(g.n, 4).astype(np.int64)
    n = g.n
    t0 = tt[:, 0].min()
    start = (tt[:, 0] - t0) / 1e3  # us
    end = (tt[:, 7] - t0) / 1e3
    dur = end - start
    # per-phase durations (a skipped phase inherits the previous timestamp)
    ph = tt.copy()
    for i in range(1, 8):
        ph[:, i] = np.where(ph[:, i] == 0, ph[:, i - 1], ph[:, i])
    pdur = np.diff(ph, axis=1) / 1e3
    names = ["gather+sort", "merge", "lkk+column", "wsort+suffix", "sample+emit", "fence+decrement",
             "ready+publish"]
    raw = g_fdeg = None
    m = st.merged_degree
    fills = st.fills_received
    # forward degree per position
    pos = o.perm
    src = np.repeat(np.arange(n), np.diff(g.ptr))
    fwd = np.zeros(n, np.int64)
    np.add.at(fwd, pos[src][pos[g.adj] > pos[src]], 1)
    raw = fwd + fills
    # ready time: last decrement = end of the latest column containing k
    ready = np.full(n, -1.0)
    cols = np.repeat(np.arange(n), np.diff(f.col_ptr))
    np.maximum.at(ready, f.rows, end[cols])
    hop = np.where(ready >= 0, start - np.maximum(ready, 0), start)
    total = end.max()
    out = {"n": n, "eliminate_ms": st.eliminate_ms, "span_us": float(total),
           "service_us_mean": float(dur.mean()), "hop_us_median": float(np.median(hop[ready >= 0]))}
    # rate profile
    edges = np.linspace(0, total, 21)
    hist, _ = np.histogram(end, bins=edges)
    out["completions_per_5pct"] = hist.tolist()
    # service time by raw size
    bins = [0, 8, 16, 32, 64, 128, 256, 1024, 1 << 30]
    by = []
    for lo, hi in zip(bins[:-1], bins[1:]):
        sel = (raw >= lo) & (raw < hi)
        if sel.any():
            by.append({"raw": f"[{lo},{hi})", "count": int(sel.sum()),
                       "service_us_mean": float(dur[sel].mean()),
                       "service_us_p99": float(np.percentile(dur[sel], 99)),
                       "phases_us": {nm: round(float(pdur[sel, i].mean()), 2)
                                     for i, nm in enumerate(names)}})
    out["service_by_raw"] = by
    # realised critical path: walk back from the last finisher via its latest dep
    parent_of = np.full(n, -1, np.int64)
    best = np.full(n, -1.0)
    order = np.argsort(cols, kind="stable")
    # latest-finishing dependency per row
    for_rows = f.rows
    e_cols = end[cols]
    idx = np.lexsort((e_cols, for_rows))
    last = np.ones(len(idx), bool)
    last[:-1] = for_rows[idx][1:] != for_rows[idx][:-1]
    sel = idx[last]
    parent_of[for_rows[sel]] = cols[sel]
    k = int(np.argmax(end))
    chain = []
    while k >= 0:
        chain.append(k)
        k = int(parent_of[k])
    chain = chain[::-1]
    ch = np.array(chain)
    out["critical_path"] = {
        "length": len(chain), "service_us": float(dur[ch].sum()), "hop_us": float(hop[ch].sum()),
        "initial_wait_us": float(start[ch[0]]), "raw_mean": float(raw[ch].mean()),
        "m_mean": float(m[ch].mean()), "service_us_per_vertex": float(dur[ch].mean()),
        "hop_us_per_vertex": float(hop[ch[1:]].mean()) if len(ch) > 1 else 0.0,
        "phases_us_per_vertex": {nm: round(float(pdur[ch, i].mean()), 2) for i, nm in enumerate(names)},
    }
    # sub-phase split of the critical path (where stamped)
    def span(a, b):
        ok = (a > 0) & (b > 0)
        return float(((b - a)[ok] / 1e3).mean()) if ok.any() else None
    chs = ch
    out["critical_path"]["sub_us"] = {
        "setup(claim->counts+dir)": span(tt[chs, 0], sub[chs, 0]),
        "gather landed": span(sub[chs, 0], sub[chs, 1]),
        "raw sort": span(sub[chs, 1], tt[chs, 1]),
        "weight sort": span(tt[chs, 3], sub[chs, 2]),
        "suffix chain": span(sub[chs, 2], tt[chs, 4]),
        "draw samples": span(tt[chs, 4], sub[chs, 3]),
        "emit fills": span(sub[chs, 3], sub[chs, 4]),
        "levels+fence": span(sub[chs, 4], sub[chs, 5]),
        "decrement": span(sub[chs, 5], tt[chs, 6]),
    }
    # hand-off analysis along the critical path: kept (same warp/CTA continued)
    # vs claimed from a ready queue; small (warp) vs big (CTA) eliminator
    kept = sub[chs, 7] == 1
    bigc = (sub[chs, 6] & 0xff) == 0xff
    hops = hop[chs]
    def stat(sel):
        if not sel.any():
            return {"count": 0}
        return {"count": int(sel.sum()), "hop_us_mean": float(hops[sel].mean()),
                "p50": float(np.percentile(hops[sel], 50)), "p90": float(np.percentile(hops[sel], 90)),
                "max": float(hops[sel].max()), "sum_us": float(hops[sel].sum())}
    prev_big = np.concatenate([[False], bigc[:-1]])
    out["critical_path"]["handoffs"] = {
        "kept": stat(kept), "claimed": stat(~kept),
        "claimed_big_after_small": stat(~kept & bigc & ~prev_big),
        "claimed_big_after_big": stat(~kept & bigc & prev_big),
        "claimed_small": stat(~kept & ~bigc),
        "big_eliminations": int(bigc.sum()),
    }
    cc = cyc[chs]
    wide = cc[:, 0] > 10**15  # wide columns store globaltimer stamps here, not cycles
    if wide.any():
        w = cc[wide].astype(np.float64)
        s0 = sub[chs][wide, 0].astype(np.float64)
        t3 = tt[chs][wide, 3].astype(np.float64)
        out["critical_path"]["wide_columns"] = {
            "count": int(wide.sum()), "raw_mean": float(raw[chs][wide].mean()),
            "m_mean": float(m[chs][wide].mean()),
            "gather_us": float(((w[:, 0] - s0) / 1e3).mean()),
            "raw_sort_us": float(((w[:, 1] - w[:, 0]) / 1e3).mean()),
            "raw_sort_tiles_us": float(((sub[chs][wide, 1].astype(np.float64) - w[:, 0]) / 1e3).mean()),
            "merge_us": float(((w[:, 2] - w[:, 1]) / 1e3).mean()),
            "lkk_column_us": float(((t3 - w[:, 2]) / 1e3).mean()),
            "weight_sort_us": float(((w[:, 3] - t3) / 1e3)[w[:, 3] > 0].mean()) if (w[:, 3] > 0).any() else None}
    cc = np.where(wide[:, None], 0, cc)
    okc = cc[:, 2] > 0
    if okc.any():
        # cta_hash_merge step barriers (clock64 from the gather's landing)
        out["critical_path"]["cta_hash_merge_cycles"] = {
            "count": int(okc.sum()), "inserted": float(cc[okc, 0].mean()),
            "runs_walked": float(cc[okc, 1].mean()), "runs_summed": float(cc[okc, 2].mean()),
            "rows_ranked": float(cc[okc, 3].mean())}
        # the same by raw-size bucket, with the critical path's raw-size mix
        rr = raw[chs]
        byb = {}
        for lo, hi in ((0, 129), (129, 257), (257, 513), (513, 1025), (1025, 1 << 30)):
            sel = (rr >= lo) & (rr < hi)
            selc = sel & okc
            byb[f"[{lo},{hi})"] = {
                "count": int(sel.sum()), "m_mean": float(m[chs][sel].mean()) if sel.any() else None,
                "service_us": float(dur[chs][sel].mean()) if sel.any() else None,
                "cycles": [float(x) for x in cc[selc].mean(axis=0)] if selc.any() else None}
        out["critical_path"]["by_raw"] = byb
    top = np.argsort(-hops)[:8]
    out["critical_path"]["worst_hops"] = [
        {"pos": int(chs[i]), "hop_us": float(hops[i]), "start_us": float(start[chs[i]]),
         "ready_us": float(ready[chs[i]]), "raw": int(raw[chs[i]]), "m": int(m[chs[i]]),
         "eliminator": int(sub[chs[i], 6]), "kept": int(sub[chs[i], 7]),
         "path_index": int(i)} for i in top]
    print(json.dumps(out, indent=1))
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
