#!/usr/bin/env python3
"""Analyse a PARAC_SWEEP_TRACE dump (tools: apply_preconditioner at 128^3):
per-level durations of the forward / backward sweeps, service vs wait."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(path, n3):
    import paper_2505_02977_b200 as P
    os.environ["PARAC_SWEEP_TRACE"] = path
    g = P.gen_poisson3d(n3)
    o = P.ordering_random(g.n, 0)
    ctx = P.GpuContext(0)
    ctx.set_preconditioner_mode(os.environ.get("SWEEP_MODE", "default"))
    f = P.factor_gpu(g, o, 0, ctx=ctx)
    r = P.make_rhs(g, "random_projected", 0)
    for _ in range(3):
        P.apply_preconditioner_gpu(f, r, ctx=ctx)
    np.save(path + ".rowlen.npy", np.bincount(f.rows, minlength=g.n))
    np.save(path + ".collen.npy", np.diff(f.col_ptr))


def analyse(path):
    raw = open(path, "rb").read()
    n = int(np.frombuffer(raw[:4], np.int32)[0])
    tr = np.frombuffer(raw[4:4 + 48 * n], np.uint64).astype(np.int64).reshape(2, n, 3)
    lv = np.frombuffer(raw[4 + 48 * n:], np.int32)[:n]
    depth = lv.max()
    for name, t in (("forward", tr[0]), ("backward", tr[1])):
        t0 = t[:, 0].min()
        start, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
        span = end.max()
        fin = np.zeros(depth + 2)
        np.maximum.at(fin, lv, end)
        sizes = np.bincount(lv, minlength=depth + 2)
        order = range(1, depth + 1) if name == "forward" else range(depth, 0, -1)
        prev, per = 0.0, []
        for L in order:
            per.append(fin[L] - prev)
            prev = fin[L]
        per = np.array(per)
        svc = end - start
        claim = (t[:, 2] - t0) / 1e3
        # hand-off: level L-1 (fwd) / L+1 (bwd) finish -> row start
        prevL = lv - 1 if name == "forward" else lv + 1
        ok = (prevL >= 1) & (prevL <= depth)
        hand = start[ok] - fin[prevL[ok]]
        late = claim[ok] - fin[prevL[ok]]
        tail = ok & (sizes[lv] < 4)
        print(f"   hand-off (prev level done -> start) median {np.median(hand):.2f} us p90 {np.percentile(hand, 90):.2f}; "
              f"tail levels: {np.median(start[tail] - fin[prevL[tail]]):.2f} us; rows claimed after prev level done: "
              f"{(late > 0).mean() * 100:.1f}% (tail {(claim[tail] > fin[prevL[tail]]).mean() * 100:.1f}%)")
        print(f"{name}: span {span:.0f} us, depth {depth}, per-level median {np.median(per):.2f} us, "
              f"mean {per.mean():.2f}, service mean {svc.mean():.2f} us p99 {np.percentile(svc, 99):.2f}")
        lens = np.load(path + (".rowlen.npy" if name == "forward" else ".collen.npy"))
        tl = sizes[lv] < 4
        print(f"   tail rows: n={tl.sum()} length mean {lens[tl].mean():.0f} max {lens[tl].max()} "
              f"service mean {svc[tl].mean():.2f} us; all rows length mean {lens.mean():.1f}")
        small = sizes[1:depth + 1] < 64
        print(f"   levels with <64 rows: {small.sum()}, their total time {per[small[::1] if name=='forward' else small[::-1]].sum():.0f} us")
        qs = [0, 5, 10, 20, 50, 100, 200, 500, 1000, depth - 1]
        print("   level: size, finish us:", [(int(q + 1), int(sizes[q + 1]), round(float(fin[q + 1]), 1)) for q in qs if q + 1 <= depth])


if __name__ == "__main__":
    path = sys.argv[1] if len(sys.argv) > 1 else "/tmp/sweep_trace.bin"
    if len(sys.argv) <= 2:
        run(path, 128)
    analyse(path)


def bands(path):
    """Per level band: level duration, and per-row (ready-notice) = start - finish(prev level)."""
    raw = open(path, "rb").read()
    n = int(np.frombuffer(raw[:4], np.int32)[0])
    tr = np.frombuffer(raw[4:4 + 48 * n], np.uint64).astype(np.int64).reshape(2, n, 3)
    lv = np.frombuffer(raw[4 + 48 * n:], np.int32)[:n]
    depth = lv.max()
    t = tr[0]
    t0 = t[:, 2].min()
    start, end, claim = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
    fin = np.zeros(depth + 2)
    np.maximum.at(fin, lv, end)
    for lo, hi in ((2, 6), (6, 20), (20, 50), (50, 100), (100, 200), (200, 500), (500, 1000), (1000, depth + 1)):
        sel = (lv >= lo) & (lv < hi)
        notice = start[sel] - fin[lv[sel] - 1]
        durl = np.diff(fin[lo - 1:hi])
        # rows finishing last in their level: how late did they start?
        lastrow = np.zeros(depth + 2, np.int64)
        order = np.lexsort((end, lv))
        lastrow[lv[order]] = order
        lr = lastrow[lo:hi]
        print(f"levels [{lo},{hi}): rows {sel.sum():7d} level dur median {np.median(durl):7.2f} us | "
              f"notice median {np.median(notice):7.2f} p90 {np.percentile(notice, 90):7.2f} | "
              f"last row: notice {np.median(start[lr] - fin[lv[lr] - 1]):6.2f} claim-after-prev {np.median(claim[lr] - fin[lv[lr] - 1]):7.2f}")


if __name__ == "__main__" and os.environ.get("BANDS"):
    bands(sys.argv[1] if len(sys.argv) > 1 else "/tmp/sweep.bin")
