#!/usr/bin/env python3
"""Per-level timing of the fast-mode preconditioner sweeps (PARAC_SWEEP_PROFILE):
head cluster sweep forward/backward and the one-CTA tail sweeps, 128^3 by default."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
path = "/tmp/sweep_profile.bin"
os.environ["PARAC_SWEEP_PROFILE"] = path
import paper_2505_02977_b200 as P
n3 = int(sys.argv[1]) if len(sys.argv) > 1 else 128
g = P.gen_poisson3d(n3)
o = P.ordering_random(g.n, 0)
ctx = P.GpuContext(0)
ctx.set_preconditioner_mode("fast")
f = P.factor_gpu(g, o, 0, ctx=ctx)
r = P.make_rhs(g, "random_projected", 0)
for _ in range(3):
    P.apply_preconditioner_gpu(f, r, ctx=ctx)
lv, depth = P.schedule_levels_gpu(f, ctx=ctx)
raw = open(path, "rb").read()
H, D, nt, Lw = np.frombuffer(raw[:16], np.int32)
t_all = np.frombuffer(raw[16:], np.uint64).astype(np.int64)
t = t_all[:4 * (D + 2)].reshape(4, D + 2)
w = np.bincount(lv, minlength=D + 2)
rowlen = np.bincount(f.rows, minlength=g.n)
collen = np.diff(f.col_ptr)
ent_f = np.bincount(lv, weights=rowlen, minlength=D + 2)
ent_b = np.bincount(lv, weights=collen, minlength=D + 2)
print(f"H={H} depth={D} tail rows={nt} wide levels={Lw}")
def show(name, ts, levels, ent):
    ts = ts[:len(levels)]
    d = np.diff(ts) / 1e3
    lv_ = levels[1:]
    print(f"{name}: {len(levels)} levels, span {(ts[-1]-ts[0])/1e3:.1f} us, per-level median {np.median(d):.2f} mean {d.mean():.2f}")
    for lo, hi in ((0, 5), (5, 20), (20, 50), (50, 100), (100, 200), (200, 400), (400, 800), (800, 2000)):
        sel = (np.arange(len(d)) >= lo) & (np.arange(len(d)) < hi)
        if sel.any():
            L = lv_[sel]
            print(f"   steps [{lo},{hi}): levels {L.min()}..{L.max()} time {d[sel].sum():8.1f} us  mean {d[sel].mean():6.2f} us"
                  f"  rows/level {w[L].mean():9.1f}  entries/level {ent[L].mean():10.1f}")
show("head fwd", t[0], np.arange(1, H + 1), ent_f)
if nt:
    print(f"tail: levels {H + 1}..{D} ({nt} rows) by the dense-inverse GEMVs (no per-level stamps)")
show("head bwd", t[3], np.arange(H, 0, -1), ent_b)

# DS cluster head: warp 0 phase cycles per level (see head_sweep_kernel dbg)
nh = H - Lw
def phases(name, base, nlev):
    a = t_all[base:base + 4 * nlev]
    if nlev < 2 or len(a) < 4 * nlev:
        return
    a = a.reshape(nlev, 4)[:-1].astype(np.int64)
    if a.max() <= 0 or a.max() > 10**8:
        return
    print(f"{name} warp-0 cycles per level: load-issue / gather+products / sums+stores / wait+barrier")
    for lo, hi in ((0, 50), (50, 150), (150, nlev)):
        print(f"   steps [{lo},{hi}):", a[lo:hi].mean(axis=0).round(0))
phases("head fwd", Lw + 20 * (nh + 8), nh)
phases("head bwd", 3 * (D + 2) + 4 * (nh + 8), nh)
