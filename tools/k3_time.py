#!/usr/bin/env python3
"""K3 timing sweep (tuning aid): median device / eliminate ms of a resident
factorization per fill-slot setting, L2 flushed between runs.

  python tools/k3_time.py [--workload poisson3d_128] [--c0 0,64,128,256] [--reps 5]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2505_02977_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="poisson3d_128")
    ap.add_argument("--c0", default="0")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    g = bench.build_graph(P, args.workload, 0)
    o = P.ordering_random(g.n, 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    with P.GpuContext(0) as ctx:
        ctx.upload(g, o)
        for c0 in [int(x) for x in args.c0.split(",")]:
            opts = P.GpuOptions(first_chunk=c0, record_stats=False)
            dev, k3 = [], []
            for r in range(args.reps + 2):
                flush.zero_()
                torch.cuda.synchronize()
                info = ctx.factor_resident(0, opts)
                if r >= 2:
                    dev.append(info.device_ms)
                    k3.append(info.eliminate_ms)
            f, _ = ctx.download(with_stats=False)
            print(json.dumps({"workload": args.workload, "c0": c0, "device_ms": statistics.median(dev),
                              "eliminate_ms": statistics.median(k3), "min_k3": min(k3),
                              "checksum": f"{f.checksum():016x}"}), flush=True)


if __name__ == "__main__":
    main()
