#!/usr/bin/env python3
"""Benchmark of the rchol hot path (BASELINE.json metric): randomized approximate
Cholesky factorization of the 3D 7-point Poisson Laplacian 128^3 (config[1]) on
B200, reported as factor nnz/s (LdlFactor::nnz() / factor seconds), with the PCG
solve to 1e-8 that consumes the factor measured in the same run.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload poisson3d_128|poisson2d_256|poisson27_96|rmat_22|batch_64x64]

One process per GPU (torchrun for N>1). A single factorization does not shard
(SURVEY §8(e)): every rank factors its own independent Laplacian (seed = rank),
so per-GPU work is fixed and scaling is "weak"; there is no data-path collective.

Step = one factorization of the workload with its inputs resident in HBM
(`value`, device time from CUDA events on the library's stream, L2 flushed
between steps). `e2e` = the same factorization through the C ABI
(parac_gpu_factor_to_host: upload, factor, and the factor copied out while the
elimination runs) from and into pinned host buffers, host<->device copies
inside the timed region. `--impl reference` times the reference's own
multithreaded CPU path (oracle/_ref: factor_parallel_left/right, unmodified
sources) on this host's cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "factorization time & factor nnz/s; PCG iters+solve time, 3D Poisson 128³"
FALLBACK_HBM = 6650.0

WORKLOADS = {
    # name: (builder, description)
    "poisson3d_128": ("gen_poisson3d", 128, "3D 7-point Poisson 128^3 (config[1])"),
    "poisson2d_256": ("gen_poisson2d", 256, "2D 5-point Poisson 256^2 (config[0])"),
    "poisson27_96": ("gen_poisson27", 96, "3D 27-point 96^3, w=0.5+1.5U (config[2])"),
    "rmat_22": ("gen_rmat", 22, "R-MAT scale 22, ef 16 (config[3])"),
    "batch_64x64": ("gen_poisson3d", 64, "batch of 64 x 3D Poisson 64^3 (config[4])"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def build_graph(P, workload: str, seed: int):
    kind, size, _ = WORKLOADS[workload]
    if kind == "gen_poisson3d":
        return P.gen_poisson3d(size)
    if kind == "gen_poisson2d":
        return P.gen_poisson2d(size)
    if kind == "gen_poisson27":
        return P.gen_poisson27(size, 1)
    if kind == "gen_rmat":
        return P.gen_rmat(size, 16, seed)
    raise KeyError(workload)


def algorithmic_bytes(n: int, E: int, Z: int, F: int) -> dict:
    """B_fact = 16(n+1) + 8n + 12E + 40F + 20Z. The dominant kernel
    (K3, eliminate) accounts for all of it except the 8(n+1) col_ptr written by K4."""
    b_fact = 16 * (n + 1) + 8 * n + 12 * E + 40 * F + 20 * Z
    return {"fact": b_fact, "k3": b_fact - 8 * (n + 1)}


def read_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if s > 300] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(n_gpus: int):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if os.environ.get("PARAC_BENCH_SAME_DEVICE") == "1":
            # test hook (tests/test_multirank_gpu.py): every rank on cuda:0 over
            # gloo, so the N>1 path runs on a one-GPU box. Not a bench setting.
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    return rank, world, local, pg


def _reduce_device(pg, device):
    """Tensors for torch.distributed ops: the GPU under NCCL, the host under gloo."""
    return device if pg is not None and pg.get_backend() == "nccl" else "cpu"


def barrier(pg, device):
    import torch
    torch.cuda.synchronize(device)
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize(device)


def allreduce(pg, device, value: float, op: str) -> float:
    if pg is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=_reduce_device(pg, device))
    pg.all_reduce(t, op=getattr(pg.ReduceOp, op))
    return float(t.item())


def gather_to_all(pg, obj):
    """Every rank's `obj`, in rank order (reporting only, never on the data path)."""
    if pg is None:
        return [obj]
    out = [None] * pg.get_world_size()
    pg.all_gather_object(out, obj)
    return out


def workload_config(workload: str, n: int, edges: int) -> dict:
    """`config` of BOTH arms (identical dicts: the driver compares them). Only
    what identifies the workload; arm-specific details live outside it."""
    cfg = {"workload": workload, "desc": WORKLOADS[workload][2], "n": n, "edges": edges}
    if workload == "batch_64x64":
        cfg.update({"problems": 64, "ordering": "problem i: ordering_random(n, i)", "seed": "problem i: i"})
    else:
        cfg.update({"ordering": "ordering_random(n, seed)", "seed": "rank (0 at N=1)"})
    cfg["l2"] = "GPU arm: flushed between steps (256 MiB memset); working set > L2 anyway"
    return cfg


def batch_share(rank: int, world: int, total: int = 64):
    """Problems of the 64-problem batch that rank `rank` of `world` factors
    (round-robin; every problem exactly once over the ranks)."""
    return list(range(rank, total, world))


# ---------------------------------------------------------------- reference CPU
# Everything in this section runs the UNMODIFIED reference (oracle/_ref) on its
# own inputs: graphs from the reference's gen_poisson3d / from_edges (the
# port's harness generators for the configs the reference has no generator
# for), orderings from its ordering_random. The product library is never
# imported here.
def cpu_reference_factor(R, h, n, perm, seed, workers_list, repeats=1):
    """Wall clock around the reference API call (host graph in, LdlFactor out),
    BASELINE.md §2: min over {par-left, par-right} x workers."""
    best = None
    rows = []
    for backend, bname in ((R.LEFT, "par-left"), (R.RIGHT, "par-right")):
        for w in workers_list:
            for _ in range(repeats):
                f, wall = R.factor(h, perm, seed, backend=backend, workers=w)
                nnz = R.L.pref_factor_nnz_off(f) + n
                R.free_factor(f)
                rows.append((wall, bname, w))
                if best is None or wall < best[0]:
                    best = (wall, bname, w, nnz)
    return best, rows


def cpu_reference_pcg(R, h, perm, seed, tol=1e-8):
    """pcg_solve (src/solver.cpp:95-175, single-threaded by design) on the
    reference's own factor of the same graph/ordering/seed, rhs
    make_rhs(random_projected, 0): the same-box baseline of the metric's
    second half. Timed by the reference's SolveReport::solve_seconds."""
    f, _ = R.factor(h, perm, seed, backend=R.LEFT, workers=os.cpu_count() or 1)
    try:
        b = R.make_rhs(h, 1, 0)  # RhsMode::random_projected
        _, rep = R.pcg(h, f, b, tol=tol)
    finally:
        R.free_factor(f)
    return {"seconds": rep["seconds"], "iterations": rep["iterations"],
            "relative_residual": rep["relative_residual"], "converged": rep["converged"], "cores": 1,
            "kind": "reference", "sample": "1 full pcg_solve to tol 1e-8 (single-threaded by design)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # other ranks exit without work (the CPU path does not shard)
    import oracle
    workload = args.workload
    cores = os.cpu_count() or 1
    if not oracle.Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libparac_ref.so not built "
                          "(needs /root/reference at build time)"}), flush=True)
        return
    R = oracle.Reference()
    if workload == "batch_64x64":
        return run_reference_batch(args, R, cores)
    h = R.workload_graph(workload, 0)
    n = R.L.pref_graph_n(h)
    E = R.L.pref_graph_nnz(h) // 2
    perm = R.ordering_random(n, 0)
    cands = sorted({w for w in (cores, max(1, cores // 2), min(cores, 32), min(cores, 16), 8) if w <= cores})
    # warm-up: pick the best backend x workers (BASELINE.md §2 T_cpu rule)
    (w0, bname, wk, nnz), rows = cpu_reference_factor(R, h, n, perm, 0, cands)
    log("reference sweep:", [(round(a, 3), b, c) for a, b, c in rows])
    backend = R.LEFT if bname == "par-left" else R.RIGHT
    for _ in range(max(0, args.warmup - 1)):
        f, _ = R.factor(h, perm, 0, backend=backend, workers=wk)
        R.free_factor(f)
    times = []
    for _ in range(args.steps):
        f, wall = R.factor(h, perm, 0, backend=backend, workers=wk)
        R.free_factor(f)
        times.append(wall)
    pcg = None
    if not args.no_pcg and workload != "rmat_22":  # R-MAT is disconnected: pcg_solve refuses it
        cb = cpu_reference_pcg(R, h, perm, 0)
        pcg = {"iterations": cb["iterations"], "relative_residual": cb["relative_residual"],
               "converged": cb["converged"], "solve_ms": cb["seconds"] * 1e3, "tol": 1e-8, "cpu_baseline": cb}
    R.free_graph(h)
    sec = sum(times) / len(times)
    value = nnz / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "nnz/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(workload, n, E),
        "reference": {"backend": bname, "workers": wk, "library": "oracle/_ref/libparac_ref.so (unmodified sources)"},
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": wk, "kind": "reference",
                         "sample": f"{args.steps} full factorizations of {workload}, {bname} x {wk} threads, "
                                   f"wall clock around the API call (host graph in, LdlFactor out)"},
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "pcg": pcg,
    }
    print(json.dumps(line), flush=True)


def cpu_reference_batch(R, cores, count):
    """SURVEY §8(d) batch rule: nproc threads x factor_randomized, one problem per
    thread (the reference has no batch API). Returns (seconds, total nnz, count)."""
    h = R.poisson3d(64)
    n = R.L.pref_graph_n(h)
    perms = [R.ordering_random(n, i) for i in range(count)]
    nnz = [0] * count

    def work(i):
        f, _ = R.factor(h, perms[i], i, backend=R.SEQ, workers=1)
        nnz[i] = R.L.pref_factor_nnz_off(f) + n
        R.free_factor(f)

    from concurrent.futures import ThreadPoolExecutor
    t = time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as ex:
        list(ex.map(work, range(count)))
    sec = time.perf_counter() - t
    R.free_graph(h)
    return sec, sum(nnz), count


def run_reference_batch(args, R, cores):
    # a bounded sample: `cores` problems per step (one per host thread), so a
    # step is one wave of the 64-problem batch
    count = min(64, cores)
    for _ in range(max(0, args.warmup - 2)):
        cpu_reference_batch(R, cores, count)
    secs, nnz = [], 0
    for _ in range(args.steps):
        sec, nnz, _ = cpu_reference_batch(R, cores, count)
        secs.append(sec)
    sec = sum(secs) / len(secs)
    value = nnz / sec
    h = R.poisson3d(64)
    n, E = R.L.pref_graph_n(h), R.L.pref_graph_nnz(h) // 2
    R.free_graph(h)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "nnz/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config("batch_64x64", n, E),
        "reference": {"backend": "factor_randomized x threads", "workers": cores, "problems_per_step": count},
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": cores, "kind": "reference",
                         "sample": f"{count} problems of the batch per step, {cores} threads x "
                                   f"factor_randomized (one problem per thread), wall clock"},
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- ours (GPU)
def pinned_copy(P, arr: np.ndarray):
    nbytes = arr.nbytes
    ptr = P.rchol.lib.parac_host_alloc(max(nbytes, 1))
    if not ptr:
        raise MemoryError("parac_host_alloc failed")
    buf = (C.c_char * max(nbytes, 1)).from_address(ptr)
    out = np.frombuffer(buf, dtype=arr.dtype, count=arr.size)
    out[:] = arr
    return ptr, out


def run_ours(args):
    import torch

    import paper_2505_02977_b200 as P
    from paper_2505_02977_b200 import _lib as L

    rank, world, local, pg = dist_setup(args.gpus)
    if args.workload == "batch_64x64":
        return run_ours_batch(args, P, L, torch, rank, world, local, pg)
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    seed = rank
    workload = args.workload
    lib = P.rchol.lib

    g = build_graph(P, workload, seed)
    order = P.ordering_random(g.n, seed)
    n, E = g.n, g.num_edges()
    ctx = P.GpuContext(local)
    opts = P.GpuOptions().native()
    info = L.parac_gpu_factor_info()

    # pinned host inputs/outputs for the end-to-end leg
    hp = [pinned_copy(P, a) for a in (g.ptr, g.adj, g.w, order.perm)]
    csr = L.parac_csr(n, hp[0][0], hp[1][0], hp[2][0])
    perm_ptr = hp[3][0]

    def check(rc):
        if rc != 0:
            raise P.Error(rc, lib.parac_gpu_last_error().decode())

    # resident input for the device-time leg
    check(lib.parac_gpu_upload(ctx.handle, C.byref(csr), perm_ptr))
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=device)

    attempts = []

    def device_step():
        check(lib.parac_gpu_factor_resident(ctx.handle, seed, C.byref(opts), C.byref(info)))
        attempts.append(info.attempts)  # device_ms includes any budget-growth retries
        return info.device_ms, info.eliminate_ms

    for _ in range(args.warmup):
        device_step()
    Z = info.nnz_off_diagonal
    F = info.total_fills
    nnz = Z + n
    out_bufs = [pinned_copy(P, np.zeros(k, dt)) for k, dt in
                ((n + 1, np.int64), (max(Z, 1), np.int32), (max(Z, 1), np.float64), (max(n, 1), np.float64))]

    # ---- timed: resident inputs, device time (CUDA events on the library stream)
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    l0 = lib.parac_gpu_launch_count()
    barrier(pg, device)
    dev_ms, k3_ms = [], []
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush (256 MiB > 126 MB L2) between steps, outside the events
        torch.cuda.synchronize(device)
        a, b = device_step()
        dev_ms.append(a)
        k3_ms.append(b)
    barrier(pg, device)
    wall_resident = time.perf_counter() - t_wall
    launches = lib.parac_gpu_launch_count() - l0
    clk = clocks.stop() if clocks else None
    total_dev_s = sum(dev_ms) / 1e3
    max_dev_s = allreduce(pg, device, total_dev_s, "MAX")
    total_nnz = allreduce(pg, device, float(nnz * args.steps), "SUM")
    value = total_nnz / max_dev_s

    # ---- timed: end to end through the C ABI from pinned host memory
    barrier(pg, device)
    e2e_s = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        # upload, factor, and the factor copied out while it is computed
        # (parac_gpu_factor_to_host: the streamed assembly + download)
        check(lib.parac_gpu_factor_to_host(ctx.handle, C.byref(csr), perm_ptr, seed, C.byref(opts), C.byref(info),
                                           out_bufs[0][0], out_bufs[1][0], out_bufs[2][0], out_bufs[3][0],
                                           max(Z, 1)))
        e2e_s.append(time.perf_counter() - t0)
    barrier(pg, device)
    e2e_total = allreduce(pg, device, sum(e2e_s), "MAX")
    e2e_value = total_nnz / e2e_total
    h2d = 8 * (n + 1) + 12 * 2 * E + 4 * n
    d2h = 8 * (n + 1) + 12 * Z + 8 * n
    # parity of the e2e output against the resident run (same bits every call)
    f_e2e = P.LdlFactor(n, out_bufs[0][1], out_bufs[1][1][:Z], out_bufs[2][1][:Z], out_bufs[3][1][:n], order.perm)
    checksum = f_e2e.checksum()

    # ---- PCG to 1e-8 on the resident factor (BASELINE metric, second half)
    pcg = None
    if not args.no_pcg and workload != "rmat_22":
        check(lib.parac_gpu_factor_resident(ctx.handle, seed, C.byref(opts), C.byref(info)))
        b = P.make_rhs(g, "random_projected", 0)
        # first call on a new factor also builds the solve layout (G transpose,
        # level order, tail tables): reported as first_call_wall_ms
        _, rep0 = P.rchol._pcg_resident(ctx, b, P.SolveConfig(tol=1e-8))
        x, rep = P.rchol._pcg_resident(ctx, b, P.SolveConfig(tol=1e-8))
        pcg = {"iterations": rep.iterations, "relative_residual": rep.relative_residual,
               "converged": rep.converged, "solve_ms": rep.device_ms, "wall_ms": rep.solve_seconds * 1e3,
               "first_call_wall_ms": rep0.solve_seconds * 1e3, "tol": 1e-8}

    # ---- the drop-in C++ call (parac::factor_gpu through the shim, the
    # reference's own types, pageable std::vector outputs): tools/_build/dropin_time
    dropin = None
    if rank == 0 and world == 1 and workload == "poisson3d_128" and not args.no_dropin:
        exe = os.path.join(ROOT, "tools", "_build", "dropin_time")
        if os.path.exists(exe):
            try:
                out = subprocess.run([exe, "128", str(max(3, args.steps)), "2"], capture_output=True, text=True,
                                     timeout=600)
                d = json.loads(out.stdout.strip().splitlines()[-1])
                dropin = {"value": d["nnz"] / (d["ms_per_call"] / 1e3), "unit": "nnz/s",
                          "ms_per_step": d["ms_per_call"], "calls_ms": d["calls"], "checksum": d["checksum"],
                          "what": "parac::factor_gpu(LaplacianGraph, Ordering, seed) -> LdlFactor (C++ shim, "
                                  "cached device context, pageable std::vector in/out), host clock around the call"}
            except Exception as exc:
                dropin = {"value": None, "unit": "nnz/s", "error": str(exc)}
        else:
            dropin = {"value": None, "unit": "nnz/s", "error": "tools/_build/dropin_time not built"}

    peak, peak_src = read_peaks()
    by = algorithmic_bytes(n, E, Z, F)
    k3_avg_s = sum(k3_ms) / len(k3_ms) / 1e3
    achieved = by["k3"] / k3_avg_s / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as fh:
                traffic = json.load(fh).get(workload, {}).get("eliminate_kernel_dram_bytes")
        except Exception:
            traffic = None

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            R = oracle.Reference()
            cores = os.cpu_count() or 1
            h = R.workload_graph(workload, seed)
            rperm = R.ordering_random(n, seed)
            (wall, bname, wk, cnnz), _ = cpu_reference_factor(R, h, n, rperm, seed, [cores])
            cpu_base = {"value": cnnz / wall, "unit": "nnz/s", "cores": wk, "kind": "reference",
                        "sample": f"1 full {workload} factorization, {bname} x {wk} threads "
                                  f"(best of par-left/par-right), wall clock around the API call",
                        "seconds": wall}
            if pcg is not None:
                pcg["cpu_baseline"] = cpu_reference_pcg(R, h, rperm, seed)
            R.free_graph(h)
        except Exception as exc:  # oracle/_ref missing -> port timing would be 1-core
            cpu_base = {"value": None, "unit": "nnz/s", "cores": 0, "kind": "reference",
                        "sample": f"unavailable: {exc}"}

    ctx.close()
    # BASELINE config[4] at this N: the 64 x 64^3 batch split over the ranks
    # (the north_star's "reported at 1, 2, 4 and 8 GPUs"), as a sub-record of
    # the headline line so the driver's scaling run yields that curve too
    batch = None
    if not args.no_batch and workload == "poisson3d_128":
        try:
            batch = measure_batch(args, P, L, torch, rank, world, local, pg, e2e=False)
            batch.pop("clocks", None)
            batch["n_gpus"] = world
        except Exception as exc:
            batch = {"value": None, "error": str(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": max_dev_s / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (host generators = reference gen_poisson3d etc.; ordering_random(n, rank), seed = rank)",
            "config": workload_config(workload, n, E),
            "factor": {"nnz_G": nnz, "fills": F, "factor_checksum": f"{checksum:016x}",
                       "per_gpu": "one independent factorization per rank", "parallelism": f"replicas x{world}"},
            "factor_ms": {"device": max_dev_s / args.steps * 1e3,
                          "eliminate_k3": sum(k3_ms) / len(k3_ms), "wall_resident_loop_s": wall_resident,
                          "device_passes_per_step": max(attempts) if attempts else 1},
            "e2e": {"value": e2e_value, "unit": "nnz/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_total / args.steps * 1e3},
            "e2e_dropin": dropin,
            "pcg": pcg,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "eliminate_kernel (K3)", "algorithmic_bytes": by["k3"],
                         "peak_source": peak_src},
            "cpu_baseline": cpu_base,
            "gpu_launches": launches,
            "clocks": clk,
            "batch": batch,
        }
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


def measure_batch(args, P, L, torch, rank, world, local, pg, e2e=True):
    """BASELINE config[4]: 64 independent gen_poisson3d(64) problems (problem i:
    ordering_random(n, i), seed i) split round-robin over the ranks; each rank
    factors its share in ONE device pass (disjoint-union batch, byte-identical
    per-problem factors). No collective on the data path: the ranks only meet
    at the timing barriers and the max/sum reductions of the result."""
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    lib = P.rchol.lib
    mine = batch_share(rank, world)
    g = P.gen_poisson3d(64)
    perms = [P.ordering_random(g.n, i).perm for i in mine]
    ctx = P.GpuContext(local)
    opts = P.GpuOptions().native()
    info = L.parac_gpu_factor_info()

    def check(rc):
        if rc != 0:
            raise P.Error(rc, lib.parac_gpu_last_error().decode())

    # pinned host inputs (one graph, per-problem orderings) for the e2e leg
    hg = [pinned_copy(P, a) for a in (g.ptr, g.adj, g.w)]
    hp = [pinned_copy(P, p) for p in perms]
    csr1 = L.parac_csr(g.n, hg[0][0], hg[1][0], hg[2][0])
    csrs = (L.parac_csr * len(mine))(*([csr1] * len(mine)))
    pptr = (C.c_void_p * len(mine))(*[p[0] for p in hp])
    seeds = np.array(mine, dtype=np.uint64)
    check(lib.parac_gpu_upload_batch(ctx.handle, len(mine), csrs, pptr, seeds.ctypes.data))
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=device)
    for _ in range(args.warmup):
        check(lib.parac_gpu_factor_resident(ctx.handle, 0, C.byref(opts), C.byref(info)))
    nnz_total = info.nnz_off_diagonal + info.n
    F, Z = info.total_fills, info.nnz_off_diagonal
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    l0 = lib.parac_gpu_launch_count()
    barrier(pg, device)
    dev_ms, k3_ms = [], []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize(device)
        check(lib.parac_gpu_factor_resident(ctx.handle, 0, C.byref(opts), C.byref(info)))
        dev_ms.append(info.device_ms)
        k3_ms.append(info.eliminate_ms)
    barrier(pg, device)
    launches = lib.parac_gpu_launch_count() - l0
    clk = clocks.stop() if clocks else None
    max_dev_s = allreduce(pg, device, sum(dev_ms) / 1e3, "MAX")
    total_nnz = allreduce(pg, device, float(nnz_total * args.steps), "SUM")
    zs = []
    for i in range(len(mine)):
        z = C.c_int64()
        check(lib.parac_gpu_batch_nnz(ctx.handle, i, C.byref(z)))
        zs.append(int(z.value))
    outs = [[pinned_copy(P, np.zeros(k, dt)) for k, dt in
             ((g.n + 1, np.int64), (max(z, 1), np.int32), (max(z, 1), np.float64), (g.n, np.float64))]
            for z in zs]
    res = {"value": total_nnz / max_dev_s, "unit": "nnz/s", "ms_per_step": max_dev_s / args.steps * 1e3,
           "eliminate_k3_ms": sum(k3_ms) / len(k3_ms), "problems": 64, "problems_per_gpu": len(mine),
           "nnz_G_per_gpu": nnz_total, "fills_per_gpu": F, "nnz_off_per_gpu": Z, "n_per_gpu": info.n,
           "edges_per_gpu": g.num_edges() * len(mine), "launches": launches, "clocks": clk,
           "scaling": "strong", "what": "64 x gen_poisson3d(64) split round-robin over the ranks, "
                                       "one disjoint-union device pass per rank, max-over-ranks device time"}
    # e2e: parac_gpu_factor_batch_to_host from pinned host inputs into pinned host outputs
    if e2e:
        out_arrays = [(C.c_void_p * len(outs))(*[o[j][0] for o in outs]) for j in range(4)]
        caps = np.array([max(z, 1) for z in zs], np.int64)
        barrier(pg, device)
        e2e_s = []
        e2e_parts = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize(device)
            t0 = time.perf_counter()
            # upload, factor, and every member copied out while the union is
            # factored (parac_gpu_factor_batch_to_host: the streamed download)
            check(lib.parac_gpu_factor_batch_to_host(ctx.handle, len(mine), csrs, pptr, seeds.ctypes.data,
                                                     C.byref(opts), C.byref(info), *out_arrays, caps.ctypes.data))
            e2e_s.append(time.perf_counter() - t0)
            e2e_parts.append((info.upload_ms, info.device_ms))
        barrier(pg, device)
        e2e_total = allreduce(pg, device, sum(e2e_s), "MAX")
        h2d = len(mine) * (8 * (g.n + 1) + 12 * 2 * g.num_edges() + 4 * g.n)
        d2h = sum(8 * (g.n + 1) + 12 * z + 8 * g.n for z in zs)
        res["e2e"] = {"value": total_nnz / e2e_total, "unit": "nnz/s", "h2d_bytes_per_step": h2d,
                      "d2h_bytes_per_step": d2h, "ms_per_step": e2e_total / args.steps * 1e3,
                      "upload_wall_ms": sum(u for u, _ in e2e_parts) / len(e2e_parts),
                      "device_ms": sum(d for _, d in e2e_parts) / len(e2e_parts)}
    else:  # outputs of the last resident pass
        for i, o in enumerate(outs):
            check(lib.parac_gpu_download_batch(ctx.handle, i, o[0][0], o[1][0], o[2][0], o[3][0]))
    sums = {}
    for i, (p, o, z) in enumerate(zip(mine, outs, zs)):
        f = P.LdlFactor(g.n, o[0][1], o[1][1][:z], o[2][1][:z], o[3][1], perms[i])
        sums[p] = f"{f.checksum():016x}"
    allsums = {}
    for part in gather_to_all(pg, sums):
        allsums.update(part)
    res["checksums"] = [allsums.get(i) for i in range(64)]
    res["factor0_checksum"] = allsums.get(0)
    ctx.close()
    return res


def run_ours_batch(args, P, L, torch, rank, world, local, pg):
    res = measure_batch(args, P, L, torch, rank, world, local, pg)
    device = torch.device("cuda", local)
    peak, peak_src = read_peaks()
    g_n, g_e = 64 ** 3, res["edges_per_gpu"] // res["problems_per_gpu"]
    by = algorithmic_bytes(res["n_per_gpu"], res["edges_per_gpu"], res["nnz_off_per_gpu"], res["fills_per_gpu"])
    achieved = by["k3"] / (res["eliminate_k3_ms"] / 1e3) / 1e9
    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            cores = os.cpu_count() or 1
            sec, cnnz, cnt = cpu_reference_batch(oracle.Reference(), cores, min(64, cores))
            cpu_base = {"value": cnnz / sec, "unit": "nnz/s", "cores": cores, "kind": "reference",
                        "sample": f"{cnt} of the 64 problems, {cores} threads x factor_randomized "
                                  f"(one problem per thread), wall clock", "seconds": sec}
        except Exception as exc:
            cpu_base = {"value": None, "unit": "nnz/s", "cores": 0, "kind": "reference",
                        "sample": f"unavailable: {exc}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": "nnz/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gen_poisson3d(64) x 64; problem i: ordering_random(n, i), seed i)",
            "config": workload_config("batch_64x64", g_n, g_e),
            "factor": {"problems_per_gpu": res["problems_per_gpu"], "nnz_G_per_gpu": res["nnz_G_per_gpu"],
                       "factor0_checksum": res["factor0_checksum"], "checksums": res["checksums"],
                       "per_gpu": "its share of the 64 problems as one disjoint-union device pass",
                       "parallelism": f"batch split x{world}"},
            "factor_ms": {"device": res["ms_per_step"], "eliminate_k3": res["eliminate_k3_ms"]},
            "e2e": res["e2e"],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "kernel": "eliminate_kernel (K3)",
                         "algorithmic_bytes": by["k3"], "peak_source": peak_src},
            "cpu_baseline": cpu_base,
            "gpu_launches": res["launches"],
            "clocks": res["clocks"],
        }
        print(json.dumps(line), flush=True)
    del device
    if pg is not None:
        pg.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="poisson3d_128")
    ap.add_argument("--no-pcg", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dropin", action="store_true")
    ap.add_argument("--no-batch", action="store_true", help="skip the 64x64^3 batch sub-record")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: --warmup < 3 violates the timing rules; using 3")
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
