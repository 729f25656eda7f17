"""`parac`-compatible command-line runner with a `gpu` backend.

Mirrors the reference CLI (proj/tools/parac_cli.cpp) for the commands on the
factor / solve path -- `gen`, `factor`, `solve`, `bench` -- with the same
flags, the same JSON keys (stats, report, --trace) and the same
`parac-bench-v1` CSV schema, so GPU rows sit next to the reference's own CPU
rows in one table:

    python -m paper_2505_02977_b200.cli bench --gens "poisson3d:n=64" \\
        --orderings random --backends gpu --seeds 0,1 --solve --csv -

Only the `gpu` backend exists here (the CPU backends are the reference's);
any other backend name is a parse error, exit code 10 + Errc like the
reference's (parac_cli.cpp:39). Generator specs accept the reference's
`poisson3d:n=..,variant=..,epsilon=..,contrast=..,seed=..`
(src/generators.cpp:67-108) plus this harness's BASELINE shapes:
`poisson2d:n=..`, `poisson27:n=..,seed=..`, `rmat:scale=..,edge_factor=..,seed=..`.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from typing import List, Optional

import numpy as np

from . import rchol as R

BENCH_SCHEMA = "parac-bench-v1"  # parac_cli.cpp:36


class CliError(Exception):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def _parse_fail(msg: str):
    raise CliError(int(R.Errc.parse_error), msg)


# ------------------------------------------------------------------ inputs
def parse_gen_spec(text: str) -> R.LaplacianGraph:
    """parse_poisson_spec (src/generators.cpp:67-108) + harness generators."""
    kind, _, rest = text.partition(":")
    opts = {}
    if rest:
        for item in rest.split(","):
            key, eq, value = item.partition("=")
            if not eq:
                _parse_fail(f'bad generator option "{item}"')
            opts[key] = value

    def num(key, conv, default):
        if key not in opts:
            return default
        try:
            return conv(opts.pop(key))
        except ValueError:
            _parse_fail(f'bad value for "{key}"')

    if kind == "poisson3d":
        n = num("n", int, 16)
        variant = opts.pop("variant", "uniform")
        if variant not in ("uniform", "anisotropic", "contrast"):
            _parse_fail(f'unknown variant "{variant}"')
        eps, contrast, seed = num("epsilon", float, 1e-3), num("contrast", float, 1e4), num("seed", int, 0)
        if opts:
            _parse_fail(f'unknown generator option "{next(iter(opts))}"')
        if eps <= 0.0 or contrast <= 0.0:
            _parse_fail("epsilon and contrast must be positive")
        return R.gen_poisson3d(n, variant, eps, contrast, seed)
    if kind == "poisson2d":
        g = R.gen_poisson2d(num("n", int, 16))
    elif kind == "poisson27":
        g = R.gen_poisson27(num("n", int, 16), num("seed", int, 1))
    elif kind == "rmat":
        g = R.gen_rmat(num("scale", int, 10), num("edge_factor", int, 16), num("seed", int, 0))
    else:
        _parse_fail('generator spec must start with "poisson3d:" (or poisson2d:, poisson27:, rmat:)')
    if opts:
        _parse_fail(f'unknown generator option "{next(iter(opts))}"')
    return g


def load_graph(input_path: str, gen: str) -> R.LaplacianGraph:
    if input_path and gen:
        _parse_fail("--input and --gen are mutually exclusive")
    if input_path:
        return R.read_laplacian(input_path)
    if gen:
        return parse_gen_spec(gen)
    _parse_fail("one of --input or --gen is required")


def make_ordering(graph: R.LaplacianGraph, text: str, seed: int, ctx) -> R.Ordering:
    """make_ordering (parac_cli.cpp:90-100); nnz-sort runs on the device."""
    if text == "natural":
        return R.Ordering.identity(graph.n)
    if text == "random":
        return R.ordering_random(graph.n, seed)
    if text == "nnz-sort":
        return R.ordering_nnz_sort_gpu(graph, seed, ctx=ctx)
    if text.startswith("file:"):
        return R.ordering_from_file(text[5:], graph.n)
    _parse_fail(f'unknown ordering "{text}" (natural|random|nnz-sort|file:<path>)')


def fill_ratio(graph: R.LaplacianGraph, factor: R.LdlFactor) -> float:
    """fill_ratio (src/etree.cpp:137-142)."""
    return 2.0 * factor.nnz() / float(int(graph.ptr[graph.n]) + graph.n)


def resolve_seed(seed: Optional[int]) -> int:
    if seed is not None:
        return seed
    env = os.environ.get("PARAC_SEED")
    if env is None:
        return 0
    try:
        return int(env)
    except ValueError:
        _parse_fail(f"PARAC_SEED is not an integer: {env}")


def run_factor(graph, ordering, backend: str, seed: int, ctx, record_times=False):
    if backend != "gpu":
        _parse_fail(f'unknown backend "{backend}" (gpu; the CPU backends are the reference\'s)')
    stats = R.FactorStats()
    opts = R.GpuOptions(record_times=record_times)
    f = R.factor_gpu(graph, ordering, seed, opts, stats, ctx=ctx)
    return f, stats


def hbm_peak_gbs() -> float:
    """The measured HBM copy bandwidth (MEASURED_PEAKS.json at the repo root,
    driver-written), else the B200 profiling recipe's fallback."""
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0


def device_metrics(graph: R.LaplacianGraph, factor: R.LdlFactor, st: R.FactorStats) -> dict:
    """SURVEY §5 metrics next to the reference's stats keys: device and
    wall seconds of the factorization and the achieved HBM bandwidth of its
    algorithmic bytes B_fact = 16(n+1) + 8n + 12E + 40F + 20Z."""
    n, E, Z, F = factor.n, graph.num_edges(), factor.nnz_off_diagonal(), int(st.total_fills)
    b_fact = 16 * (n + 1) + 8 * n + 12 * E + 40 * F + 20 * Z
    dev_s = st.device_ms / 1e3
    gbs = b_fact / dev_s / 1e9 if dev_s > 0 else 0.0
    return {"device_seconds": dev_s, "wall_seconds": st.seconds, "eliminate_seconds": st.eliminate_ms / 1e3,
            "algorithmic_bytes": b_fact, "hbm_gbs": gbs, "roofline_fraction": gbs / hbm_peak_gbs()}


def emit_json(payload, path: str) -> None:
    """emit_json (parac_cli.cpp:136-144): nlohmann dump(2) = sorted keys, 2-space indent."""
    text = json.dumps(payload, indent=2, sort_keys=True) + "\n"
    emit_text(text, path)


def emit_text(text: str, path: str) -> None:
    if not path or path == "-":
        sys.stdout.write(text)
        sys.stdout.flush()
        return
    try:
        with open(path, "w") as fh:
            fh.write(text)
    except OSError:
        raise CliError(int(R.Errc.io_error), f"cannot write {path}")


def provenance(input_name, ordering, backend, workers, seed):
    return {"input": input_name, "ordering": ordering, "backend": backend, "workers": workers, "seed": seed,
            "identity_hash": False}


def write_trace(path, factor, stats, ordering, ctx, times=None):
    """write_trace (parac_cli.cpp:156-180)."""
    levels, depth = R.schedule_levels_gpu(factor, ctx=ctx)
    inv = ordering.inverse
    verts = []
    for k in range(factor.n):
        v = {"position": k, "label": int(inv[k]), "round": int(levels[k]),
             "fills": int(stats.fills_received[k]) if len(stats.fills_received) else 0,
             "samples": int(stats.samples_emitted[k]) if len(stats.samples_emitted) else 0}
        if times is not None:
            v["seconds"] = float(times[k])
        verts.append(v)
    emit_json({"n": factor.n, "rounds": depth, "total_fills": int(stats.total_fills), "vertices": verts}, path)


def _g(x: float) -> str:
    """std::ostream << double with the default precision (printf %g)."""
    return "%g" % x


def _csv_field(value: str) -> str:
    if not any(c in value for c in ',"\n'):
        return value
    return '"' + value.replace('"', '""') + '"'


# ---------------------------------------------------------------- commands
def cmd_gen(a) -> int:
    if not a.gen:
        _parse_fail("gen requires --gen")
    g = parse_gen_spec(a.gen)
    R.write_matrix_market(a.output, g)
    print(f"wrote {a.output}: {g.n} vertices, {g.num_edges()} edges")
    return 0


def cmd_factor(a, ctx) -> int:
    seed = resolve_seed(a.seed)
    g = load_graph(a.input, a.gen)
    o = make_ordering(g, a.ordering, seed, ctx)
    f, st = run_factor(g, o, a.backend, seed, ctx, record_times=a.trace_times)
    if a.output:
        R.write_factor(f, a.output)
        R.write_permutation(a.output + ".perm.txt", o)
    if a.trace:
        times = None
        if a.trace_times:
            t = ctx.vertex_times()
            times = (t[:, 7].astype(np.float64) - float(t[:, 0].min())) / 1e9
        write_trace(a.trace, f, st, o, ctx, times)
    _, depth = R.schedule_levels_gpu(f, ctx=ctx)
    stats = {"config": provenance(a.input or a.gen, a.ordering, a.backend, a.workers, seed), "n": f.n,
             "nnz_g": f.nnz(), "nnz_g_off_diagonal": f.nnz_off_diagonal(), "fill_ratio": fill_ratio(g, f),
             "schedule_depth": depth, "total_fills": int(st.total_fills), "factor_seconds": st.seconds,
             "checksum": f.checksum()}
    stats.update(device_metrics(g, f, st))
    if st.arena_used > 0:
        stats["arena_used"] = int(st.arena_used)
    emit_json(stats, a.stats)
    return 0


def cmd_solve(a, ctx) -> int:
    seed = resolve_seed(a.seed)
    g = load_graph(a.input, a.gen)
    factor_seconds = 0.0
    if a.factor:
        perm = a.perm or (a.factor + ".perm.txt" if os.path.exists(a.factor + ".perm.txt") else "")
        f = R.read_factor(a.factor, perm)
    else:
        o = make_ordering(g, a.ordering, seed, ctx)
        f, st = run_factor(g, o, a.backend, seed, ctx)
        factor_seconds = st.seconds
    if a.rhs:
        b = R.read_vector(a.rhs)
    elif a.rhs_mode in ("random-projected", "from-random-x"):
        b = R.make_rhs(g, a.rhs_mode.replace("-", "_"), seed)
    else:
        _parse_fail(f'unknown rhs mode "{a.rhs_mode}" (random-projected|from-random-x)')
    x, rep = R.pcg_solve_gpu(g, f, b, R.SolveConfig(tol=a.tol, max_iters=a.max_iters), ctx=ctx)
    if a.solution:
        R.write_vector(a.solution, x)
    emit_json({"config": provenance(a.input or a.gen, a.ordering, a.backend, a.workers, seed), "tol": a.tol,
               "max_iters": a.max_iters, "iterations": rep.iterations,
               "relative_residual": rep.relative_residual, "recurrence_residual": rep.recurrence_residual,
               "converged": bool(rep.converged), "factor_seconds": factor_seconds,
               "solve_seconds": rep.solve_seconds}, a.report)
    return 0 if rep.converged else 3


def _split(text: str, sep: str = ",") -> List[str]:
    return [s for s in text.split(sep) if s] if text else []


def cmd_bench(a, ctx) -> int:
    """cmd_bench (parac_cli.cpp:325-444) for the gpu backend."""
    graphs = [(p, R.read_laplacian(p)) for p in _split(a.inputs)]
    graphs += [(spec, parse_gen_spec(spec)) for spec in _split(a.gens, ";")]
    if not graphs:
        _parse_fail("bench needs --inputs or --gens")
    workers = [int(w) for w in _split(a.workers)] or [1]
    seeds = [int(s) for s in _split(a.seeds)] or [0]
    cells = []
    for name, g in graphs:
        for okind in _split(a.orderings):
            for backend in _split(a.backends):
                for w in workers[:1]:  # the device backend has no worker count (like seq/exact)
                    for seed in seeds:
                        c = {"input": name, "ordering": okind, "backend": backend, "workers": 1, "seed": seed,
                             "factor_seconds": 0.0, "solve_seconds": 0.0, "iterations": 0, "residual": 0.0,
                             "converged": False, "nnz_g": 0, "fill": 0.0, "depth": 0, "checksum": 0, "error": ""}
                        try:
                            o = make_ordering(g, okind, seed, ctx)
                            times = []
                            for rep in range(max(a.repeats, 1)):
                                f, st = run_factor(g, o, backend, seed, ctx)
                                times.append(st.seconds)
                                if rep == 0:
                                    c["nnz_g"] = f.nnz()
                                    c["fill"] = fill_ratio(g, f)
                                    c["depth"] = R.schedule_levels_gpu(f, ctx=ctx)[1]
                                    c["checksum"] = f.checksum()
                                    if a.solve:
                                        b = R.make_rhs(g, "random_projected", seed)
                                        _, r = R.pcg_solve_gpu(g, f, b, R.SolveConfig(a.tol, a.max_iters), ctx=ctx)
                                        c.update(iterations=r.iterations, residual=r.relative_residual,
                                                 converged=bool(r.converged), solve_seconds=r.solve_seconds)
                            c["factor_seconds"] = float(np.median(times))
                        except R.Error as e:
                            c["error"] = _errc_name(int(e.code))
                        except CliError as e:
                            c["error"] = _errc_name(e.code)
                        cells.append(c)
    base = {}
    for c in cells:
        if c["workers"] == 1 and not c["error"]:
            base[(c["input"], c["ordering"], c["backend"], c["seed"])] = c["factor_seconds"]
    out = ["schema,input,ordering,backend,workers,seed,factor_seconds,solve_seconds,iterations,"
           "relative_residual,converged,nnz_g,fill_ratio,schedule_depth,checksum,speedup_vs_w1,error\n"]
    for c in cells:
        b = base.get((c["input"], c["ordering"], c["backend"], c["seed"]))
        speed = _g(b / c["factor_seconds"]) if (b is not None and c["factor_seconds"] > 0 and not c["error"]) else ""
        out.append(",".join([BENCH_SCHEMA, _csv_field(c["input"]), c["ordering"], c["backend"], str(c["workers"]),
                             str(c["seed"]), _g(c["factor_seconds"]), _g(c["solve_seconds"]), str(c["iterations"]),
                             _g(c["residual"]), "1" if c["converged"] else "0", str(c["nnz_g"]), _g(c["fill"]),
                             str(c["depth"]), str(c["checksum"]), speed, c["error"]]) + "\n")
    emit_text("".join(out), a.csv)
    return 0


def _errc_name(code: int) -> str:
    return R.lib.parac_errc_name(code).decode()


# -------------------------------------------------------------------- main
def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="parac-gpu", description="parac CLI with the B200 backend")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p, backend=True):
        p.add_argument("--input", default="")
        p.add_argument("--gen", default="")
        p.add_argument("--seed", type=int, default=None)
        if backend:
            p.add_argument("--ordering", default="natural")
            p.add_argument("--backend", default="gpu")
            p.add_argument("--workers", type=int, default=1)

    g = sub.add_parser("gen", help="generate a test matrix and write it")
    common(g, backend=False)
    g.add_argument("--output", default="laplacian.mtx")
    f = sub.add_parser("factor", help="build an approximate factorization")
    common(f)
    f.add_argument("--output", default="")
    f.add_argument("--stats", default="-")
    f.add_argument("--trace", default="")
    f.add_argument("--trace-times", action="store_true")
    s = sub.add_parser("solve", help="solve L x = b with PCG")
    common(s)
    s.add_argument("--factor", default="")
    s.add_argument("--perm", default="")
    s.add_argument("--rhs", default="")
    s.add_argument("--rhs-mode", default="random-projected")
    s.add_argument("--tol", type=float, default=1e-6)
    s.add_argument("--max-iters", type=int, default=1000)
    s.add_argument("--report", default="-")
    s.add_argument("--solution", default="")
    b = sub.add_parser("bench", help="factor/solve timing matrix")
    b.add_argument("--inputs", default="")
    b.add_argument("--gens", default="")
    b.add_argument("--orderings", default="natural")
    b.add_argument("--backends", default="gpu")
    b.add_argument("--workers", default="1")
    b.add_argument("--seeds", default="0")
    b.add_argument("--repeats", type=int, default=1)
    b.add_argument("--tol", type=float, default=1e-6)
    b.add_argument("--max-iters", type=int, default=1000)
    b.add_argument("--solve", action="store_true")
    b.add_argument("--csv", default="-")
    return ap


def main(argv=None) -> int:
    a = build_parser().parse_args(argv)
    try:
        if a.cmd == "gen":
            return cmd_gen(a)
        if a.cmd in ("factor", "solve") and a.backend != "gpu" and not (a.cmd == "solve" and a.factor):
            run_factor(None, None, a.backend, 0, None)  # the reference's unknown-backend parse error
        ctx = R.default_context()
        return {"factor": cmd_factor, "solve": cmd_solve, "bench": cmd_bench}[a.cmd](a, ctx)
    except CliError as e:
        sys.stderr.write(f"error: {_errc_name(e.code)}: {e}\n")
        return 10 + e.code
    except R.Error as e:
        sys.stderr.write(f"error: {e}\n")
        return 10 + int(e.code)


if __name__ == "__main__":
    sys.exit(main())
