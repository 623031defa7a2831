"""Command-line front end mirroring the reference's ``tpflow`` CLI (cli.py).

    python -m paper_2403_04578_b200 solve --network NET.json --loads LOADS.csv --out V.csv \
        [--method dense|sparse] [--tol 1e-10] [--max-iter 100] [--threads N] [--meta M.json] \
        [--devices 0,1,...] [--dtype complex128|complex64]
    python -m paper_2403_04578_b200 gen-net --buses N [--kmax 5] [--seed 0] ... --out NET.json
    python -m paper_2403_04578_b200 gen-loads --network NET.json --tau T [--seed 0] [--scale 1]
        [--correlation 0.5] --out LOADS.csv
    python -m paper_2403_04578_b200 bench [--methods dense,sparse] [--sizes 9,100] [--taus 1,100] --out R.csv
    python -m paper_2403_04578_b200 fit --records R.csv --variable tau|b_phi [--method dense]

``solve`` runs the GPU engine (cli.py:54-76 semantics: same metadata keys,
non-convergence is data, exit 1 with ``error: ...`` on FileFormatError /
NetworkError / ValueError / MemoryError, cli.py:315-317); ``gen-net`` and
``gen-loads`` are the reference's seeded generators (bit-identical networks and
loads, cli.py:79-95).  Tables are read and written by the native file layer
(fileio.py in this package); identical invocations produce byte-identical
data files.  ``bench`` / ``fit`` are the reference's harness (bench.py:120-222)
over the GPU methods, in the same record format, plus per-cell roofline
figures in the metadata.  The reference's twobus subcommands are outside the
accelerated path.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

from . import fileio
from ._types import SolveOptions
from .dispatch import solve_batch
from .fileio import FileFormatError
from .network import NetworkError
from .synth import GenSpec, build_network, gen_scenarios

__all__ = ["main", "build_parser"]


def _threads(args) -> int:
    """Host threads for the file layer (cli.py:29-38: --threads, else TPF_THREADS, else all)."""
    if args.threads is not None:
        return max(1, args.threads)
    env = os.environ.get("TPF_THREADS")
    if env:
        try:
            return max(1, int(env))
        except ValueError as exc:
            raise ValueError(f"TPF_THREADS={env!r} is not an integer") from exc
    return 0


def _warm_cuda():
    """Create the CUDA context and load libtpf.so while the tables are parsed."""
    import threading

    def work():
        try:
            import torch
            from . import _capi
            torch.empty(1, device="cuda")
            _capi.load()
        except Exception:  # the solve itself reports a missing device or library
            pass
    t = threading.Thread(target=work, daemon=True)
    t.start()
    return t


def _cmd_solve(args) -> int:
    warm = _warm_cuda()
    model = fileio.read_network(args.network)
    warm.join()
    import torch
    loads = fileio.read_loads(args.loads, threads=_threads(args), pinned=torch.cuda.is_available())
    opts = SolveOptions(tolerance=args.tol, max_iterations=args.max_iter)
    kw = {}
    if args.devices:
        kw["devices"] = [f"cuda:{d.strip()}" for d in args.devices.split(",") if d.strip()]
    if args.dtype != "complex128":
        kw["dtype"] = np.dtype(args.dtype)
    t0 = time.perf_counter()
    batch = solve_batch(args.method, model, loads, opts, **kw)
    wall = time.perf_counter() - t0
    fileio.write_voltages(args.out, batch, threads=_threads(args))
    res = np.asarray(batch.residuals, dtype=float)
    meta = {
        "method": args.method,
        "n_demand": model.n_demand,
        "tau": batch.tau,
        "iterations": batch.iterations,
        "converged_cases": int(np.asarray(batch.converged_mask).sum()),
        "nonconverged_cases": [int(j) for j in np.where(~np.asarray(batch.converged_mask))[0]],
        "max_residual": float(np.nanmax(res)) if res.size and not np.isnan(res).all() else float("nan"),
        "tolerance": opts.tolerance,
        "wall_seconds": wall,
        "engine": "paper_2403_04578_b200 (B200)",
    }
    fileio.write_metadata(args.meta or f"{args.out}.meta.json", meta)
    return 0


def _cmd_gen_net(args) -> int:
    spec = GenSpec(n_buses=args.buses, k_max=args.kmax, seed=args.seed,
                   r_range=(args.r_min, args.r_max), x_range=(args.x_min, args.x_max))
    fileio.write_network(args.out, build_network(spec))
    return 0


def _cmd_gen_loads(args) -> int:
    model = fileio.read_network(args.network)
    spec = GenSpec(n_buses=model.n_demand + 1, seed=args.seed, load_scale=args.scale,
                   correlation=args.correlation)
    fileio.write_loads(args.out, gen_scenarios(model, args.tau, spec))
    return 0


def _int_list(text: str) -> tuple[int, ...]:
    try:
        return tuple(int(x) for x in text.split(",") if x.strip())
    except ValueError as exc:
        raise ValueError(f"expected a comma-separated integer list, got {text!r}") from exc


def _cmd_bench(args) -> int:
    from .harness import BenchConfig, roofline_meta, run_benchmark, write_bench_records
    config = BenchConfig(methods=tuple(args.methods.split(",")), sizes=_int_list(args.sizes),
                         taus=_int_list(args.taus), seed=args.seed, repeats=args.repeats, timeout=args.timeout,
                         options=SolveOptions(tolerance=args.tol, max_iterations=args.max_iter))
    cells: list = []
    records = run_benchmark(config, roofline=cells)
    write_bench_records(args.out, records)
    fileio.write_metadata(args.meta or f"{args.out}.meta.json", {
        "methods": list(config.methods), "sizes": list(config.sizes), "taus": list(config.taus),
        "seed": config.seed, "repeats": config.repeats, "failed_cells": sum(not r.ok for r in records),
        "roofline": roofline_meta(cells)})
    return 0


def _cmd_fit(args) -> int:
    from .harness import fit_complexity, read_bench_records
    records = read_bench_records(args.records)
    if args.method:
        records = [r for r in records if r.method == args.method]
    fit = fit_complexity(records, args.variable)
    print(f"t = {fit.c:.6g} * {fit.variable}^{fit.k:.4f}   (R^2 = {fit.r_squared:.6f}, {fit.n_points} points)")
    if args.out:
        fileio.write_metadata(args.out, {"c": fit.c, "k": fit.k, "r_squared": fit.r_squared,
                                         "variable": fit.variable, "n_points": fit.n_points})
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2403_04578_b200",
                                     description="B200 engine for batched fixed-point power flow")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("solve", help="solve a load batch against a network")
    p.add_argument("--network", required=True)
    p.add_argument("--loads", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--meta", default=None, help="metadata path (default <out>.meta.json)")
    p.add_argument("--method", choices=("dense", "sparse"), default="dense")
    p.add_argument("--tol", type=float, default=1e-10, help="voltage step tolerance (default 1e-10)")
    p.add_argument("--max-iter", type=int, default=100, help="iteration cap (default 100)")
    p.add_argument("--threads", type=int, default=None,
                   help="host threads of the table reader/writer (default: TPF_THREADS or all)")
    p.add_argument("--devices", default=None, help="comma-separated CUDA device indices (default: current)")
    p.add_argument("--dtype", choices=("complex128", "complex64"), default="complex128")
    p.set_defaults(func=_cmd_solve)

    p = sub.add_parser("gen-net", help="generate a random radial network")
    p.add_argument("--buses", type=int, required=True)
    p.add_argument("--kmax", type=int, default=5)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--r-min", type=float, default=0.001)
    p.add_argument("--r-max", type=float, default=0.01)
    p.add_argument("--x-min", type=float, default=0.001)
    p.add_argument("--x-max", type=float, default=0.01)
    p.add_argument("--out", required=True)
    p.set_defaults(func=_cmd_gen_net)

    p = sub.add_parser("gen-loads", help="generate a load scenario batch")
    p.add_argument("--network", required=True)
    p.add_argument("--tau", type=int, required=True)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--scale", type=float, default=1.0)
    p.add_argument("--correlation", type=float, default=0.5)
    p.add_argument("--out", required=True)
    p.set_defaults(func=_cmd_gen_loads)

    p = sub.add_parser("bench", help="time (method x size x tau) cells on the GPU (bench.py:120-176)")
    p.add_argument("--methods", default="dense,sparse")
    p.add_argument("--sizes", default="9,100")
    p.add_argument("--taus", default="1,100")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--repeats", type=int, default=3)
    p.add_argument("--timeout", type=float, default=300.0, help="per-cell wall-time cutoff in seconds")
    p.add_argument("--tol", type=float, default=1e-10)
    p.add_argument("--max-iter", type=int, default=100)
    p.add_argument("--out", required=True)
    p.add_argument("--meta", default=None)
    p.set_defaults(func=_cmd_bench)

    p = sub.add_parser("fit", help="fit t = c * n^k to benchmark records")
    p.add_argument("--records", required=True)
    p.add_argument("--variable", choices=("tau", "b_phi"), required=True)
    p.add_argument("--method", default=None)
    p.add_argument("--out", default=None)
    p.set_defaults(func=_cmd_fit)
    return parser


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (FileFormatError, NetworkError, ValueError, MemoryError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
