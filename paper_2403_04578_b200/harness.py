"""Benchmark harness and complexity fit over the GPU methods (SURVEY.md 8(f)
item 3), mirroring the reference's bench.py:38-222 and its record file
(fileio.py:260-300):

* ``run_benchmark(BenchConfig)`` times every (size, tau, method) cell on
  freshly generated inputs (``GenSpec(b_phi + 1, seed + b_phi)``), median of
  the timed repeats after the warm-up, per-method setup included, file I/O
  and generation excluded (bench.py:120-176); a failing or overlong cell is
  recorded with an error and the sweep continues;
* ``fit_complexity`` fits t = c * n^k over records that vary one variable
  (bench.py:179-222);
* records are written / read in the reference's 7-column CSV, so either
  package's ``fit`` reads the other's files.

Each cell also carries the roofline figures of SURVEY 8(d) (``RooflineCell``:
per-case iteration sum, algorithmic work, achieved rate over the cell's wall
time), written to the metadata document next to the records.
"""

from __future__ import annotations

import statistics
import time
import warnings
from dataclasses import asdict, dataclass, field
from pathlib import Path

import numpy as np

from ._types import SolveOptions
from .dispatch import solve_batch
from .synth import GenSpec, build_network, gen_scenarios

__all__ = ["METHODS", "BenchRecord", "BenchConfig", "RooflineCell", "ComplexityFit", "run_benchmark",
           "fit_complexity", "write_bench_records", "read_bench_records"]

METHODS = ("dense", "sparse")  # the accelerated methods; fpi / nr stay in the reference


@dataclass(frozen=True)
class BenchRecord:
    """One timed benchmark cell (bench.py:38-51)."""

    method: str
    b_phi: int
    tau: int
    wall_seconds: float
    iterations: int
    repeats: int
    error: str | None = None

    @property
    def ok(self) -> bool:
        return self.error is None


@dataclass(frozen=True)
class RooflineCell:
    """SURVEY 8(d) work of one cell: dense 8 b^2 sum_j n_j flop, sparse
    48 b sum_j n_j bytes, and that work over the cell's median wall time."""

    method: str
    b_phi: int
    tau: int
    sum_iterations: int
    work: float
    unit: str
    achieved: float


@dataclass(frozen=True)
class BenchConfig:
    """bench.py:54-74."""

    methods: tuple[str, ...] = METHODS
    sizes: tuple[int, ...] = (9, 100)
    taus: tuple[int, ...] = (1, 100)
    seed: int = 0
    repeats: int = 3
    warmup: int = 1
    timeout: float = 300.0
    options: SolveOptions = field(default_factory=SolveOptions)
    device: object = None

    def __post_init__(self) -> None:
        if not (self.methods and self.sizes and self.taus):
            raise ValueError("methods, sizes and taus must be non-empty")
        unknown = set(self.methods) - set(METHODS)
        if unknown:
            raise ValueError(f"unknown methods {sorted(unknown)}")
        if self.repeats < 1:
            raise ValueError("repeats must be >= 1")


def run_benchmark(config: BenchConfig, roofline: list | None = None) -> list[BenchRecord]:
    """Time every (size, tau, method) cell; ``roofline`` (a list) collects a
    RooflineCell per successful cell."""
    records: list[BenchRecord] = []
    for b_phi in config.sizes:
        spec = GenSpec(n_buses=b_phi + 1, seed=config.seed + b_phi)
        model = build_network(spec)
        for tau in config.taus:
            loads = gen_scenarios(model, tau, spec)
            for method in config.methods:
                rec, cell = _time_cell(method, model, loads, b_phi, tau, config)
                records.append(rec)
                if roofline is not None and cell is not None:
                    roofline.append(cell)
    return records


def _time_cell(method, model, loads, b_phi, tau, config):
    times: list[float] = []
    iterations = 0
    out = None
    try:
        for rep in range(config.warmup + config.repeats):
            t0 = time.perf_counter()
            out = solve_batch(method, model, loads, config.options, device=config.device)
            iterations = out.iterations
            dt = time.perf_counter() - t0
            if rep >= config.warmup:
                times.append(dt)
            if dt > config.timeout:
                raise TimeoutError(f"cell exceeded the {config.timeout:.0f}s timeout")
    except Exception as exc:  # per-cell failures must not stop the sweep
        return BenchRecord(method=method, b_phi=b_phi, tau=tau, wall_seconds=float("nan"), iterations=0,
                           repeats=len(times), error=f"{type(exc).__name__}: {exc}"), None
    wall = statistics.median(times)
    b = model.n_demand
    sum_n = int(np.asarray(out.iterations_per_case, dtype=np.int64).sum())
    work, unit, scale = ((8.0 * b * b * sum_n, "GFLOP/s", 1e9) if method == "dense"
                         else (48.0 * b * sum_n, "GB/s", 1e9))
    cell = RooflineCell(method=method, b_phi=b_phi, tau=tau, sum_iterations=sum_n, work=work, unit=unit,
                        achieved=work / wall / scale)
    return BenchRecord(method=method, b_phi=b_phi, tau=tau, wall_seconds=wall, iterations=iterations,
                       repeats=len(times)), cell


@dataclass(frozen=True)
class ComplexityFit:
    """Least-squares fit of log t = log c + k log n (bench.py:168-176)."""

    c: float
    k: float
    r_squared: float
    variable: str
    n_points: int


def fit_complexity(records: list[BenchRecord], variable: str, min_points: int = 3) -> ComplexityFit:
    """Fit t = c * n^k over records varying only ``variable`` ("tau" or "b_phi")."""
    if variable not in ("tau", "b_phi"):
        raise ValueError("variable must be 'tau' or 'b_phi'")
    usable = []
    for rec in records:
        if not rec.ok or not np.isfinite(rec.wall_seconds) or rec.wall_seconds <= 0:
            warnings.warn(f"excluding unusable record {rec.method} b_phi={rec.b_phi} tau={rec.tau} "
                          f"({rec.error or 'nonpositive time'})", stacklevel=2)
            continue
        usable.append(rec)
    if len({r.method for r in usable}) > 1:
        raise ValueError("fit mixes methods; filter the records first")
    other = "b_phi" if variable == "tau" else "tau"
    if len({getattr(r, other) for r in usable}) > 1:
        raise ValueError(f"fit requires a fixed {other}; filter the records first")
    n = np.array([getattr(r, variable) for r in usable], dtype=float)
    t = np.array([r.wall_seconds for r in usable])
    if len(usable) < min_points or len(np.unique(n)) < min_points:
        raise ValueError(f"need at least {min_points} distinct {variable} values, got {len(np.unique(n))}")
    log_n, log_t = np.log(n), np.log(t)
    k, log_c = np.polyfit(log_n, log_t, 1)
    pred = k * log_n + log_c
    ss_res = float(np.sum((log_t - pred) ** 2))
    ss_tot = float(np.sum((log_t - log_t.mean()) ** 2))
    return ComplexityFit(c=float(np.exp(log_c)), k=float(k), r_squared=1.0 - ss_res / ss_tot if ss_tot > 0 else 1.0,
                         variable=variable, n_points=len(usable))


_HEADER = "method,b_phi,tau,wall_seconds,iterations,repeats,error"


def write_bench_records(path, records) -> None:
    """The reference's record table (fileio.py:260-268)."""
    with open(path, "w") as fh:
        fh.write(_HEADER + "\n")
        for r in records:
            err = (r.error or "").replace(",", ";")
            fh.write(f"{r.method},{r.b_phi},{r.tau},{r.wall_seconds:.17g},{r.iterations},{r.repeats},{err}\n")


def read_bench_records(path) -> list[BenchRecord]:
    """fileio.py:271-300."""
    from .fileio import FileFormatError
    path = Path(path)
    if not path.exists():
        raise FileFormatError(f"{path}: no such file")
    records = []
    with open(path) as fh:
        header = fh.readline().strip()
        if header != _HEADER:
            raise FileFormatError(f"{path}: unexpected header {header!r}")
        for lineno, line in enumerate(fh, start=2):
            line = line.strip()
            if not line:
                continue
            parts = line.split(",")
            if len(parts) != 7:
                raise FileFormatError(f"{path}: line {lineno}: expected 7 fields, got {len(parts)}")
            try:
                records.append(BenchRecord(method=parts[0], b_phi=int(parts[1]), tau=int(parts[2]),
                                           wall_seconds=float(parts[3]), iterations=int(parts[4]),
                                           repeats=int(parts[5]), error=parts[6] or None))
            except ValueError as exc:
                raise FileFormatError(f"{path}: line {lineno}: {exc}") from exc
    return records


def roofline_meta(cells: list[RooflineCell]) -> list[dict]:
    return [asdict(c) for c in cells]
