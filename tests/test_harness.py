"""Benchmark harness host logic (fit, records) -- CPU."""

import numpy as np
import pytest

from paper_2403_04578_b200.harness import (BenchConfig, BenchRecord, fit_complexity, read_bench_records,
                                           write_bench_records)


def _recs(k=1.5, c=2e-3, var="tau"):
    out = []
    for n in (10, 100, 1000, 10000):
        t = c * n ** k
        out.append(BenchRecord("dense", 100 if var == "tau" else n, n if var == "tau" else 10, t, 5, 3))
    return out


def test_fit_recovers_exponent():
    f = fit_complexity(_recs(), "tau")
    assert abs(f.k - 1.5) < 1e-12 and abs(f.c - 2e-3) < 1e-12 and f.r_squared == pytest.approx(1.0)
    f = fit_complexity(_recs(k=2.0, var="b_phi"), "b_phi")
    assert abs(f.k - 2.0) < 1e-12


def test_fit_rejects_mixed_and_short():
    r = _recs()
    with pytest.raises(ValueError, match="mixes methods"):
        fit_complexity(r + [BenchRecord("sparse", 100, 5, 1.0, 3, 3)], "tau")
    with pytest.raises(ValueError, match="fixed b_phi"):
        fit_complexity(r + [BenchRecord("dense", 7, 5, 1.0, 3, 3)], "tau")
    with pytest.raises(ValueError, match="at least 3"):
        fit_complexity(r[:2], "tau")
    with pytest.warns(UserWarning, match="excluding"):
        fit_complexity(r + [BenchRecord("dense", 100, 7, float("nan"), 0, 0, "TimeoutError: x")], "tau")


def test_records_roundtrip_and_reference_format(tmp_path):
    r = _recs() + [BenchRecord("sparse", 9, 1, float("nan"), 0, 2, "RuntimeError: a, b")]
    write_bench_records(tmp_path / "r.csv", r)
    lines = (tmp_path / "r.csv").read_text().splitlines()
    assert lines[0] == "method,b_phi,tau,wall_seconds,iterations,repeats,error"
    assert lines[-1] == "sparse,9,1,nan,0,2,RuntimeError: a; b"
    back = read_bench_records(tmp_path / "r.csv")
    assert back[0] == r[0] and back[-1].error == "RuntimeError: a; b"


def test_config_validation():
    with pytest.raises(ValueError, match="unknown methods"):
        BenchConfig(methods=("fpi",))
    with pytest.raises(ValueError):
        BenchConfig(sizes=())
