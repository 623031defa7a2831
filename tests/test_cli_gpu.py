"""`python -m paper_2403_04578_b200 solve` against the reference CLI's own output
(tests/golden/fileio, written by tests/golden/make_golden_fileio.py)."""

import json
import os

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fileio")
REF_KEYS = {"method", "n_demand", "tau", "iterations", "converged_cases", "nonconverged_cases", "max_residual",
            "tolerance", "wall_seconds"}


def fx(name):
    return os.path.join(FIX, name)


def table(path):
    lines = open(path).read().splitlines()
    rows = [ln.split(",") for ln in lines[1:]]
    vals = np.array([[float(c) for c in r[:-1]] for r in rows])
    return lines[0], vals, [r[-1] for r in rows]


@pytest.mark.parametrize("method", ["dense", "sparse"])
def test_solve_matches_reference_cli(tmp_path, method):
    from paper_2403_04578_b200.cli import main
    out = tmp_path / "v.csv"
    assert main(["solve", "--network", fx("net9.json"), "--loads", fx("loads9.csv"), "--method", method,
                 "--out", str(out)]) == 0
    h, v, f = table(out)
    rh, rv, rf = table(fx(f"v9_{method}.csv"))
    assert h == rh and f == rf
    assert np.abs(v - rv).max() <= 1e-9  # per-case freeze vs joint stop
    meta = json.loads((tmp_path / "v.csv.meta.json").read_text())
    ref = json.loads(open(fx(f"v9_{method}.csv.meta.json")).read())
    assert REF_KEYS <= set(meta)
    for k in ("method", "n_demand", "tau", "iterations", "converged_cases", "nonconverged_cases", "tolerance"):
        assert meta[k] == ref[k], k
    # identical invocations -> byte-identical data files
    out2 = tmp_path / "v2.csv"
    main(["solve", "--network", fx("net9.json"), "--loads", fx("loads9.csv"), "--method", method, "--out", str(out2)])
    assert out.read_bytes() == out2.read_bytes()


def test_nonconvergence_is_data(tmp_path):
    from paper_2403_04578_b200.cli import main
    out = tmp_path / "v.csv"
    assert main(["solve", "--network", fx("net9.json"), "--loads", fx("heavy9.csv"), "--out", str(out)]) == 0
    _, v, f = table(out)
    _, rv, rf = table(fx("heavy9_dense.csv"))
    assert f == rf == ["1", "0"]
    assert np.abs(v[0] - rv[0]).max() <= 1e-9
    meta = json.loads((tmp_path / "v.csv.meta.json").read_text())
    assert meta["nonconverged_cases"] == [1] and meta["converged_cases"] == 1


def test_solve_devices_and_c64_flags(tmp_path):
    from paper_2403_04578_b200.cli import main
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    assert main(["solve", "--network", fx("net9.json"), "--loads", fx("loads9.csv"), "--out", str(a)]) == 0
    assert main(["solve", "--network", fx("net9.json"), "--loads", fx("loads9.csv"), "--out", str(b),
                 "--devices", "0,0"]) == 0
    assert a.read_bytes() == b.read_bytes()
    c = tmp_path / "c.csv"
    assert main(["solve", "--network", fx("net9.json"), "--loads", fx("loads9.csv"), "--out", str(c),
                 "--dtype", "complex64", "--tol", "1e-6"]) == 0
    _, v, _ = table(c)
    _, rv, _ = table(fx("v9_dense.csv"))
    # c64 north-star bar: |V_c64 - V_ref| <= 1e-5 p.u. (V rebuilt from the |V|, angle columns)
    cv = v[:, 0::2] * np.exp(1j * v[:, 1::2])
    crv = rv[:, 0::2] * np.exp(1j * rv[:, 1::2])
    assert np.abs(cv - crv).max() <= 1e-5


def test_bench_and_fit_subcommands(tmp_path, capsys):
    from paper_2403_04578_b200.cli import main
    out = tmp_path / "r.csv"
    assert main(["bench", "--methods", "dense,sparse", "--sizes", "9", "--taus", "10,100,1000", "--repeats", "2",
                 "--out", str(out)]) == 0
    meta = json.loads((tmp_path / "r.csv.meta.json").read_text())
    assert meta["failed_cells"] == 0 and len(meta["roofline"]) == 6
    assert main(["fit", "--records", str(out), "--variable", "tau", "--method", "dense"]) == 0
    assert "t = " in capsys.readouterr().out
