"""File formats around the path: the native table reader
and writer against fixtures written by the reference CLI
(tests/golden/make_golden_fileio.py) and against Python's float()/format()."""

import os
import struct

import numpy as np
import pytest

from paper_2403_04578_b200 import GenSpec, LoadMatrix, VoltageBatch, build_network, gen_scenarios
from paper_2403_04578_b200 import fileio
from paper_2403_04578_b200.fileio import FileFormatError

FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fileio")


def fx(name):
    return os.path.join(FIX, name)


def test_read_network_matches_generator():
    m = fileio.read_network(fx("net9.json"))
    g = build_network(GenSpec(n_buses=9, seed=0))
    assert (m.admittance.y_dd != g.admittance.y_dd).nnz == 0
    assert np.array_equal(m.source_injection(), g.source_injection())


def test_network_roundtrip(tmp_path):
    g = build_network(GenSpec(n_buses=30, seed=4))
    fileio.write_network(tmp_path / "n.json", g)
    m = fileio.read_network(tmp_path / "n.json")
    assert (m.admittance.y_dd != g.admittance.y_dd).nnz == 0


def test_read_loads_exact_and_write_loads_reference_bytes(tmp_path):
    model = fileio.read_network(fx("net9.json"))
    ref = gen_scenarios(model, 50, GenSpec(n_buses=9, seed=3))
    got = fileio.read_loads(fx("loads9.csv"))
    assert np.array_equal(got.values, ref.values)  # 17 digits round-trip exactly
    fileio.write_loads(tmp_path / "l.csv", ref, threads=3)
    assert (tmp_path / "l.csv").read_bytes() == open(fx("loads9.csv"), "rb").read()


def test_write_voltages_reference_bytes(tmp_path):
    d = np.load(fx("v9_dense_batch.npz"))
    batch = VoltageBatch(values=d["values"], iterations=0, converged_mask=d["converged_mask"],
                         residuals=np.zeros(d["values"].shape[1]))
    for threads in (1, 4):
        fileio.write_voltages(tmp_path / "v.csv", batch, threads=threads)
        assert (tmp_path / "v.csv").read_bytes() == open(fx("v9_dense.csv"), "rb").read()


def test_cell_format_is_python_17g(tmp_path):
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2**63, size=4000, dtype=np.uint64)
    x = np.array([struct.unpack("<d", struct.pack("<Q", int(u)))[0] for u in bits])
    special = [0.0, -0.0, 1e-300, 5e-324, 1.7976931348623157e308, 0.1, 123456789012345678.0, 1e16, 1e-5,
               1e-4, np.inf, -np.inf, np.nan, -np.nan, struct.unpack("<d", struct.pack("<Q", 0xFFF8000000000001))[0]]
    x = np.concatenate([x, special])
    x = x[: x.size // 2 * 2]
    z = np.empty(x.size // 2, dtype=np.complex128)
    z.real, z.imag = x[0::2], x[1::2]
    loads = LoadMatrix(values=z.reshape(1, -1))
    # write_loads formats real, imag of each case: compare with Python's format
    fileio.write_loads(tmp_path / "f.csv", loads, threads=2)
    lines = (tmp_path / "f.csv").read_text().splitlines()[1:]
    v = loads.values[0]
    expect = [f"{z.real:.17g},{z.imag:.17g}" for z in v]
    assert lines == expect


def test_reader_whitespace_blank_lines_crlf(tmp_path):
    p = tmp_path / "l.csv"
    p.write_bytes(b"p_1,q_1,p_2,q_2\r\n 0.5 , 0.25,1e-3,-2\r\n\r\n   \n0.1,0.2,0.3,0.4\n")
    got = fileio.read_loads(p)
    ref = fileio._read_loads_python(p)
    assert np.array_equal(got.values, ref.values) and got.values.shape == (2, 2)


def test_reader_float_only_syntax_goes_to_exact_reader(tmp_path):
    p = tmp_path / "l.csv"
    p.write_text("p_1,q_1\n1_000.5,-2.5\nnan,-Infinity\n")
    got = fileio.read_loads(p)
    ref = fileio._read_loads_python(p)  # float() semantics, incl. the reference's p + 1j*q quirks
    assert got.values[0, 0] == 1000.5 - 2.5j
    assert np.array_equal(got.values, ref.values, equal_nan=True)


@pytest.mark.parametrize("text,msg", [
    ("", "empty file"),
    ("p_1,q_1,p_2\n1,2,3\n", "header must hold p_<node>,q_<node> pairs"),
    ("p_1,q_2\n1,2\n", "does not match the expected p_1,q_1,...,p_1,q_1 layout"),
    ("p_1,q_1\n", "no load cases"),
    ("p_1,q_1\n1,2\n1,2,3\n", "line 3: expected 2 fields, got 3"),
    ("p_1,q_1\n1,abc\n", "line 2: could not convert string to float: 'abc'"),
])
def test_reader_errors_match_reference(tmp_path, text, msg):
    p = tmp_path / "bad.csv"
    p.write_text(text)
    with pytest.raises(FileFormatError) as exc:
        fileio.read_loads(p)
    assert str(p) in str(exc.value) and msg in str(exc.value)


def test_missing_file(tmp_path):
    with pytest.raises(FileFormatError, match="no such file"):
        fileio.read_loads(tmp_path / "nope.csv")
    with pytest.raises(FileFormatError, match="no such file"):
        fileio.read_network(tmp_path / "nope.json")


def test_cli_generators_match_reference(tmp_path):
    from paper_2403_04578_b200.cli import main
    assert main(["gen-net", "--buses", "9", "--seed", "0", "--out", str(tmp_path / "n.json")]) == 0
    assert (tmp_path / "n.json").read_bytes() == open(fx("net9.json"), "rb").read()
    assert main(["gen-loads", "--network", fx("net9.json"), "--tau", "50", "--seed", "3",
                 "--out", str(tmp_path / "l.csv")]) == 0
    assert (tmp_path / "l.csv").read_bytes() == open(fx("loads9.csv"), "rb").read()


def test_cli_error_exit_code(tmp_path, capsys):
    from paper_2403_04578_b200.cli import main
    bad = tmp_path / "bad.csv"
    bad.write_text("p_1,q_1\n1,x\n")
    assert main(["solve", "--network", fx("net9.json"), "--loads", str(bad), "--out",
                 str(tmp_path / "v.csv")]) == 1
    err = capsys.readouterr().err
    assert err.startswith("error: ") and "line 2" in err and "bad.csv" in err


def test_native_reader_writer_ignore_lc_numeric(tmp_path):
    """Python's float()/format ignore LC_NUMERIC; so must the native table I/O
    (strtod_l / uselocale with the "C" locale).  Needs a comma-decimal locale
    installed in the image; skipped otherwise."""
    import locale
    old = locale.setlocale(locale.LC_NUMERIC)
    for name in ("de_DE.UTF-8", "de_DE.utf8", "fr_FR.UTF-8", "de_DE", "fr_FR"):
        try:
            locale.setlocale(locale.LC_NUMERIC, name)
            break
        except locale.Error:
            continue
    else:
        pytest.skip("no comma-decimal locale installed")
    try:
        assert locale.localeconv()["decimal_point"] == ","
        ref = gen_scenarios(fileio.read_network(fx("net9.json")), 50, GenSpec(n_buses=9, seed=3))
        fileio.write_loads(tmp_path / "l.csv", ref, threads=3)
        assert (tmp_path / "l.csv").read_bytes() == open(fx("loads9.csv"), "rb").read()
        assert np.array_equal(fileio.read_loads(fx("loads9.csv")).values, ref.values)
    finally:
        locale.setlocale(locale.LC_NUMERIC, old)
