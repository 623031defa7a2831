"""The C-ABI library loads and exports every entry point include/tpf.h declares.

No compute calls here (no GPU in the build container)."""

import os
import re

import pytest

from conftest import ROOT
from paper_2403_04578_b200 import _capi


def declared():
    txt = open(os.path.join(ROOT, "include", "tpf.h")).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(tpf_\w+)\s*\(", txt, flags=re.M)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("tpf_dense_fpi_c128", "tpf_sparse_fpi_c128", "tpf_residual_c128",
                 "tpf_batch_summary", "tpf_last_error", "tpf_version"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _capi.load()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    assert set(declared()) <= set(_capi.SIGNATURES)


def test_version_and_error_string():
    lib = _capi.load()
    assert lib.tpf_version() >= 100
    assert isinstance(lib.tpf_last_error(), bytes)


def test_invalid_arguments_fail_without_touching_the_gpu():
    lib = _capi.load()
    rc = lib.tpf_dense_fpi_c128(10, 0, None, 0, 0, None, None, 1.0, 0.0, 1e-10, 100,
                                None, 0, 0, None, None, 0, None)
    assert rc == _capi.TPF_ERR_INVALID
    assert b"b >= 1" in lib.tpf_last_error()
    with pytest.raises(ValueError):
        _capi.check(rc)
    rc = lib.tpf_dense_fpi_c128(10, 200, None, 0, 0, None, None, 1.0, 0.0, 1e-10, 100,
                                None, 0, 0, None, None, 0, None)
    assert rc == _capi.TPF_ERR_UNSUPPORTED
