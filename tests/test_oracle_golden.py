"""Pin the CPU oracle (oracle/tpf_oracle.py) to the reference's own outputs.

The golden files were produced by running the reference `tpflow` (see
tests/golden/make_golden.py); these tests run anywhere (no reference, no GPU).
"""

import numpy as np
import pytest

from conftest import golden_names
from oracle import tpf_oracle as orc

DENSE = [n for n in golden_names() if n not in ("c3_slice6",)]
SPARSE = [n for n in golden_names() if n not in ("c5_slice32",)]


@pytest.mark.parametrize("name", DENSE)
def test_dense_joint_matches_reference(golden, name):
    g = golden(name)
    y, src, v_s = g.args
    o = g.opts()
    V, n, mask, res = orc.dense_joint(y, src, v_s, g.S, o.tolerance, o.max_iterations,
                                      o.residual_tolerance)
    assert n == int(g["dense_iterations"])
    assert np.array_equal(mask, g["dense_mask"])
    good = g["dense_mask"]
    assert np.abs(V[:, good] - g["dense_V"][:, good]).max(initial=0.0) < 1e-12
    fin = np.isfinite(g["dense_residuals"])
    assert np.allclose(res[fin], g["dense_residuals"][fin], rtol=1e-6, atol=1e-15)


@pytest.mark.parametrize("name", DENSE)
def test_per_case_freeze_matches_joint_count(golden, name):
    """max_j n_j == the reference's joint count; values within 1e-9."""
    g = golden(name)
    y, src, v_s = g.args
    o = g.opts()
    V, n_case, mask, res = orc.dense_per_case(y, src, v_s, g.S, o.tolerance, o.max_iterations,
                                              o.residual_tolerance)
    assert int(n_case.max()) == int(g["dense_iterations"])
    assert np.array_equal(mask, g["dense_mask"])
    good = g["dense_mask"]
    assert np.abs(V[:, good] - g["dense_V"][:, good]).max(initial=0.0) < 1e-9
    if "fpi_iterations" in g:
        # per-case counts equal the reference single-case solver's (fpi.py:134-206)
        assert np.abs(n_case - g["fpi_iterations"]).max() <= 1
        assert np.mean(n_case == g["fpi_iterations"]) > 0.99
        assert np.abs(V[:, good] - g["fpi_V"][:, good]).max(initial=0.0) < 1e-10


@pytest.mark.parametrize("name", SPARSE)
def test_sparse_block_matches_reference(golden, name):
    g = golden(name)
    if g.S.shape[0] * g.S.shape[1] > 40000:
        pytest.skip("block-diagonal SuperLU restatement kept to small batches in the CPU suite")
    y, src, v_s = g.args
    o = g.opts()
    V, n, mask, res = orc.sparse_block(y, src, v_s, g.S, o.tolerance, o.max_iterations,
                                       o.residual_tolerance)
    assert n == int(g["sparse_iterations"])
    assert np.array_equal(mask, g["sparse_mask"])
    good = g["sparse_mask"]
    assert np.abs(V[:, good] - g["sparse_V"][:, good]).max(initial=0.0) < 1e-12


def test_two_bus_known_answer(golden):
    g = golden("twobus_known")
    v_high = (1 + np.sqrt(0.96)) / 2
    assert abs(g["dense_V"][0, 0] - v_high) < 1e-12
    y, src, v_s = g.args
    V, _, _, _ = orc.dense_per_case(y, src, v_s, g.S)
    assert abs(V[0, 0] - v_high) < 1e-12


def test_c2_statistics_recorded(golden):
    """Survey probe: C2 per-case counts sum to 2,615,281 with max 7."""
    g = golden("c2_slice192")
    assert int(g["c2_sum_n"]) == 2615281
    assert int(g["c2_max_n"]) == 7


@pytest.mark.parametrize("name", ["zip9_mixed", "zip9_heavy", "zip9_pure_zi", "zip101_mixed", "zip9_mesh",
                                  "zip101_mesh"])
def test_zip_oracle_matches_reference(name):
    """The ZIP restatement (per-case fpi_solve) against the reference's own batch."""
    import os
    from scipy import sparse as sp
    d = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "zip", name + ".npz"))
    b = d["S"].shape[0]
    y = sp.csc_matrix((d["ydd_data"], d["ydd_indices"], d["ydd_indptr"]), shape=(b, b))
    V, n, mask, res, it = orc.dense_zip_batch(y, d["src"], 1.0 + 0j, d["alpha_z"], d["alpha_i"], d["alpha_p"],
                                              d["S"], float(d["tol"]), int(d["max_iter"]), float(d["residual_tol"]))
    assert it == int(d["iterations"])
    assert np.array_equal(n, d["n_case"])
    assert np.array_equal(mask, d["mask"])
    good = d["mask"]
    assert np.abs(V[:, good] - d["V"][:, good]).max(initial=0) <= 1e-12
