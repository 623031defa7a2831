"""complex64 twins: FP32 dense and sparse kernels against the float64 oracle.

The reference has no complex64 path; the c64 bar is FP32 accuracy: with
tol = 1e-6 every case converges, per-case counts are within one of the
float64 per-case restatement at the same tolerance, and values agree to 2e-5
p.u. (a few hundred FP32 ulps of |v| ~ 1 after ~5 iterations of a 100-term
complex sum).  The residual post-check multiplies V by Y_dd (|Y| ~ 1/z ~ 1e3
on these feeders), so FP32 solutions have residuals ~1e-4: the c64 residual
tolerance is 1e-3.
"""

import numpy as np
import pytest

from conftest import gpu_available

from oracle import tpf_oracle as orc

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

TOL, RTOL = 1e-6, 1e-3


def _opts():
    from paper_2403_04578_b200 import SolveOptions
    return SolveOptions(tolerance=TOL, max_iterations=100, residual_tolerance=RTOL)


def _case(n_buses, tau, seed=0):
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios
    spec = GenSpec(n_buses=n_buses, seed=seed)
    model = build_network(spec)
    return model, gen_scenarios(model, tau, spec)


@pytest.mark.parametrize("method", ["dense", "sparse"])
@pytest.mark.parametrize("n_buses,tau", [(2, 50), (35, 700), (101, 600)])
def test_c64_matches_float64_oracle(method, n_buses, tau):
    from paper_2403_04578_b200 import solve_batch
    model, loads = _case(n_buses, tau)
    out = solve_batch(method, model, loads, _opts(), dtype=np.complex64)
    assert out.values.dtype == np.complex64
    V, n, mask, _ = orc.dense_per_case(model.admittance.y_dd, model.source_injection(), model.slack.v_s,
                                       loads.values, tol=TOL, residual_tol=RTOL)
    assert mask.all()
    assert out.converged_mask.all(), out.residuals.max()
    assert np.abs(out.iterations_per_case.astype(int) - n).max() <= 1
    assert out.iterations <= n.max() + 1
    assert np.abs(out.values.astype(np.complex128) - V).max() < 2e-5
    assert np.isfinite(out.residuals).all() and out.residuals.max() < RTOL


def test_c64_device_path_and_nan_case():
    import torch
    from paper_2403_04578_b200 import batch_solve_dense, LoadMatrix
    model, loads = _case(35, 200)
    S = loads.values.copy()
    S[3, 7] = np.nan
    out = batch_solve_dense(model, LoadMatrix(S), _opts(), dtype=np.complex64, return_on_device=True)
    assert out.values.dtype == torch.complex64 and out.values.is_cuda
    it = out.iterations_per_case.cpu().numpy()
    mask = out.converged_mask.cpu().numpy()
    assert it[7] == 100 and not mask[7]
    assert mask[np.arange(200) != 7].all()


def test_c64_dense_large_b_is_unsupported():
    from paper_2403_04578_b200 import batch_solve_dense
    model, loads = _case(106, 20)
    with pytest.raises(NotImplementedError):
        batch_solve_dense(model, loads, _opts(), dtype=np.complex64)


@pytest.mark.parametrize("method", ["dense", "sparse"])
def test_c64_array_passthrough_same_bits(method):
    """A complex64 array handed to the c64 twin is used as is; same bits as the
    LoadMatrix (complex128) route, whose values round to the same complex64."""
    from paper_2403_04578_b200 import batch_solve_dense, batch_solve_sparse, LoadMatrix
    solver = batch_solve_dense if method == "dense" else batch_solve_sparse
    model, loads = _case(101, 900)
    a = solver(model, LoadMatrix(loads.values), _opts(), dtype=np.complex64)
    b = solver(model, loads.values.astype(np.complex64), _opts(), dtype=np.complex64)
    assert a.values.dtype == b.values.dtype == np.complex64
    assert np.array_equal(a.values, b.values) and np.array_equal(a.iterations_per_case, b.iterations_per_case)
    assert np.array_equal(a.converged_mask, b.converged_mask) and a.iterations == b.iterations


def test_c64_quarter_kernel_node_counts():
    """Every quarter width of the default c64 kernel (b <= 32, 40, 56, 80, 104) and
    an empty last quarter (b = 5: quarters of 8 nodes)."""
    from paper_2403_04578_b200 import solve_batch
    for n_buses in (6, 33, 41, 57, 81, 105):
        model, loads = _case(n_buses, 300, seed=n_buses)
        out = solve_batch("dense", model, loads, _opts(), dtype=np.complex64)
        V, n, mask, _ = orc.dense_per_case(model.admittance.y_dd, model.source_injection(), model.slack.v_s,
                                           loads.values, tol=TOL, residual_tol=RTOL)
        assert out.converged_mask.all()
        assert np.abs(out.iterations_per_case.astype(int) - n).max() <= 1
        assert np.abs(out.values.astype(np.complex128) - V).max() < 2e-5
