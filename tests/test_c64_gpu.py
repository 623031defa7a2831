"""complex64 twins: FP32 dense and sparse kernels against the float64 oracle.

The reference has no complex64 path; the c64 bar is the north star's
(BASELINE.json): max |V_c64 - V_ref| <= 1e-5 p.u., where V_ref is the
reference's complex128 solution at its default tol = 1e-10 (the float64 oracle,
pinned to the reference by tests/golden).  The twins run at tol = 1e-6 (FP32
cannot resolve 1e-10); every case converges and per-case counts are within
one of the float64 per-case restatement at that same tolerance.  Measured on
the full C2 batch (b=100, tau=525,600, tools/c64_err_probe.py,
profiles/r2_c64_parity.json): max |dV| = 9.2e-7 dense, 4.5e-7 sparse.  The
residual post-check multiplies V by Y_dd (|Y| ~ 1/z ~ 1e3 on these feeders),
so FP32 solutions have residuals ~1e-4: the c64 residual tolerance is 1e-3.
"""

import numpy as np
import pytest

from conftest import gpu_available

from oracle import tpf_oracle as orc

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

TOL, RTOL = 1e-6, 1e-3
PARITY = 1e-5  # north-star c64 bar against the complex128 solution at tol 1e-10


def _ref(model, S):
    """The reference's converged complex128 values (oracle at the default tol = 1e-10)."""
    V, _, _, _ = orc.dense_per_case(model.admittance.y_dd, model.source_injection(), model.slack.v_s, S)
    return V


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
    assert np.abs(out.values.astype(np.complex128) - _ref(model, loads.values)).max() <= PARITY
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
        assert np.abs(out.values.astype(np.complex128) - _ref(model, loads.values)).max() <= PARITY


def test_c64_full_c2_parity_bar():
    """Full C2 (b=100, tau=525,600): every complex64 value within 1e-5 p.u. of the
    complex128 engine at tol 1e-10 (bit-pinned to the reference on the goldens), and
    a 300-column sample within 1e-5 of the float64 oracle itself."""
    import torch
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator, SparseOperator
    spec = GenSpec(n_buses=101, seed=0)
    model = build_network(spec)
    S_h = gen_scenarios(model, 525600, spec).values
    S = torch.from_numpy(S_h).cuda()
    ref, _ = DenseOperator(model).solve(S)
    S32 = S.to(torch.complex64)
    cols = np.random.default_rng(1).choice(525600, 300, replace=False)
    Vo = _ref(model, S_h[:, cols])
    for op, n in ((DenseOperator(model, dtype=np.complex64), 525600),
                  (SparseOperator(model, dtype=np.complex64), 65536)):
        V, it = op.solve(S32[:, :n], _opts())
        assert int(it.max()) < 100
        err = (V.to(torch.complex128) - ref[:, :n]).abs().max().item()
        assert err <= PARITY, err
        c = cols[cols < n]
        Vg = V[:, torch.from_numpy(c).cuda()].cpu().numpy().astype(np.complex128)
        assert np.abs(Vg - Vo[:, cols < n]).max() <= PARITY
