"""ZIP loads on the GPU (tpf_sparse_tree_zip_fpi_c128) against fixtures written
by the reference's per-case route (tests/golden/make_golden_zip.py) and the
oracle restatement (oracle.dense_zip_batch)."""

import os

import numpy as np
import pytest

from conftest import gpu_available
from oracle import tpf_oracle as orc

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "zip")


def fixture(name):
    from paper_2403_04578_b200 import GenSpec, NetworkModel, ZipCoefficients, build_network
    d = np.load(os.path.join(DIR, name + ".npz"))
    base = build_network(GenSpec(n_buses=int(d["n_buses"]), seed=int(d["seed"])))
    z = ZipCoefficients(alpha_z=d["alpha_z"], alpha_i=d["alpha_i"], alpha_p=d["alpha_p"])
    if "_mesh" in name:  # tie branches: the fixture's own Y_dd and source injection
        from scipy import sparse as sp
        b = d["S"].shape[0]
        y = sp.csc_matrix((d["ydd_data"], d["ydd_indices"], d["ydd_indptr"]), shape=(b, b))
        y_ds = sp.csc_matrix(np.asarray(d["src"]).reshape(b, 1) / base.slack.v_s)
        model = NetworkModel.from_admittance(y, y_ds, slack=base.slack, zip_coeffs=z)
        assert np.array_equal(model.source_injection(), d["src"])
    else:
        model = NetworkModel.from_branches(base.branches, int(d["n_buses"]), slack=base.slack, zip_coeffs=z)
    assert np.array_equal(model.admittance.y_dd.tocsc().data, d["ydd_data"])
    return model, d


@pytest.mark.parametrize("name", ["zip9_mixed", "zip9_heavy", "zip9_pure_zi", "zip101_mixed", "zip9_mesh",
                                  "zip101_mesh", "zip9_warm", "zip501_warm", "zip9_mesh_warm"])
def test_zip_matches_reference(name):
    """``*_warm``: opts.initial_voltage set (fpi.py:141-145), one fixture per GPU
    route (chain kernel, tree kernel, meshed LU kernel)."""
    from paper_2403_04578_b200 import LoadMatrix, SolveOptions, batch_solve_dense
    model, d = fixture(name)
    opts = SolveOptions(tolerance=float(d["tol"]), max_iterations=int(d["max_iter"]),
                        residual_tolerance=float(d["residual_tol"]),
                        initial_voltage=d["initial_voltage"] if "initial_voltage" in d else None)
    out = batch_solve_dense(model, LoadMatrix(d["S"]), opts)
    assert out.iterations == int(d["iterations"])
    assert np.array_equal(out.converged_mask, d["mask"])
    # per-case counts: the reference's own fpi_solve counts (one-case solver semantics)
    assert np.abs(out.iterations_per_case.astype(int) - d["n_case"]).max() <= 1
    good = d["mask"]
    assert np.abs(out.values[:, good] - d["V"][:, good]).max(initial=0) <= 1e-9
    fin = np.isfinite(d["residuals"])
    assert np.allclose(out.residuals[fin & good], d["residuals"][fin & good], rtol=1e-3, atol=1e-12)


def test_zip_random_feeder_vs_oracle():
    from paper_2403_04578_b200 import (GenSpec, LoadMatrix, NetworkModel, SolveOptions, ZipCoefficients,
                                       batch_solve_dense, build_network, gen_scenarios)
    spec = GenSpec(n_buses=301, seed=7, load_scale=2.0)
    base = build_network(spec)
    b = base.n_demand
    rng = np.random.default_rng(3)
    w = rng.dirichlet([0.5, 0.5, 2.0], size=b)
    z = ZipCoefficients(alpha_z=w[:, 0], alpha_i=w[:, 1], alpha_p=1.0 - w[:, 0] - w[:, 1])
    model = NetworkModel.from_branches(base.branches, 301, slack=base.slack, zip_coeffs=z)
    S = gen_scenarios(model, 200, spec).values
    out = batch_solve_dense(model, LoadMatrix(S), SolveOptions())
    V, n, mask, res, it = orc.dense_zip_batch(model.admittance.y_dd, model.source_injection(), model.slack.v_s,
                                              z.alpha_z, z.alpha_i, z.alpha_p, S)
    assert out.iterations == it and np.array_equal(out.converged_mask, mask)
    assert np.array_equal(out.iterations_per_case, n)
    assert np.abs(out.values - V).max() <= 1e-10


@pytest.mark.parametrize("n_buses", [2, 3, 40])
def test_zip_small_feeders_nan_and_empty(n_buses):
    """Edge cases: b = 1 and 2, empty batch, and a NaN load -- which makes the
    reference's splu of that case's B fail ("Factor is exactly singular" ->
    SingularSystemError for the whole batch), so it raises here too."""
    from paper_2403_04578_b200 import (GenSpec, LoadMatrix, NetworkModel, SingularSystemError, SolveOptions,
                                       ZipCoefficients, batch_solve_dense, build_network, gen_scenarios)
    spec = GenSpec(n_buses=n_buses, seed=5)
    base = build_network(spec)
    b = base.n_demand
    w = np.random.default_rng(n_buses).dirichlet([1.0, 1.0, 1.0], size=b)
    z = ZipCoefficients(alpha_z=w[:, 0], alpha_i=w[:, 1], alpha_p=1.0 - w[:, 0] - w[:, 1])
    model = NetworkModel.from_branches(base.branches, n_buses, slack=base.slack, zip_coeffs=z)
    S = gen_scenarios(model, 30, spec).values.copy()
    out = batch_solve_dense(model, LoadMatrix(S), SolveOptions())
    V, n, mask, res, it = orc.dense_zip_batch(model.admittance.y_dd, model.source_injection(), model.slack.v_s,
                                              z.alpha_z, z.alpha_i, z.alpha_p, S)
    assert np.array_equal(out.iterations_per_case, n) and np.array_equal(out.converged_mask, mask)
    assert np.abs(out.values - V).max() <= 1e-10
    empty = batch_solve_dense(model, LoadMatrix(np.zeros((b, 0), dtype=complex)), SolveOptions())
    assert empty.values.shape == (b, 0) and empty.iterations == 0
    S[0, 4] = np.nan
    with pytest.raises(SingularSystemError):
        batch_solve_dense(model, LoadMatrix(S), SolveOptions())


@pytest.mark.parametrize("n_buses,kmax", [(40, 1), (300, 1), (60, 2)])
def test_zip_deep_feeders_thread_per_case_kernel(n_buses, kmax):
    """Radial feeders the tree kernel does not take (chains: > 64 depth levels) run
    on tpf_sparse_zip_chain_c128 with the same semantics."""
    from paper_2403_04578_b200 import (GenSpec, LoadMatrix, NetworkModel, SolveOptions, ZipCoefficients,
                                       batch_solve_dense, build_network, gen_scenarios)
    spec = GenSpec(n_buses=n_buses, k_max=kmax, seed=11)
    base = build_network(spec)
    b = base.n_demand
    w = np.random.default_rng(b).dirichlet([1.0, 1.0, 1.0], size=b)
    z = ZipCoefficients(alpha_z=w[:, 0], alpha_i=w[:, 1], alpha_p=1.0 - w[:, 0] - w[:, 1])
    model = NetworkModel.from_branches(base.branches, n_buses, slack=base.slack, zip_coeffs=z)
    S = gen_scenarios(model, 150, spec).values.copy()
    S[:, 3] = 0.0
    out = batch_solve_dense(model, LoadMatrix(S), SolveOptions())
    V, n, mask, res, it = orc.dense_zip_batch(model.admittance.y_dd, model.source_injection(), model.slack.v_s,
                                              z.alpha_z, z.alpha_i, z.alpha_p, S)
    assert out.iterations == it
    assert np.array_equal(out.converged_mask, mask)
    assert np.abs(out.iterations_per_case.astype(int) - n).max() <= 1
    assert np.abs(out.values[:, mask] - V[:, mask]).max(initial=0) <= 1e-9
    fin = np.isfinite(res) & mask
    assert np.allclose(out.residuals[fin], res[fin], rtol=1e-3, atol=1e-12)


@pytest.mark.parametrize("n_buses,loops", [(3, 1), (40, 6), (301, 30), (1001, 40)])
def test_zip_meshed_vs_oracle(n_buses, loops):
    """Meshed Y_dd (tie branches between demand buses): the per-case fixed-
    pattern LU kernel (tpf_sparse_zip_lu_c128) against the oracle's per-case
    splu route; zero-load and infeasible cases included."""
    from paper_2403_04578_b200 import (Branch, GenSpec, LoadMatrix, NetworkModel, SolveOptions, ZipCoefficients,
                                       batch_solve_dense, build_network, gen_scenarios)
    from paper_2403_04578_b200.sparse import tree_parents
    spec = GenSpec(n_buses=n_buses, seed=11, load_scale=2.0)
    base = build_network(spec)
    b = base.n_demand
    rng = np.random.default_rng(n_buses)
    branches = list(base.branches)
    for _ in range(loops):
        i, j = (int(x) for x in rng.choice(np.arange(1, n_buses), 2, replace=False))
        branches.append(Branch(from_bus=i, to_bus=j, r=0.02, x=0.03))
    w = rng.dirichlet([1.0, 1.0, 2.0], size=b)
    z = ZipCoefficients(alpha_z=w[:, 0], alpha_i=w[:, 1], alpha_p=1.0 - w[:, 0] - w[:, 1])
    model = NetworkModel.from_branches(branches, n_buses, slack=base.slack, zip_coeffs=z)
    if n_buses > 3:
        assert tree_parents(model.admittance.y_dd) is None
    tau = 150
    S = gen_scenarios(model, tau, spec).values.copy()
    S[:, 1] = 0.0
    S[:, 2] *= 500.0
    opts = SolveOptions(max_iterations=40)
    out = batch_solve_dense(model, LoadMatrix(S), opts)
    V, n, mask, res, it = orc.dense_zip_batch(model.admittance.y_dd, model.source_injection(), model.slack.v_s,
                                              z.alpha_z, z.alpha_i, z.alpha_p, S, max_iter=40)
    assert np.array_equal(out.converged_mask, mask)
    assert np.abs(out.iterations_per_case.astype(int) - n).max() <= 1
    assert abs(out.iterations - it) <= 1
    assert np.abs(out.values[:, mask] - V[:, mask]).max(initial=0) <= 1e-9


def test_zip_meshed_zero_diagonal_needs_pivoting():
    """A meshed network whose B = Y_dd + diag(alpha_z s*) has an exactly zero
    diagonal entry (series capacitor and reactor cancelling at bus 2, no
    constant-impedance share there): nonsingular, so the reference's splu
    pivots past it (fpi.py:119); the GPU route for small meshed networks
    pivots too (tpf_sparse_zip_dense_c128) and matches the oracle."""
    from paper_2403_04578_b200 import (Branch, LoadMatrix, NetworkModel, SlackSpec, SolveOptions, ZipCoefficients,
                                       batch_solve_dense)
    from paper_2403_04578_b200.sparse import tree_parents
    branches = [Branch(from_bus=0, to_bus=1, r=0.0, x=0.1), Branch(from_bus=1, to_bus=2, r=0.0, x=-0.1),
                Branch(from_bus=2, to_bus=3, r=0.0, x=0.1), Branch(from_bus=1, to_bus=3, r=0.01, x=0.05)]
    z = ZipCoefficients(alpha_z=np.array([0.3, 0.0, 0.2]), alpha_i=np.array([0.3, 0.5, 0.3]),
                        alpha_p=np.array([0.4, 0.5, 0.5]))
    model = NetworkModel.from_branches(branches, 4, slack=SlackSpec(), zip_coeffs=z)
    y = model.admittance.y_dd.toarray()
    assert tree_parents(model.admittance.y_dd) is None and y[1, 1] == 0
    rng = np.random.default_rng(3)
    S = (rng.uniform(0.01, 0.2, (3, 64)) + 1j * rng.uniform(0.0, 0.05, (3, 64))).astype(np.complex128)
    opts = SolveOptions(max_iterations=60)
    out = batch_solve_dense(model, LoadMatrix(S), opts)
    V, n, mask, res, it = orc.dense_zip_batch(model.admittance.y_dd, model.source_injection(), model.slack.v_s,
                                              z.alpha_z, z.alpha_i, z.alpha_p, S, max_iter=60)
    assert np.array_equal(out.converged_mask, mask)
    assert np.abs(out.iterations_per_case.astype(int) - n).max() <= 1
    assert np.abs(out.values[:, mask] - V[:, mask]).max(initial=0) <= 1e-9


def test_zip_meshed_dense_and_fixed_pattern_kernels_agree():
    """The two meshed ZIP kernels (dense LU with row pivoting for b <= 64, fixed
    fill pattern without pivoting beyond) on one well-conditioned meshed
    network: the same counts and masks, voltages to 1e-12."""
    import torch
    from paper_2403_04578_b200 import (Branch, GenSpec, LoadMatrix, NetworkModel, SolveOptions, ZipCoefficients,
                                       build_network, gen_scenarios)
    from paper_2403_04578_b200 import dense as dense_mod
    from paper_2403_04578_b200._device import ModelContract
    spec = GenSpec(n_buses=30, seed=5, load_scale=1.5)
    base = build_network(spec)
    rng = np.random.default_rng(5)
    branches = list(base.branches) + [Branch(from_bus=3, to_bus=20, r=0.02, x=0.03),
                                      Branch(from_bus=7, to_bus=25, r=0.03, x=0.02)]
    b = base.n_demand
    w = rng.dirichlet([1.0, 1.0, 2.0], size=b)
    z = ZipCoefficients(alpha_z=w[:, 0], alpha_i=w[:, 1], alpha_p=1.0 - w[:, 0] - w[:, 1])
    model = NetworkModel.from_branches(branches, 30, slack=base.slack, zip_coeffs=z)
    L = LoadMatrix(gen_scenarios(model, 200, spec).values)
    opts = SolveOptions(max_iterations=50)
    c = ModelContract.of(model)
    a = dense_mod._solve_zip_dense(model, c, L, opts, torch.device("cuda", 0), False)
    lib = dense_mod._capi.load()  # force the fixed-pattern kernel: no dense route for any b
    orig = lib.tpf_sparse_zip_dense_max_nodes
    try:
        lib.tpf_sparse_zip_dense_max_nodes = lambda: 0
        f = dense_mod._solve_zip_lu(model, c, L, opts, torch.device("cuda", 0), False)
    finally:
        lib.tpf_sparse_zip_dense_max_nodes = orig
    assert np.array_equal(a.iterations_per_case, f.iterations_per_case)
    assert np.array_equal(a.converged_mask, f.converged_mask)
    assert np.abs(a.values - f.values).max() <= 1e-12
