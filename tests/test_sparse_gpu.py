"""Parity of the CUDA sparse engine with the reference (golden) and the dense engine."""

import numpy as np
import pytest

from conftest import gpu_available
from oracle import tpf_oracle as orc

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

SPARSE_GOLDEN = ["twobus_known", "twobus_infeasible", "nine_t500", "nine_zero_rows",
                 "nine_zero_batch", "nine_cap1", "nine_cap2", "nine_cap3", "nine_cap5", "nine_cap8",
                 "acc3_b100_t100", "acc7_mixed_zero", "asym6", "c1_slice512", "c2_slice192",
                 "c3_slice6"]


def solve(g, S=None, **kw):
    from paper_2403_04578_b200 import LoadMatrix, batch_solve_sparse
    return batch_solve_sparse(g.model, LoadMatrix(g.S if S is None else S), g.opts(), **kw)


@pytest.mark.parametrize("use_tree", [True, False], ids=["tree", "general"])
@pytest.mark.parametrize("name", SPARSE_GOLDEN)
def test_matches_reference_golden(golden, name, use_tree):
    g = golden(name)
    out = solve(g, use_tree=use_tree)
    assert out.iterations == int(g["sparse_iterations"])
    assert np.array_equal(out.converged_mask, g["sparse_mask"])
    good = g["sparse_mask"]
    # iterate sequences of the two formulations agree to accumulated rounding (test_sparse.py:170-180)
    tol = 1e-9
    assert np.abs(out.values[:, good] - g["sparse_V"][:, good]).max(initial=0.0) <= tol


def test_dense_sparse_equivalence_on_gpu(golden):
    """Acceptance criterion 3 (test_acceptance.py:90-108) on the GPU engine."""
    from paper_2403_04578_b200 import LoadMatrix, batch_solve_dense, factorization_count
    for name in ("acc3_b100_t100", "nine_t500", "acc7_mixed_zero"):
        g = golden(name)
        d = batch_solve_dense(g.model, LoadMatrix(g.S), g.opts())
        before = factorization_count()
        s = solve(g)
        assert factorization_count() - before == 1
        assert np.abs(d.values - s.values).max() < 1e-10
        assert d.iterations == s.iterations
        assert np.array_equal(d.converged_mask, s.converged_mask)


def test_chunking_preserves_results(golden):
    g = golden("nine_t500")
    whole = solve(g)
    parts = [solve(g, S=np.ascontiguousarray(g.S[:, :213])), solve(g, S=np.ascontiguousarray(g.S[:, 213:]))]
    assert np.array_equal(np.hstack([p.values for p in parts]), whole.values)


def test_two_bus_known_answer(golden):
    out = solve(golden("twobus_known"))
    assert abs(out.values[0, 0] - (1 + np.sqrt(0.96)) / 2) < 1e-12


def test_c3_feeder_per_case_vs_oracle(golden):
    """b=5,000 feeder (config C3): per-case counts and values vs the oracle's fpi_solve restatement."""
    from oracle import tpf_oracle as orc
    g = golden("c3_slice6")
    out = solve(g)
    y, src, v_s = g.args
    for j in range(g.S.shape[1]):
        v, n, ok = orc.fpi_single(y, src, v_s, g.S[:, j])
        assert ok and out.converged_mask[j]
        assert abs(int(out.iterations_per_case[j]) - n) <= 1
        assert np.abs(out.values[:, j] - v).max() < 1e-10


def test_host_pipeline_matches_device_path_bitwise(golden):
    from paper_2403_04578_b200 import LoadMatrix, batch_solve_sparse
    g = golden("c1_slice512")
    host = batch_solve_sparse(g.model, LoadMatrix(g.S), g.opts(), chunk_cases=100)
    dev = batch_solve_sparse(g.model, LoadMatrix(g.S), g.opts(), return_on_device=True)
    assert np.array_equal(host.values, dev.values.cpu().numpy())
    assert np.array_equal(host.iterations_per_case, dev.iterations_per_case.cpu().numpy())


@pytest.mark.parametrize("name", ["c1_slice512", "c2_slice192", "c3_slice6", "acc7_mixed_zero"])
def test_tree_kernel_matches_general_kernel(golden, name):
    """On-chip tree sweeps == generic CSR trisolves (same LU, same semantics)."""
    g = golden(name)
    a = solve(g, use_tree=True)
    b = solve(g, use_tree=False)
    assert np.array_equal(a.iterations_per_case, b.iterations_per_case)
    assert np.abs(a.values - b.values).max() < 1e-13


def test_tree_kernel_device_path_matches_pipeline(golden):
    g = golden("c1_slice512")
    host = solve(g, chunk_cases=100)
    dev = solve(g, return_on_device=True)
    assert np.array_equal(host.values, dev.values.cpu().numpy())


def test_sparse_nonfinite_loads_flagged():
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, batch_solve_sparse, LoadMatrix
    spec = GenSpec(n_buses=101, seed=3)
    model = build_network(spec)
    S = gen_scenarios(model, 40, spec).values.copy()
    S[10, 4] = np.nan
    for use_tree in (True, False):
        out = batch_solve_sparse(model, LoadMatrix(S), use_tree=use_tree)
        assert out.iterations_per_case[4] == 100 and not out.converged_mask[4]
        assert out.converged_mask[np.arange(40) != 4].all()


def test_sparse_fortran_order_same_bits(golden):
    g = golden("acc3_b100_t100")
    a = solve(g)
    b = solve(g, S=np.asfortranarray(g.S))
    assert np.array_equal(a.values, b.values)


def test_sparse_matches_dense_on_c1_feeder():
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, batch_solve_sparse, batch_solve_dense
    spec = GenSpec(n_buses=35, seed=0)
    model = build_network(spec)
    loads = gen_scenarios(model, 2000, spec)
    d = batch_solve_dense(model, loads)
    s = batch_solve_sparse(model, loads)
    assert np.array_equal(d.iterations_per_case, s.iterations_per_case)
    assert np.abs(d.values - s.values).max() < 1e-12


@pytest.mark.parametrize("name", ["c3_slice6", "c1_slice512", "nine_t500", "acc7_mixed_zero"])
def test_fused_residual_bitwise_equals_residual_kernel(golden, name):
    """tpf_sparse_tree_fpi_resid_c128's in-kernel post-check == tpf_residual_c128 on the same V."""
    import torch
    from paper_2403_04578_b200 import SparseOperator
    from paper_2403_04578_b200._device import residual_and_summary
    g = golden(name)
    op = SparseOperator(g.model, "cuda:0")
    if op.tree is None:
        pytest.skip("not a tree schedule")
    S = torch.from_numpy(np.ascontiguousarray(g.S)).to("cuda:0")
    tau = S.shape[1]
    fused = torch.full((tau,), -1.0, dtype=torch.float64, device="cuda:0")
    V, iters = op.solve(S, g.opts(), resid=fused)
    ref, _, _ = residual_and_summary(op.contract, S, V, iters, 1e-8, op.device)
    a, b = fused.cpu().numpy(), ref.cpu().numpy()
    assert np.array_equal(np.isnan(a), np.isnan(b))
    assert np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])


def test_fused_residual_nonfinite_case():
    import torch
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, SparseOperator, SolveOptions
    from paper_2403_04578_b200._device import residual_and_summary
    spec = GenSpec(n_buses=101, seed=3)
    model = build_network(spec)
    S = gen_scenarios(model, 40, spec).values.copy()
    S[10, 4] = np.nan
    op = SparseOperator(model, "cuda:0")
    St = torch.from_numpy(S).to("cuda:0")
    fused = torch.empty(40, dtype=torch.float64, device="cuda:0")
    V, iters = op.solve(St, SolveOptions(), resid=fused)
    ref, _, _ = residual_and_summary(op.contract, St, V, iters, 1e-8, op.device)
    a, b = fused.cpu().numpy(), ref.cpu().numpy()
    assert np.isnan(a[4]) and np.isnan(b[4])
    keep = np.arange(40) != 4
    assert np.array_equal(a[keep], b[keep])


@pytest.mark.parametrize("use_tree", [True, False], ids=["tree", "general"])
def test_devices_split_bitwise_equal(golden, use_tree):
    from paper_2403_04578_b200 import LoadMatrix, batch_solve_sparse
    g = golden("c1_slice512")
    one = batch_solve_sparse(g.model, LoadMatrix(g.S), g.opts(), use_tree=use_tree)
    many = batch_solve_sparse(g.model, LoadMatrix(g.S), g.opts(), use_tree=use_tree,
                              devices=["cuda:0", "cuda:0", "cuda:0"])
    assert np.array_equal(one.values, many.values)
    assert np.array_equal(one.iterations_per_case, many.iterations_per_case)
    assert np.array_equal(one.residuals, many.residuals)
    assert one.iterations == many.iterations


def test_tree_chunked_long_batches_bitwise(golden, monkeypatch):
    """Long node-major batches are solved in compact chunks (SparseOperator): same bits."""
    import torch
    import paper_2403_04578_b200.sparse as sp
    from paper_2403_04578_b200 import SparseOperator
    g = golden("c1_slice512")
    S = torch.from_numpy(np.ascontiguousarray(g.S)).cuda()
    op = SparseOperator(g.model, "cuda:0")
    tau = S.shape[1]
    r1 = torch.empty(tau, dtype=torch.float64, device="cuda:0")
    V1, it1 = op.solve(S, g.opts(), resid=r1)
    monkeypatch.setattr(sp, "TREE_CHUNK", 100)
    r2 = torch.empty(tau, dtype=torch.float64, device="cuda:0")
    V2, it2 = op.solve(S, g.opts(), resid=r2)
    assert torch.equal(V1, V2) and torch.equal(it1, it2) and torch.equal(r1, r2)


def test_feeder_beyond_tree_kernel_limits_uses_general_kernel():
    """b > 5,120 does not fit the tree kernel's shared memory: the general CSR kernel runs instead."""
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, batch_solve_sparse, SparseOperator
    spec = GenSpec(n_buses=5301, seed=1)
    model = build_network(spec)
    assert SparseOperator(model, "cuda:0").tree is None
    loads = gen_scenarios(model, 64, spec)
    out = batch_solve_sparse(model, loads)
    assert out.converged_mask.all() and 3 <= out.iterations <= 10


@pytest.mark.parametrize("name", ["acc3_b100_t100", "nine_t500", "acc7_mixed_zero", "c3_slice6", "nine_zero_batch",
                                  "twobus_infeasible"])
@pytest.mark.parametrize("layout", ["node", "case"])
def test_subtree_and_level_kernels_bitwise(golden, name, layout):
    """Warp-per-subtree kernel (default for radial feeders) == level kernel: same
    V, counts and fused residual bits, node-major (chunked transposes) and
    case-major (1-D bulk copies) layouts."""
    import torch
    from paper_2403_04578_b200 import SparseOperator
    g = golden(name)
    sub = SparseOperator(g.model, kernel="subtree")
    lvl = SparseOperator(g.model, kernel="tree")
    if sub.sub is None or lvl.tree is None:
        pytest.skip("not a radial feeder the tree kernels take")
    S = torch.from_numpy(g.S).cuda()
    if layout == "case":
        S = S.t().contiguous().t()
    out = []
    for op in (sub, lvl):
        r = torch.empty(S.shape[1], dtype=torch.float64, device="cuda")
        V, it = op.solve(S, g.opts(), V=torch.empty_like(S), resid=r)
        out.append((V, it, r))
    assert sub.kernel == "sparse_subtree_kernel"
    assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1])
    assert torch.equal(torch.isnan(out[0][2]), torch.isnan(out[1][2]))
    keep = ~torch.isnan(out[0][2])
    assert torch.equal(out[0][2][keep], out[1][2][keep])


@pytest.mark.parametrize("n_buses,seed", [(35, 4), (301, 5), (1001, 6), (5001, 0)])
def test_subtree_kernel_random_feeders(n_buses, seed):
    """Subtree kernel vs level kernel on generated feeders of several shapes (bitwise)."""
    import torch
    from paper_2403_04578_b200 import GenSpec, build_network, SparseOperator, SolveOptions
    from paper_2403_04578_b200.synth import gen_scenarios_device
    spec = GenSpec(n_buses=n_buses, seed=seed)
    model = build_network(spec)
    S = gen_scenarios_device(model, 3000, spec, device="cuda:0")
    res = []
    for k in ("subtree", "tree"):
        op = SparseOperator(model, kernel=k)
        r = torch.empty(3000, dtype=torch.float64, device="cuda")
        V, it = op.solve(S, SolveOptions(), resid=r)
        res.append((V, it, r, op.kernel))
    assert res[0][3] == "sparse_subtree_kernel"
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])
    assert torch.equal(res[0][2], res[1][2])


def test_sparse_full_c3_sampled_vs_oracle():
    """Full config C3 (b=5,000, tau=525,600, device-generated loads) through the
    default sparse path (subtree kernel, case-major chunks): every case
    converges, and 300 sampled columns match the oracle's single-case solver
    (fpi.py:107-206: SuperLU of Y_dd) to 1e-12 with the same counts."""
    import torch
    from paper_2403_04578_b200 import GenSpec, build_network, SparseOperator
    from paper_2403_04578_b200.synth import gen_scenarios_device
    spec = GenSpec(n_buses=5001, seed=0)
    model = build_network(spec)
    tau = 525600
    S = gen_scenarios_device(model, tau, spec, device="cuda:0")
    op = SparseOperator(model)
    assert op.kernel == "sparse_subtree_kernel"
    resid = torch.empty(tau, dtype=torch.float64, device="cuda")
    V, it = op.solve(S, resid=resid)
    it_h = it.cpu().numpy()
    assert it_h.max() < 100 and bool((resid < 1e-8).all())
    cols = np.random.default_rng(0).choice(tau, 300, replace=False)
    idx = torch.from_numpy(cols).cuda()
    Sh = S[:, idx].cpu().numpy()
    Vg = V[:, idx].cpu().numpy()
    del S, V
    y, src, v_s = model.admittance.y_dd, model.source_injection(), model.slack.v_s
    exact = 0
    for k, j in enumerate(cols):
        v, n, conv = orc.fpi_single(y, src, v_s, Sh[:, k])
        assert conv
        assert abs(n - int(it_h[j])) <= 1
        exact += n == int(it_h[j])
        assert np.abs(Vg[:, k] - v).max() < 1e-12
    assert exact >= 297
