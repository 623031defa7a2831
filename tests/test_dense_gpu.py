"""Parity of the CUDA dense engine with the reference (golden) and the oracle.

Bars (BASELINE.json north star): max|V - V_ref| <= 1e-9 p.u. and the same
iteration count (+-1; exact is asserted where the oracle proves it), complex128.
"""

import numpy as np
import pytest

from conftest import gpu_available
from oracle import tpf_oracle as orc

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

V_TOL = 1e-9

DENSE_GOLDEN = ["twobus_known", "twobus_infeasible", "nine_t500", "nine_zero_rows",
                "nine_zero_batch", "nine_cap1", "nine_cap2", "nine_cap3", "nine_cap5", "nine_cap8",
                "acc3_b100_t100", "acc7_mixed_zero", "asym6", "c1_slice512", "c2_slice192"]


def solve(g, S=None, **kw):
    from paper_2403_04578_b200 import LoadMatrix, batch_solve_dense
    return batch_solve_dense(g.model, LoadMatrix(g.S if S is None else S), g.opts(), **kw)


@pytest.mark.parametrize("name", DENSE_GOLDEN)
def test_matches_reference_golden(golden, name):
    g = golden(name)
    out = solve(g)
    assert out.iterations == int(g["dense_iterations"])
    assert np.array_equal(out.converged_mask, g["dense_mask"])
    good = g["dense_mask"]
    assert np.abs(out.values[:, good] - g["dense_V"][:, good]).max(initial=0.0) <= V_TOL
    # converged cases: both below residual_tol (the joint loop of the reference keeps
    # refining early columns, so their residuals are smaller than a frozen case's)
    assert (out.residuals[good] < float(g["residual_tol"])).all()
    bad = ~good & np.isfinite(g["dense_residuals"])
    assert np.allclose(out.residuals[bad], g["dense_residuals"][bad], rtol=1e-6)


@pytest.mark.parametrize("name", DENSE_GOLDEN)
def test_matches_oracle_per_case(golden, name):
    """Same semantics as the oracle's per-case freeze: counts exact, values to GEMM rounding."""
    g = golden(name)
    y, src, v_s = g.args
    o = g.opts()
    V, n_case, mask, res = orc.dense_per_case(y, src, v_s, g.S, o.tolerance, o.max_iterations,
                                              o.residual_tolerance)
    out = solve(g)
    assert np.array_equal(out.iterations_per_case, n_case)
    good = mask
    assert np.abs(out.values[:, good] - V[:, good]).max(initial=0.0) < 1e-12


def test_two_bus_known_answer(golden):
    out = solve(golden("twobus_known"))
    assert abs(out.values[0, 0] - (1 + np.sqrt(0.96)) / 2) < 1e-12


def test_infeasible_column_flagged_others_converge(golden):
    out = solve(golden("twobus_infeasible"))
    assert list(out.converged_mask) == [True, False, True, True]
    assert out.iterations == 100
    assert out.iterations_per_case[1] == 100


def test_zero_load_batch(golden):
    from scipy.sparse.linalg import spsolve
    g = golden("nine_zero_batch")
    out = solve(g)
    assert out.converged_mask.all() and out.iterations <= 1
    no_load = spsolve(g.model.admittance.y_dd.tocsc(), -g.model.source_injection())
    assert np.abs(out.values - no_load[:, None]).max() < 1e-12


def test_permutation_equivariance_bitwise(golden):
    g = golden("c2_slice192")
    perm = np.random.default_rng(3).permutation(g.S.shape[1])
    a = solve(g)
    b = solve(g, S=np.ascontiguousarray(g.S[:, perm]))
    assert np.array_equal(b.values, a.values[:, perm])
    assert np.array_equal(b.iterations_per_case, a.iterations_per_case[perm])


def test_shard_invariance_bitwise(golden):
    """tau split into 1/2/4/8 contiguous shards -> identical bits."""
    g = golden("c1_slice512")
    whole = solve(g)
    for parts in (2, 4, 8):
        edges = np.linspace(0, g.S.shape[1], parts + 1).astype(int)
        vals = np.hstack([solve(g, S=np.ascontiguousarray(g.S[:, lo:hi])).values
                          for lo, hi in zip(edges[:-1], edges[1:])])
        assert np.array_equal(vals, whole.values)


def test_replicated_case_identical_columns(golden):
    g = golden("nine_t500")
    out = solve(g, S=np.repeat(g.S[:, :1], 7, axis=1))
    for j in range(1, 7):
        assert np.array_equal(out.values[:, j], out.values[:, 0])


def test_fortran_order_input_same_bits(golden):
    """read_loads gives an F-order view (fileio.py:233); layout must not change bits."""
    g = golden("acc3_b100_t100")
    a = solve(g)
    b = solve(g, S=np.asfortranarray(g.S))
    assert np.array_equal(a.values, b.values)


def test_rerun_is_deterministic(golden):
    g = golden("c2_slice192")
    a, b = solve(g), solve(g)
    assert np.array_equal(a.values, b.values) and np.array_equal(a.residuals, b.residuals)


def test_dense_full_c2_properties():
    """Full config C2 (b=100, tau=525,600): per-case counts reproduce the survey
    probe exactly (sum 2,615,281, max 7), every case converges, and a sample of
    columns matches the oracle's per-case solution."""
    import torch
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator
    from paper_2403_04578_b200._device import residual_and_summary
    spec = GenSpec(n_buses=101, seed=0)
    model = build_network(spec)
    S_h = gen_scenarios(model, 525600, spec).values
    op = DenseOperator(model)
    S = torch.from_numpy(S_h).cuda()
    V, iters = op.solve(S)
    resid, mask, summ = residual_and_summary(op.contract, S, V, iters, 1e-8, op.device)
    it = iters.cpu().numpy()
    assert int(it.sum()) == 2615281 and int(it.max()) == 7
    assert int(summ[0]) == 7 and int(summ[1]) == 525600
    cols = np.random.default_rng(0).choice(525600, 300, replace=False)
    Vo, no, _, _ = orc.dense_per_case(model.admittance.y_dd, model.source_injection(),
                                      model.slack.v_s, S_h[:, cols])
    Vg = V[:, torch.from_numpy(cols).cuda()].cpu().numpy()
    assert np.array_equal(it[cols], no)
    assert np.abs(Vg - Vo).max() < 1e-12


def test_host_pipeline_matches_device_path_bitwise(golden):
    """The native chunked H2D/solve/D2H pipeline (several chunks) == one device solve."""
    from paper_2403_04578_b200 import LoadMatrix, batch_solve_dense
    g = golden("c2_slice192")
    host = batch_solve_dense(g.model, LoadMatrix(g.S), g.opts(), chunk_cases=50)
    dev = batch_solve_dense(g.model, LoadMatrix(g.S), g.opts(), return_on_device=True)
    assert np.array_equal(host.values, dev.values.cpu().numpy())
    assert np.array_equal(host.iterations_per_case, dev.iterations_per_case.cpu().numpy())
    assert np.array_equal(host.residuals, dev.residuals.cpu().numpy())
    assert host.iterations == dev.iterations


def test_large_b_c5_matches_reference(golden):
    """b=1,000 near voltage collapse (config C5): active-set DMMA path vs reference."""
    g = golden("c5_slice32")
    out = solve(g)
    assert out.iterations == int(g["dense_iterations"]) == 58
    assert np.array_equal(out.converged_mask, g["dense_mask"])
    assert np.abs(out.values - g["dense_V"]).max() <= V_TOL
    y, src, v_s = g.args
    V, n_case, mask, _ = orc.dense_per_case(y, src, v_s, g.S)
    assert np.array_equal(out.iterations_per_case, n_case)
    assert np.abs(out.values - V).max() < 1e-11


def test_large_b_path_on_small_feeder_matches_small_kernel(golden):
    """The generic large-b kernel agrees with the shared-memory kernel where both apply."""
    import torch
    from paper_2403_04578_b200 import DenseOperator
    g = golden("acc3_b100_t100")
    op = DenseOperator(g.model)
    S = torch.from_numpy(g.S).cuda()
    V1, it1 = op.solve(S)
    op.large = True
    V2, it2 = op.solve(S)
    assert torch.equal(it1, it2)
    assert (V1 - V2).abs().max().item() < 1e-13


def test_large_b_permutation_invariance_bitwise(golden):
    g = golden("c5_slice32")
    perm = np.random.default_rng(5).permutation(g.S.shape[1])
    a = solve(g)
    b = solve(g, S=np.ascontiguousarray(g.S[:, perm]))
    assert np.array_equal(b.values, a.values[:, perm])


def _large_solve_both_tails(monkeypatch, model, S):
    """(V, iterations) from the persistent tail kernel and from the
    per-iteration launches (TPF_LARGE_TAIL_LAUNCHES=1)."""
    import torch
    from paper_2403_04578_b200 import DenseOperator
    op = DenseOperator(model)
    assert op.large
    St = torch.from_numpy(np.ascontiguousarray(S)).cuda()
    monkeypatch.delenv("TPF_LARGE_TAIL_LAUNCHES", raising=False)
    V1, it1 = op.solve(St)
    monkeypatch.setenv("TPF_LARGE_TAIL_LAUNCHES", "1")
    V2, it2 = op.solve(St)
    return (V1.cpu().numpy(), it1.cpu().numpy()), (V2.cpu().numpy(), it2.cpu().numpy())


def test_large_b_persistent_tail_same_bits_c5_slice(golden, monkeypatch):
    """32 cases near collapse: the persistent kernel runs all 58 iterations;
    the per-iteration launches (GEMM tiles, then tail_kernel) give the same bits."""
    g = golden("c5_slice32")
    (V1, it1), (V2, it2) = _large_solve_both_tails(monkeypatch, g.model, g.S)
    assert int(it1.max()) == 58
    assert np.array_equal(it1, it2)
    assert np.array_equal(V1.view(np.int64), V2.view(np.int64))


def test_large_b_persistent_hand_off_same_bits(monkeypatch):
    """600 cases of the C5 feeder: GEMM tiles while more than 256 are active,
    then the persistent kernel; bitwise the per-iteration path, and the
    heavy tail (a few cases to 50+ iterations) is exercised."""
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios
    spec = GenSpec(n_buses=1001, seed=0, load_scale=21.0)
    m = build_network(spec)
    S = gen_scenarios(m, 600, GenSpec(n_buses=1001, seed=3, load_scale=21.0)).values
    (V1, it1), (V2, it2) = _large_solve_both_tails(monkeypatch, m, S)
    assert np.array_equal(it1, it2)
    assert np.array_equal(V1.view(np.int64), V2.view(np.int64))
    assert (it1 > 16).sum() >= 1 and int(it1.max()) >= 30


def test_large_b_device_loop_matches_host_loop(golden, monkeypatch):
    """The iteration loop as a CUDA graph WHILE node (default) and as
    max_iter host launches (TPF_LARGE_HOST_LOOP=1) give the same bits."""
    import torch
    from paper_2403_04578_b200 import DenseOperator
    g = golden("c5_slice32")
    op = DenseOperator(g.model)
    S = torch.from_numpy(g.S).cuda()
    monkeypatch.delenv("TPF_LARGE_HOST_LOOP", raising=False)
    V1, it1 = op.solve(S)
    monkeypatch.setenv("TPF_LARGE_HOST_LOOP", "1")
    V2, it2 = op.solve(S)
    assert torch.equal(it1, it2) and int(it1.max()) == 58
    assert torch.equal(V1.view(torch.int64), V2.view(torch.int64))


def test_large_b_solve_inside_stream_capture(golden):
    """Captured into a torch CUDA graph (the loop's WHILE node joins the
    captured graph) and replayed twice: the eager result, bitwise."""
    import torch
    from paper_2403_04578_b200 import DenseOperator
    g = golden("c5_slice32")
    op = DenseOperator(g.model)
    S = torch.from_numpy(g.S).cuda()
    V0, it0 = op.solve(S)
    op.solve(S)  # workspace and memos allocated outside the capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        Vg, itg = op.solve(S)
    for _ in range(2):
        Vg.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(itg, it0)
        assert torch.equal(Vg.view(torch.int64), V0.view(torch.int64))


@pytest.mark.parametrize("kernel", ["pairs"])
@pytest.mark.parametrize("name", ["c2_slice192", "c1_slice512", "nine_t500", "twobus_infeasible", "asym6",
                                  "nine_zero_batch"])
def test_ws_and_pair_kernels_agree(golden, name, kernel):
    """The two dispatched b <= 104 kernels, warp-specialised vs pairs (both 3M +
    Newton reciprocal): same counts, same bits."""
    import torch
    from paper_2403_04578_b200 import DenseOperator
    g = golden(name)
    op = DenseOperator(g.model)
    S = torch.from_numpy(g.S).cuda()
    o = g.opts()
    V1, it1 = op.solve(S, o, kernel="ws")
    V2, it2 = op.solve(S, o, kernel=kernel)
    assert torch.equal(it1, it2)
    if kernel == "pairs":
        assert torch.equal(V1, V2)
    fin = torch.isfinite(V2).all(dim=0)
    assert torch.equal(fin, torch.isfinite(V1).all(dim=0))
    if fin.any():
        assert (V1[:, fin] - V2[:, fin]).abs().max().item() <= 1e-13


def test_ws_kernel_full_c2_counts():
    import torch
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, DenseOperator
    spec = GenSpec(n_buses=101, seed=0)
    model = build_network(spec)
    S = torch.from_numpy(gen_scenarios(model, 525600, spec).values).cuda()
    op = DenseOperator(model)
    V1, it1 = op.solve(S, kernel="ws")
    assert int(it1.sum()) == 2615281  # the reference's per-case total
    V2, it2 = op.solve(S, kernel="pairs")
    assert torch.equal(it1, it2)
    assert (V1 - V2).abs().max().item() <= 1e-13


def test_large_b_beyond_persistent_limit(monkeypatch):
    """b = 1,300: 163 CTAs of 8 nodes cannot all be resident, so the device
    loop runs GEMM tiles and tail_kernel every iteration down to zero active
    cases; counts exact vs the oracle, bitwise the host loop."""
    import torch
    from paper_2403_04578_b200 import DenseOperator, GenSpec, build_network, gen_scenarios
    spec = GenSpec(n_buses=1301, seed=7, load_scale=4.0)
    model = build_network(spec)
    loads = gen_scenarios(model, 96, spec)
    op = DenseOperator(model)
    S = torch.from_numpy(np.ascontiguousarray(loads.values)).cuda()
    monkeypatch.delenv("TPF_LARGE_HOST_LOOP", raising=False)
    V1, it1 = op.solve(S)
    monkeypatch.setenv("TPF_LARGE_HOST_LOOP", "1")
    V2, it2 = op.solve(S)
    assert torch.equal(it1, it2) and torch.equal(V1.view(torch.int64), V2.view(torch.int64))
    V, n, mask, _ = orc.dense_per_case(model.admittance.y_dd, model.source_injection(), model.slack.v_s,
                                       loads.values)
    assert np.array_equal(it1.cpu().numpy(), n)
    assert np.abs(V1.cpu().numpy() - V).max() < 1e-11


@pytest.mark.parametrize("nb,scale", [(101, 1.0), (1001, 21.0)])
def test_one_operator_two_streams_concurrently(nb, scale):
    """One DenseOperator solving on two CUDA streams from two threads at once
    (b = 100: the shared-memory kernel; b = 1,000: the device loop and the
    cooperative persistent kernel): per-stream scratch, the sequential bits."""
    import threading
    import torch
    from paper_2403_04578_b200 import DenseOperator, GenSpec, build_network, gen_scenarios
    m = build_network(GenSpec(n_buses=nb, seed=0, load_scale=scale))
    S = [torch.from_numpy(np.ascontiguousarray(
        gen_scenarios(m, 600, GenSpec(n_buses=nb, seed=s, load_scale=scale)).values)).cuda() for s in (1, 2)]
    op = DenseOperator(m)
    ref = [op.solve(x) for x in S]
    torch.cuda.synchronize()
    out = [None, None]

    def run(i):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for _ in range(4):
                out[i] = op.solve(S[i])
            st.synchronize()

    ts = [threading.Thread(target=run, args=(i,)) for i in (0, 1)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in (0, 1):
        assert torch.equal(out[i][1], ref[i][1])
        assert torch.equal(out[i][0].view(torch.int64), ref[i][0].view(torch.int64))


@pytest.mark.parametrize("b", [1, 3, 8, 9, 33, 50, 56, 64, 72, 80, 88, 96, 100, 101, 104, 105, 128])
def test_feeder_sizes_across_kernel_boundaries(b):
    """Every node-block count of the shared-memory kernels (b <= 104) and the
    switch to the large-b kernel (b = 105): counts exact vs the oracle."""
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, batch_solve_dense
    spec = GenSpec(n_buses=b + 1, seed=b)
    model = build_network(spec)
    loads = gen_scenarios(model, 300, spec)
    out = batch_solve_dense(model, loads)
    V, n, mask, _ = orc.dense_per_case(model.admittance.y_dd, model.source_injection(), model.slack.v_s,
                                       loads.values)
    assert np.array_equal(out.iterations_per_case, n)
    assert np.array_equal(out.converged_mask, mask)
    assert np.abs(out.values - V).max() < 1e-12


def test_nonfinite_and_zero_loads_are_data():
    """NaN / inf loads never pass the step test: those cases run to the cap and are
    flagged, the rest of the batch is unaffected (dense.py:189-193, 198-199)."""
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, batch_solve_dense, LoadMatrix
    spec = GenSpec(n_buses=35, seed=1)
    model = build_network(spec)
    S = gen_scenarios(model, 64, spec).values.copy()
    clean = batch_solve_dense(model, LoadMatrix(S))
    S[3, 5] = np.nan
    S[7, 9] = np.inf
    S[:, 11] = 0.0
    out = batch_solve_dense(model, LoadMatrix(S))
    assert out.iterations_per_case[5] == 100 and out.iterations_per_case[9] == 100
    assert not out.converged_mask[5] and not out.converged_mask[9]
    assert out.converged_mask[11] and out.iterations_per_case[11] <= 1
    keep = np.ones(64, bool)
    keep[[5, 9, 11]] = False
    assert np.array_equal(out.values[:, keep], clean.values[:, keep])


def test_empty_batch():
    from paper_2403_04578_b200 import GenSpec, build_network, batch_solve_dense, LoadMatrix
    model = build_network(GenSpec(n_buses=9, seed=42))
    out = batch_solve_dense(model, LoadMatrix(np.zeros((8, 0), complex)))
    assert out.values.shape == (8, 0) and out.iterations == 0


def test_max_iterations_cap_and_tolerance_options(golden):
    """SolveOptions are honoured: a 2-iteration cap stops every case at 2."""
    from paper_2403_04578_b200 import LoadMatrix, batch_solve_dense, SolveOptions
    g = golden("c2_slice192")
    out = batch_solve_dense(g.model, LoadMatrix(g.S), SolveOptions(max_iterations=2))
    assert (out.iterations_per_case == 2).all() and out.iterations == 2
    loose = batch_solve_dense(g.model, LoadMatrix(g.S), SolveOptions(tolerance=1e-4))
    assert loose.iterations < 7


def test_ws_and_pairs_same_bits_default_build(golden):
    """libtpf.so carries only the dispatched 3M kernels (the 4M / split / solo A/B
    variants need -DTPF_AB_VARIANTS): ws and pairs give the same bits."""
    import torch
    from paper_2403_04578_b200 import DenseOperator, _capi
    assert not hasattr(_capi.load(), "tpf_dense_solo_fpi_c128")
    g = golden("c2_slice192")
    op = DenseOperator(g.model)
    S = torch.from_numpy(g.S).cuda()
    V1, _ = op.solve(S, g.opts(), kernel="ws")
    V2, _ = op.solve(S, g.opts(), kernel="pairs")
    assert torch.equal(V1, V2)


@pytest.mark.parametrize("devs", [["cuda:0", "cuda:0"], ["cuda:0", "cuda:0", "cuda:0"]])
def test_devices_split_bitwise_equal(golden, devs):
    """devices=[...]: contiguous case slices on concurrent per-device pipelines
    (here the same B200 several times) give the single-device bits."""
    from paper_2403_04578_b200 import LoadMatrix, batch_solve_dense
    g = golden("c2_slice192")
    one = batch_solve_dense(g.model, LoadMatrix(g.S), g.opts())
    many = batch_solve_dense(g.model, LoadMatrix(g.S), g.opts(), devices=devs)
    assert np.array_equal(one.values, many.values)
    assert np.array_equal(one.iterations_per_case, many.iterations_per_case)
    assert np.array_equal(one.residuals, many.residuals)
    assert np.array_equal(one.converged_mask, many.converged_mask)
    assert one.iterations == many.iterations
    # a pageable F-order input takes the same route
    many_f = batch_solve_dense(g.model, LoadMatrix(np.asfortranarray(g.S)), g.opts(), devices=devs)
    assert np.array_equal(one.values, many_f.values)


@pytest.mark.parametrize("order", ["C", "F"])
def test_pageable_staging_matches_pinned(golden, order):
    """Pageable loads go through pinned staging chunk by chunk: same bits as pinned input."""
    import torch
    from paper_2403_04578_b200 import LoadMatrix, batch_solve_dense
    g = golden("c1_slice512")
    S = np.array(g.S, order=order)
    pinned = torch.from_numpy(np.ascontiguousarray(g.S)).pin_memory().numpy()
    a = batch_solve_dense(g.model, LoadMatrix(S), g.opts(), chunk_cases=64)        # staged (pageable)
    b = batch_solve_dense(g.model, LoadMatrix(pinned), g.opts(), chunk_cases=64)   # direct DMA
    assert np.array_equal(a.values, b.values)
    assert np.array_equal(a.iterations_per_case, b.iterations_per_case)
    assert np.array_equal(a.residuals, b.residuals)


@pytest.mark.parametrize("method", ["dense", "sparse"])
@pytest.mark.parametrize("layout", ["node_major", "case_major"])
@pytest.mark.parametrize("tau,chunk", [(2000, 300), (1201, 300), (4097, 1024)])
def test_host_pipeline_ragged_ramp_chunks_bitwise(tau, chunk, layout, method):
    """Quarter-size first/last chunks (tau > 4*chunk) and a ragged tail, staged from pageable
    host memory in both host layouts, == one device-resident solve, bit for bit."""
    import torch
    from paper_2403_04578_b200 import (GenSpec, LoadMatrix, build_network, gen_scenarios,
                                       batch_solve_dense, batch_solve_sparse)
    solver = batch_solve_dense if method == "dense" else batch_solve_sparse
    spec = GenSpec(n_buses=101, seed=0)
    model = build_network(spec)
    S = gen_scenarios(model, tau, GenSpec(n_buses=101, seed=7)).values
    if layout == "case_major":
        S = np.asfortranarray(S)
    host = solver(model, LoadMatrix(S), chunk_cases=chunk)
    dev = solver(model, LoadMatrix(np.ascontiguousarray(S)), return_on_device=True)
    torch.cuda.synchronize()
    assert np.array_equal(host.values, dev.values.cpu().numpy())
    assert np.array_equal(host.iterations_per_case, dev.iterations_per_case.cpu().numpy())
    assert np.array_equal(host.converged_mask, dev.converged_mask.cpu().numpy())
    assert host.iterations == dev.iterations


def test_two_threads_same_device_bitwise(golden):
    """Concurrent host-pipeline calls from two Python threads on one GPU use
    separate scratch (the native calls release the GIL): each result equals the
    single-threaded solve bit for bit."""
    import threading
    from paper_2403_04578_b200 import LoadMatrix, batch_solve_dense, batch_solve_sparse
    g1, g2 = golden("c2_slice192"), golden("nine_t500")
    want = [batch_solve_dense(g1.model, LoadMatrix(g1.S), g1.opts()),
            batch_solve_sparse(g2.model, LoadMatrix(g2.S), g2.opts())]
    got = [None, None]

    def run(k):
        for _ in range(5):
            if k == 0:
                got[0] = batch_solve_dense(g1.model, LoadMatrix(g1.S), g1.opts(), chunk_cases=64)
            else:
                got[1] = batch_solve_sparse(g2.model, LoadMatrix(g2.S), g2.opts(), chunk_cases=100)

    ts = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for w, o in zip(want, got):
        assert np.array_equal(w.values, o.values) and np.array_equal(w.residuals, o.residuals)
        assert np.array_equal(w.iterations_per_case, o.iterations_per_case)


def test_residual_row_blocks_same_bits(monkeypatch):
    """tpf_residual_c128 splits a small batch's rows over a second grid
    dimension and combines the per-case maxima by atomicMax on the bits: the
    same numbers as one thread per case (TPF_RESID_NRB forces the split)."""
    import torch
    from paper_2403_04578_b200 import DenseOperator, GenSpec, build_network, gen_scenarios
    from paper_2403_04578_b200._device import residual_and_summary
    m = build_network(GenSpec(n_buses=301, seed=4))
    S = torch.from_numpy(gen_scenarios(m, 3000, GenSpec(n_buses=301, seed=4)).values).cuda()
    op = DenseOperator(m)
    V, it = op.solve(S)
    out = {}
    for nrb in ("1", "3", "16"):
        monkeypatch.setenv("TPF_RESID_NRB", nrb)
        r, _, _ = residual_and_summary(op.contract, S, V, it, 1e-8, op.device)
        out[nrb] = r.clone()
    assert torch.equal(out["1"], out["3"]) and torch.equal(out["1"], out["16"])
