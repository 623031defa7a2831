"""Multi-rank tau-sharding host logic, world_size 2 over gloo on CPU.

Each rank solves its contiguous slice (here with the CPU oracle standing in
for the GPU engine, which only the B200 box has), the batch iteration count is
an all_reduce(MAX) and V is all_gathered; the result must equal the unsharded
solve bit for bit (per-case freeze makes every case independent of its rank).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2403_04578_b200.shard import shard_bounds


def test_shard_bounds_cover_and_balance():
    for tau in (0, 1, 7, 100, 525600):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(tau, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == tau
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _oracle_solver(model, loads, opts):
    from oracle import tpf_oracle as orc
    from paper_2403_04578_b200 import VoltageBatch
    V, n, mask, res = orc.dense_per_case(model.admittance.y_dd, model.source_injection(), model.slack.v_s,
                                         loads.values, opts.tolerance, opts.max_iterations,
                                         opts.residual_tolerance)
    return VoltageBatch(values=V, iterations=int(n.max(initial=0)), converged_mask=mask, residuals=res,
                        iterations_per_case=n)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios
    from paper_2403_04578_b200.shard import solve_sharded
    from paper_2403_04578_b200 import SolveOptions
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = GenSpec(n_buses=35, seed=0)
        model = build_network(spec)
        loads = gen_scenarios(model, 301, spec)
        out = solve_sharded(model, loads, SolveOptions(), solve_fn=_oracle_solver)
        local = solve_sharded(model, loads, SolveOptions(), solve_fn=_oracle_solver, gather=False)
        # each rank hands over only its own (uneven) slice: slices concatenate in rank order
        cut = 170
        mine = loads.values[:, :cut] if rank == 0 else loads.values[:, cut:]
        own = solve_sharded(model, mine, SolveOptions(), solve_fn=_oracle_solver, local=True,
                            return_on_device=True)
        if rank == 0:
            q.put((out.values, out.iterations, out.iterations_per_case, out.converged_mask, out.residuals,
                   local.values.shape, local.iterations, own.values.numpy(), own.iterations))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_matches_unsharded():
    from paper_2403_04578_b200 import GenSpec, build_network, gen_scenarios, SolveOptions
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    vals, iters, per_case, mask, res, local_shape, local_it, own_vals, own_it = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = GenSpec(n_buses=35, seed=0)
    model = build_network(spec)
    loads = gen_scenarios(model, 301, spec)
    ref = _oracle_solver(model, loads, SolveOptions())
    assert np.array_equal(per_case, ref.iterations_per_case)
    assert iters == ref.iterations == local_it
    assert np.array_equal(mask, ref.converged_mask)
    assert np.abs(vals - ref.values).max() < 1e-14
    assert local_shape == (34, 151)
    assert np.abs(own_vals - vals).max() < 1e-14 and own_it == iters  # oracle BLAS blocking: not bitwise


def _stats_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2403_04578_b200.probabilistic import combine_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(rank)
        vmin = torch.from_numpy(rng.uniform(0.9, 1.0, 7))
        vmax = torch.from_numpy(rng.uniform(1.0, 1.1, 7))
        vsum = torch.from_numpy(rng.uniform(0.0, 5.0, 7))
        counts = torch.tensor([rank, 10 * (rank + 1), 5 + 2 * rank], dtype=torch.int64)
        combine_ranks(vmin, vmax, vsum, counts)
        if rank == 0:
            q.put((vmin.numpy(), vmax.numpy(), vsum.numpy(), counts.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_scenario_statistics_combine():
    """C4 scenario statistics over ranks (probabilistic.combine_ranks): per-node
    MIN / MAX / SUM of |V|, summed counts, MAX of the batch iteration count."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_stats_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    vmin, vmax, vsum, counts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r = [np.random.default_rng(k) for k in range(2)]
    parts = [(g.uniform(0.9, 1.0, 7), g.uniform(1.0, 1.1, 7), g.uniform(0.0, 5.0, 7)) for g in r]
    assert np.array_equal(vmin, np.minimum(parts[0][0], parts[1][0]))
    assert np.array_equal(vmax, np.maximum(parts[0][1], parts[1][1]))
    assert np.allclose(vsum, parts[0][2] + parts[1][2], rtol=0, atol=1e-15)
    assert counts.tolist() == [1, 30, 7]
