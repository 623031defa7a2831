"""Probabilistic power flow (config C4): scenario batches generated,
solved and reduced on the device.

The reference reaches C4 by calling ``gen_scenarios`` (synth.py:131-156) once per
scenario and ``batch_solve_dense`` on the result (dense.py:129-205); its 841 GB
of loads cannot exist on a host.  Here every scenario batch s (seed
``first_seed + s``, the reference's GenSpec semantics) is generated in HBM by
``synth.gen_scenarios_device``, solved by the dense (or sparse) engine with the
fused residual post-check and summary, and folded into per-node statistics of
|V| by ``tpf_voltage_stats_c128`` (deterministic, no atomics); only the
statistics, counts and optional sampled columns leave the device.  Under
``torch.distributed`` the scenarios are dealt round-robin over ranks and the
statistics are combined by all-reduce (MIN / MAX / SUM) -- the one exchange step
of the path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _capi
from ._device import complex_strides, require_cuda, residual_and_summary, stream_ptr
from ._types import SolveOptions

__all__ = ["ScenarioStats", "probabilistic_pf", "combine_ranks"]


@dataclass
class ScenarioStats:
    """Per-node |V| statistics over every case of every scenario, and counts."""

    vmin: np.ndarray          # float64[b]
    vmean: np.ndarray         # float64[b]
    vmax: np.ndarray          # float64[b]
    n_scenarios: int
    n_cases: int
    nonconverged: int         # cases failing the residual post-check (dense.py:198-199)
    max_iterations: int       # max over scenarios of the batch iteration count
    sum_iterations: int       # sum of the per-case update counts
    samples: dict = field(default_factory=dict)  # scenario -> (cols, S[:, cols], V[:, cols]) on the host


def combine_ranks(vmin, vmax, vsum, counts, group=None) -> None:
    """All-reduce of the per-rank statistics (in place): MIN / MAX / SUM of the
    per-node |V| arrays, SUM of the non-converged and iteration counts, MAX of
    the batch iteration count (counts = [nonconverged, sum_iterations, max])."""
    import torch.distributed as dist
    dist.all_reduce(vmin, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(vmax, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(vsum, op=dist.ReduceOp.SUM, group=group)
    mx = counts[2:3].clone()
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    counts[2] = mx[0]


def probabilistic_pf(model, n_scenarios: int, tau: int = 525600, *, method: str = "dense", first_seed: int = 1000,
                     load_scale: float = 1.0, opts: SolveOptions = SolveOptions(), device=None,
                     sample: dict | None = None, group=None) -> ScenarioStats:
    """Solve ``n_scenarios`` scenario batches of ``tau`` cases each on the device.

    ``sample``: {scenario: column indices} -- those columns' loads and voltages
    are copied to the host (parity checks against the oracle).  With
    ``torch.distributed`` initialised (or ``group``), rank r takes scenarios
    r, r + world, ...; every rank returns the combined statistics.
    """
    from . import GenSpec
    from .dense import DenseOperator
    from .sparse import SparseOperator
    from .synth import gen_scenarios_device
    import torch.distributed as dist

    dev = require_cuda(device)
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    op = DenseOperator(model, dev) if method == "dense" else SparseOperator(model, dev)
    b = op.b
    lib = _capi.load()
    V = torch.empty((b, tau), dtype=torch.complex128, device=dev)
    iters = torch.empty(tau, dtype=torch.int32, device=dev)
    csr = op.contract.csr_on(dev)
    post = (torch.empty(tau, dtype=torch.float64, device=dev), torch.empty(tau, dtype=torch.uint8, device=dev),
            torch.empty(2, dtype=torch.int32, device=dev))
    vmin = torch.full((b,), np.inf, dtype=torch.float64, device=dev)
    vmax = torch.full((b,), -np.inf, dtype=torch.float64, device=dev)
    vsum = torch.zeros(b, dtype=torch.float64, device=dev)
    ws = torch.empty(int(lib.tpf_voltage_stats_workspace_bytes(tau, b)), dtype=torch.uint8, device=dev)
    counts = torch.zeros(3, dtype=torch.int64, device=dev)  # nonconverged, sum of iterations, max batch iterations
    samples = {}
    fused = method != "dense"
    mine = range(rank, n_scenarios, world)
    for k, s in enumerate(mine):
        spec = GenSpec(n_buses=b + 1, seed=first_seed + s, load_scale=load_scale)
        S = gen_scenarios_device(model, tau, spec, device=dev)
        if fused:
            op.solve(S, opts, V=V, iters=iters, resid=post[0])
        else:
            op.solve(S, opts, V=V, iters=iters)
        resid, mask, summ = residual_and_summary(op.contract, S, V, iters, opts.residual_tolerance, dev, csr=csr,
                                                 out=post, have_resid=fused)
        vn, vc = complex_strides(V)
        _capi.call("tpf_voltage_stats_c128", tau, b, V.data_ptr(), vn, vc, vmin.data_ptr(), vmax.data_ptr(),
                   vsum.data_ptr(), 1, ws.data_ptr(), ws.numel(), stream_ptr(dev))
        counts[0] += tau - summ[1].to(torch.int64)
        counts[1] += iters.sum(dtype=torch.int64)
        counts[2] = torch.maximum(counts[2], summ[0].to(torch.int64))
        if sample and s in sample:
            cols = torch.as_tensor(np.asarray(sample[s]), dtype=torch.int64, device=dev)
            samples[s] = (np.asarray(sample[s]), S[:, cols].cpu().numpy(), V[:, cols].cpu().numpy(),
                          iters[cols].cpu().numpy())
        del S
    if world > 1:
        combine_ranks(vmin, vmax, vsum, counts, group)
    n_cases = n_scenarios * tau
    c = counts.cpu().numpy()
    return ScenarioStats(vmin=vmin.cpu().numpy(), vmean=(vsum / n_cases).cpu().numpy(), vmax=vmax.cpu().numpy(),
                         n_scenarios=n_scenarios, n_cases=n_cases, nonconverged=int(c[0]),
                         max_iterations=int(c[2]), sum_iterations=int(c[1]), samples=samples)
