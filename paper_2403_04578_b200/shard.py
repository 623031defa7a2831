"""tau-sharding of one batch across ranks (one process per GPU).

SURVEY.md 8(e): every case (time step x scenario) is independent, and with
per-case freeze a case's bits do not depend on which rank solves it, so the
batch is split into contiguous tau-slices with NO data-path collective.
Collectives appear only after the solve, on device tensors (NCCL over
NVLink / NVSwitch on a GPU box; gloo on CPU tensors in the tests):

* all_reduce(MAX) of the per-rank iteration count -> the reference's batch
  ``iterations`` (dense.py:188-193 semantics: max over cases);
* optional all_gather of V / iters / residuals / mask straight from each
  rank's device-resident result (no host round trip); the gathered batch
  stays on the device (``return_on_device``) or is copied to the host once.

The solver is injectable so the host logic is testable without a GPU
(tests/test_shard_gloo.py runs it with the CPU oracle under gloo).
"""

from __future__ import annotations

from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from ._types import LoadMatrix, SolveOptions, VoltageBatch

__all__ = ["shard_bounds", "solve_sharded"]


def shard_bounds(tau: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) slice of tau for ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(tau, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _comm_device(group) -> torch.device:
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")


def _as_tensor(x, dev: torch.device) -> torch.Tensor:
    t = x if torch.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x))
    return t.to(dev)


def _gather_cols(local: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """all_gather of a (..., n_rank) tensor along its last axis with uneven n_rank
    (padded to the widest slice), on the tensor's device."""
    t = torch.movedim(local, -1, 0).contiguous()
    width = max(counts)
    pad = torch.zeros((width,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    out = [torch.empty_like(pad) for _ in counts]
    if t.dtype in (torch.complex128, torch.complex64):
        dist.all_gather([torch.view_as_real(o) for o in out], torch.view_as_real(pad), group=group)
    else:
        dist.all_gather(out, pad, group=group)
    return torch.movedim(torch.cat([o[:c] for o, c in zip(out, counts)], dim=0), 0, -1).contiguous()


def _default_solve(model, loads, opts: SolveOptions) -> VoltageBatch:
    """The GPU engine on this rank's device, result left on the device: a CUDA
    tensor slice goes straight to the operator, host loads through
    ``batch_solve_dense(..., return_on_device=True)``."""
    from ._device import residual_and_summary
    from .dense import DenseOperator, batch_solve_dense, finish
    if torch.is_tensor(loads) and loads.is_cuda:
        op = DenseOperator(model, loads.device)
        V, iters = op.solve(loads, opts)
        resid, mask, summ = residual_and_summary(op.contract, loads, V, iters, opts.residual_tolerance, op.device)
        return finish(V, iters, resid, mask, summ, True)
    return batch_solve_dense(model, loads, opts, device=torch.device("cuda", torch.cuda.current_device()),
                             return_on_device=True)


def solve_sharded(model, loads, opts: SolveOptions = SolveOptions(), solve_fn: Callable | None = None,
                  gather: bool = True, group=None, *, local: bool = False,
                  return_on_device: bool = False) -> VoltageBatch:
    """Solve this rank's tau-slice and combine the batch-level results.

    ``local=False``: ``loads`` is the whole batch (host LoadMatrix / array) and
    the rank takes its contiguous slice; ``local=True``: ``loads`` is this
    rank's own slice (host array or a CUDA tensor already resident), slices
    concatenating in rank order.  Returns the full VoltageBatch on every rank
    when ``gather`` (identical to an unsharded solve), else the local slice with
    the batch-level ``iterations``.  ``return_on_device``: torch tensors on
    the rank's device (the gathered batch never visits the host).
    """
    if solve_fn is None:
        solve_fn = _default_solve
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if local:
        mine = loads if torch.is_tensor(loads) or hasattr(loads, "values") else LoadMatrix(np.asarray(loads))
    else:
        vals = getattr(loads, "values", loads)
        lo, hi = shard_bounds(vals.shape[1], world, rank)
        mine = LoadMatrix(np.ascontiguousarray(vals[:, lo:hi]))
    part = solve_fn(model, mine, opts)
    per_case = part.iterations_per_case
    n_local = int(per_case.shape[0])
    it_local = int(per_case.max().item()) if n_local else int(part.iterations)

    def host(x):
        return x.cpu().numpy() if torch.is_tensor(x) else np.asarray(x)

    if world == 1:
        if return_on_device or not any(torch.is_tensor(x) for x in (part.values, per_case)):
            return part
        return VoltageBatch(values=host(part.values), iterations=part.iterations,
                            converged_mask=host(part.converged_mask).astype(bool), residuals=host(part.residuals),
                            iterations_per_case=host(per_case))
    dev = _comm_device(group)
    red = torch.tensor([it_local, n_local], dtype=torch.int64, device=dev)
    counts_t = [torch.zeros_like(red) for _ in range(world)]
    dist.all_gather(counts_t, red, group=group)
    iterations = max(int(c[0]) for c in counts_t)
    counts = [int(c[1]) for c in counts_t]
    if not gather:
        if return_on_device:
            return VoltageBatch(values=part.values, iterations=iterations, converged_mask=part.converged_mask,
                                residuals=part.residuals, iterations_per_case=per_case)
        return VoltageBatch(values=host(part.values), iterations=iterations,
                            converged_mask=host(part.converged_mask).astype(bool), residuals=host(part.residuals),
                            iterations_per_case=host(per_case))
    values = _gather_cols(_as_tensor(part.values, dev), counts, group)
    iters = _gather_cols(_as_tensor(per_case, dev).to(torch.int32), counts, group)
    resid = _gather_cols(_as_tensor(part.residuals, dev).to(torch.float64), counts, group)
    mask = _gather_cols(_as_tensor(part.converged_mask, dev).to(torch.uint8), counts, group)
    if return_on_device:
        return VoltageBatch(values=values, iterations=iterations, converged_mask=mask.bool(), residuals=resid,
                            iterations_per_case=iters)
    return VoltageBatch(values=values.cpu().numpy(), iterations=iterations,
                        converged_mask=mask.cpu().numpy().astype(bool), residuals=resid.cpu().numpy(),
                        iterations_per_case=iters.cpu().numpy())
