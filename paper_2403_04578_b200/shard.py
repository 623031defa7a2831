"""tau-sharding of one batch across ranks (one process per GPU).

SURVEY.md 8(e): every case (time step x scenario) is independent, and with
per-case freeze a case's bits do not depend on which rank solves it, so the
batch is split into contiguous tau-slices with NO data-path collective.
Collectives appear only after the solve:

* all_reduce(MAX) of the per-rank iteration count -> the reference's batch
  ``iterations`` (dense.py:188-193 semantics: max over cases);
* all_reduce(SUM) of the converged count;
* optional all_gather of V / iters / residuals / mask (NCCL over NVLink on a
  GPU box; gloo in the CPU tests).

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


def _gather_cols(local: np.ndarray, counts: list[int], group=None) -> np.ndarray:
    """all_gather of a (..., n_rank) array along its last axis with uneven n_rank."""
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")
    t = torch.from_numpy(np.ascontiguousarray(np.moveaxis(local, -1, 0))).to(dev)
    width = max(counts)
    pad = torch.zeros((width,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
    pad[: t.shape[0]] = t
    out = [torch.empty_like(pad) for _ in counts]
    if t.dtype == torch.complex128:
        dist.all_gather([torch.view_as_real(o) for o in out], torch.view_as_real(pad), group=group)
    else:
        dist.all_gather(out, pad, group=group)
    parts = [o[:c].cpu().numpy() for o, c in zip(out, counts)]
    return np.moveaxis(np.concatenate(parts, axis=0), 0, -1)


def solve_sharded(model, loads: LoadMatrix, opts: SolveOptions = SolveOptions(),
                  solve_fn: Callable | None = None, gather: bool = True, group=None) -> VoltageBatch:
    """Solve this rank's tau-slice and combine the batch-level results.

    Returns the full VoltageBatch on every rank when ``gather`` (identical to
    an unsharded solve), else the local slice with batch-level
    ``iterations``.
    """
    if solve_fn is None:
        from .dense import batch_solve_dense as solve_fn
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    tau = loads.tau
    lo, hi = shard_bounds(tau, world, rank)
    part = solve_fn(model, LoadMatrix(np.ascontiguousarray(loads.values[:, lo:hi])), opts)
    it_local = int(np.max(part.iterations_per_case, initial=0)) if len(part.iterations_per_case) \
        else int(part.iterations)
    if world == 1:
        return part
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")
    red = torch.tensor([it_local], dtype=torch.int64, device=dev)
    dist.all_reduce(red, op=dist.ReduceOp.MAX, group=group)
    iterations = int(red.item())
    if not gather:
        return VoltageBatch(values=part.values, iterations=iterations, converged_mask=part.converged_mask,
                            residuals=part.residuals, iterations_per_case=part.iterations_per_case)
    counts = [shard_bounds(tau, world, r)[1] - shard_bounds(tau, world, r)[0] for r in range(world)]
    values = _gather_cols(np.asarray(part.values), counts, group)
    iters = _gather_cols(np.asarray(part.iterations_per_case, dtype=np.int32), counts, group)
    resid = _gather_cols(np.asarray(part.residuals, dtype=np.float64), counts, group)
    mask = _gather_cols(np.asarray(part.converged_mask, dtype=np.uint8), counts, group).astype(bool)
    return VoltageBatch(values=np.ascontiguousarray(values), iterations=iterations, converged_mask=mask,
                        residuals=resid, iterations_per_case=iters)
