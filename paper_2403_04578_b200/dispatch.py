"""Method-string dispatcher, mirror of ``tpflow.bench.solve_batch`` (bench.py:96-111).

"dense" and "sparse" route to the GPU engine.  "fpi" and "nr" are the
reference's per-case loops (bench.py:77-93), which are not on the batched hot
path; they raise NotImplementedError naming the reference route.
"""

from __future__ import annotations

from ._types import LoadMatrix, SolveOptions

# bench.py:35
METHODS = ("dense", "sparse", "fpi", "nr")


def solve_batch(method: str, model, loads: LoadMatrix, opts: SolveOptions = SolveOptions(),
                workers: int = 1, **kwargs):
    """Run one batch with the chosen method; column j of the result is case j."""
    if method == "dense":
        from .dense import batch_solve_dense
        return batch_solve_dense(model, loads, opts, workers=workers, **kwargs)
    if method == "sparse":
        from .sparse import batch_solve_sparse
        return batch_solve_sparse(model, loads, opts, **kwargs)
    if method in ("fpi", "nr"):
        raise NotImplementedError(
            f"method {method!r} is the reference's per-case loop (tpflow.bench._batch_via_cases), "
            "not the batched hot path this engine accelerates")
    raise ValueError(f"unknown method {method!r}")
