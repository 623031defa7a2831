"""CPU oracle for the Tensor Power Flow hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in numpy/scipy, the reference `tpflow` algorithms on
the north-star path so that the CUDA engine can be checked against them on the
GPU box (where `/root/reference` does not exist).  It is imported only by
`tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference`
legs of `bench.py`.  The product package never imports it.

Parity of this restatement with the reference is pinned by
`tests/golden/*.npz`, produced by `tests/golden/make_golden.py` running the
reference itself (`tpflow` imported read-only from /root/reference/pkg/src),
and checked in `tests/test_oracle_golden.py`.

Inputs are plain arrays (the reference's NetworkModel is reduced to its
hot-path contract):

* ``y_dd``  -- scipy.sparse matrix, b x b complex (network.py:99-128)
* ``src``   -- complex[b] = Y_ds v_s, ``NetworkModel.source_injection``
               (network.py:270-274)
* ``v_s``   -- complex slack voltage (network.py:53-61)
* ``S``     -- complex b x tau load matrix, column j = case j (dense.py:57-78)
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np
from scipy import sparse
from scipy.sparse.linalg import splu

# fpi.py:39-41
ZERO_VOLTAGE_GUARD = 1e-12


def residual_per_case(y_dd, src, V, S):
    """Constant-power branch of ``residual_per_case`` (fpi.py:221-240).

    ``max_i |s_i + v_i conj(src_i + (Y_dd v)_i)|`` per column.
    """
    V = np.asarray(V, dtype=complex)
    S = np.asarray(S, dtype=complex)
    src = np.asarray(src, dtype=complex)
    if V.ndim == 2:
        src = src[:, None]
    mismatch = S + V * np.conj(src + y_dd @ V)
    return np.abs(mismatch).max(axis=0)


def safe_residuals(y_dd, src, V, S):
    """``_safe_residuals`` (dense.py:208-211)."""
    with np.errstate(invalid="ignore", over="ignore"):
        res = residual_per_case(y_dd, src, V, S)
    return np.atleast_1d(np.asarray(res, dtype=float))


def dense_operators(y_dd, src):
    """Setup of ``batch_solve_dense`` (dense.py:150-152): K = -inv(Y_dd), W = K src."""
    K = -np.linalg.inv(y_dd.toarray())
    W = K @ np.asarray(src, dtype=complex)
    return K, W


def _dense_step(K, s_conj, W, v, v_next, u, lo, hi):
    """One joint update on columns [lo, hi) (dense.py:114-126)."""
    cols = slice(lo, hi)
    np.conjugate(v[:, cols], out=u[:, cols])
    np.divide(s_conj[:, cols], u[:, cols], out=u[:, cols])
    np.matmul(K, u[:, cols], out=v_next[:, cols])
    np.add(v_next[:, cols], W[:, None], out=v_next[:, cols])
    np.subtract(v_next[:, cols], v[:, cols], out=u[:, cols])
    return float(np.abs(u[:, cols]).max(initial=0.0))


def dense_joint(y_dd, src, v_s, S, tol=1e-10, max_iter=100,
                residual_tol=1e-8, workers=1, K=None, W=None):
    """Restatement of ``batch_solve_dense`` (dense.py:129-205), joint stop rule.

    Returns ``(V, iterations, converged_mask, residuals)`` with V b x tau
    C-contiguous, exactly as the reference's ``VoltageBatch``.
    """
    S = np.asarray(S, dtype=complex)
    b, tau = S.shape
    if K is None or W is None:
        K, W = dense_operators(y_dd, src)
    s_conj = np.asfortranarray(np.conj(S))
    v = np.full((b, tau), abs(v_s) * (1.0 + 0.0j), order="F")
    v_next = np.empty_like(v)
    scratch = np.empty_like(v)
    workers = max(1, int(workers))
    edges = np.linspace(0, tau, workers + 1).astype(int)
    chunks = [(lo, hi) for lo, hi in zip(edges[:-1], edges[1:]) if hi > lo]
    pool = ThreadPoolExecutor(max_workers=workers) if len(chunks) > 1 else None
    n = 0
    try:
        with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
            while n < max_iter:
                # zero-voltage guard (dense.py:170-172)
                small = np.abs(v) < ZERO_VOLTAGE_GUARD
                if small.any():
                    np.copyto(v, ZERO_VOLTAGE_GUARD * (1.0 + 0.0j), where=small)
                if pool is None:
                    deltas = [_dense_step(K, s_conj, W, v, v_next, scratch, lo, hi)
                              for lo, hi in chunks]
                else:
                    deltas = list(pool.map(
                        lambda c, a=v, z=v_next: _dense_step(K, s_conj, W, a, z, scratch, *c),
                        chunks))
                v, v_next = v_next, v
                n += 1
                d = np.asarray(deltas)
                # stop rule (dense.py:189-193)
                if np.all(np.isfinite(d)) and d.max() < tol:
                    break
    finally:
        if pool is not None:
            pool.shutdown()
    res = safe_residuals(y_dd, src, v, S)
    mask = np.isfinite(res) & (res < residual_tol)
    return np.ascontiguousarray(v), n, mask, res


def dense_per_case(y_dd, src, v_s, S, tol=1e-10, max_iter=100,
                   residual_tol=1e-8, K=None, W=None):
    """Per-case freeze restatement: the semantics of the GPU engine.

    Column j is updated with the reference's arithmetic (dense.py:114-126)
    until its own ``max_i |dv_ij| < tol`` (finite), then frozen.  Returns
    ``(V, n_per_case, converged_mask, residuals)``; ``max(n_per_case)`` equals
    the reference's joint iteration count (test_dense.py:72-79).
    """
    S = np.asarray(S, dtype=complex)
    b, tau = S.shape
    if K is None or W is None:
        K, W = dense_operators(y_dd, src)
    s_conj = np.conj(S)
    V = np.full((b, tau), abs(v_s) * (1.0 + 0.0j))
    n_case = np.zeros(tau, dtype=np.int32)
    active = np.arange(tau)
    with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
        for _ in range(max_iter):
            if active.size == 0:
                break
            v = V[:, active]
            small = np.abs(v) < ZERO_VOLTAGE_GUARD
            if small.any():
                v = np.where(small, ZERO_VOLTAGE_GUARD * (1.0 + 0.0j), v)
            u = s_conj[:, active] / np.conj(v)
            v_next = K @ u + W[:, None]
            d = np.abs(v_next - v).max(axis=0, initial=0.0)
            V[:, active] = v_next
            n_case[active] += 1
            done = np.isfinite(d) & (d < tol)
            active = active[~done]
    res = safe_residuals(y_dd, src, V, S)
    mask = np.isfinite(res) & (res < residual_tol)
    return V, n_case, mask, res


def assemble_block_system(y_dd, src, S):
    """Block-diagonal system of ``assemble_block_system`` (sparse.py:115-164).

    Returns ``(M_dot, H_dot, zero_mask)``; block j = -diag(1/s_j*) Y_dd with
    zero-load rows kept unscaled and H = -src there (sparse.py:144-151).
    """
    y = sparse.csc_matrix(y_dd, dtype=complex)
    S = np.asarray(S, dtype=complex)
    b, tau = S.shape
    nnz = y.nnz
    s_conj = np.conj(S)
    zero = s_conj == 0
    with np.errstate(divide="ignore", invalid="ignore"):
        row_s = s_conj.T[:, y.indices]
        data = np.where(zero.T[:, y.indices], y.data[None, :],
                        -(y.data[None, :] / row_s)).ravel()
        h = np.where(zero.T, -src[None, :], src[None, :] / s_conj.T)
    indices = np.tile(y.indices, tau) + np.repeat(np.arange(tau, dtype=np.int64) * b, nnz)
    indptr = np.concatenate([[0], np.tile(np.diff(y.indptr), tau)]).cumsum()
    M = sparse.csc_matrix((data, indices, indptr), shape=(b * tau, b * tau))
    return M, h.ravel(), zero


def sparse_block(y_dd, src, v_s, S, tol=1e-10, max_iter=100, residual_tol=1e-8):
    """Restatement of ``batch_solve_sparse`` (sparse.py:167-207)."""
    S = np.asarray(S, dtype=complex)
    b, tau = S.shape
    M, H, zero = assemble_block_system(y_dd, src, S)
    lu = splu(M)
    zero_flat = zero.T.ravel()
    v = np.full(b * tau, abs(v_s) * (1.0 + 0.0j))
    n = 0
    with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
        while n < max_iter:
            v = np.where(np.abs(v) < ZERO_VOLTAGE_GUARD, ZERO_VOLTAGE_GUARD * (1.0 + 0.0j), v)
            recip = 1.0 / np.conj(v)
            recip[zero_flat] = 0.0
            v_next = lu.solve(recip + H)
            delta = np.abs(v_next - v).max(initial=0.0)
            v = v_next
            n += 1
            if np.isfinite(delta) and delta < tol:
                break
    V = np.ascontiguousarray(v.reshape(tau, b).T)
    res = safe_residuals(y_dd, src, V, S)
    mask = np.isfinite(res) & (res < residual_tol)
    return V, n, mask, res


def fpi_single(y_dd, src, v_s, s, tol=1e-10, max_iter=100, residual_tol=1e-8):
    """Constant-power ``fpi_solve`` (fpi.py:107-206): returns (v, iterations, converged)."""
    s = np.asarray(s, dtype=complex).ravel()
    a = np.conj(s)
    lu = splu(sparse.csc_matrix(y_dd, dtype=complex))
    w = -lu.solve(np.asarray(src, dtype=complex))
    v = np.full(s.shape[0], abs(v_s) * (1.0 + 0.0j))
    if np.all(a == 0):
        res = float(residual_per_case(y_dd, src, w, s))
        return w.copy(), 1, res < residual_tol
    n = 0
    step_met = False
    with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
        while n < max_iter:
            small = np.abs(v) < ZERO_VOLTAGE_GUARD
            if small.any():
                v = np.where(small, ZERO_VOLTAGE_GUARD * (1.0 + 0.0j), v)
            v_next = -lu.solve(a * (1.0 / np.conj(v))) + w
            n += 1
            if not np.all(np.isfinite(v_next.view(float))):
                v = v_next
                break
            step = np.abs(v_next - v).max()
            v = v_next
            if step < tol:
                step_met = True
                break
    with np.errstate(invalid="ignore", over="ignore"):
        res = float(residual_per_case(y_dd, src, v, s))
    return v, n, bool(step_met and res < residual_tol)


# --------------------------------------------------------------------- ZIP


def zip_residual(y_dd, src, az, ai, ap, v, s):
    """``residual_per_case`` with ZIP load power (fpi.py:209-240), one case."""
    v = np.asarray(v, dtype=complex)
    s = np.asarray(s, dtype=complex)
    s_load = az * s * np.abs(v) ** 2 + ai * s * v + ap * s
    return float(np.abs(s_load + v * np.conj(src + y_dd @ v)).max())


def fpi_single_zip(y_dd, src, v_s, az, ai, ap, s, tol=1e-10, max_iter=100, residual_tol=1e-8):
    """``fpi_solve`` with ZIP loads (assemble_fpi fpi.py:107-127, loop fpi.py:137-206).

    Returns (v, iterations, converged, residual, step_met).
    """
    s = np.asarray(s, dtype=complex).ravel()
    sc = np.conj(s)
    a = ap * sc
    B = (sparse.diags(az * sc) + sparse.csc_matrix(y_dd, dtype=complex)).tocsc()
    c = np.asarray(src, dtype=complex) + ai * sc
    lu = splu(B)
    w = -lu.solve(c.astype(complex))
    v = np.full(s.shape[0], abs(v_s) * (1.0 + 0.0j))
    if np.all(a == 0):
        res = zip_residual(y_dd, src, az, ai, ap, w, s)
        return w.copy(), 1, res < residual_tol, res, True
    n = 0
    step_met = False
    with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
        while n < max_iter:
            small = np.abs(v) < ZERO_VOLTAGE_GUARD
            if small.any():
                v = np.where(small, ZERO_VOLTAGE_GUARD * (1.0 + 0.0j), v)
            v_next = -lu.solve(a * (1.0 / np.conj(v))) + w
            n += 1
            if not np.all(np.isfinite(v_next.view(float))):
                v = v_next
                break
            step = np.abs(v_next - v).max()
            v = v_next
            if step < tol:
                step_met = True
                break
    with np.errstate(invalid="ignore", over="ignore"):
        res = zip_residual(y_dd, src, az, ai, ap, v, s)
    return v, n, bool(step_met and res < residual_tol), res, step_met


def dense_zip_batch(y_dd, src, v_s, az, ai, ap, S, tol=1e-10, max_iter=100, residual_tol=1e-8):
    """``_batch_via_single`` (dense.py:214-230): per-case ZIP fpi_solve.

    Returns (V, n_case, mask, residuals, batch_iterations).
    """
    S = np.asarray(S, dtype=complex)
    b, tau = S.shape
    V = np.empty((b, tau), dtype=complex)
    n = np.zeros(tau, dtype=np.int64)
    mask = np.zeros(tau, dtype=bool)
    res = np.empty(tau)
    for j in range(tau):
        V[:, j], n[j], mask[j], res[j], _ = fpi_single_zip(y_dd, src, v_s, az, ai, ap, S[:, j], tol, max_iter,
                                                           residual_tol)
    return V, n, mask, res, int(n.max(initial=0))
