"""Dense Tensor Power Flow on the GPU -- drop-in for ``tpflow.batch_solve_dense``.

Reference: pkg/src/tpflow/dense.py:129-205.  Same signature, same
``LoadMatrix -> VoltageBatch`` contract, same errors:

* ``ValueError("load matrix has N rows, model has M")`` (dense.py:143-146);
* non-constant-power ZIP models: the reference routes them through the
  single-case solver column by column (dense.py:147-148, 214-230); here they
  run as one GPU launch with the single-case semantics and start
  (``solve_zip``: radial feeders on the per-case tree-LU kernels, meshed or
  non-symmetric networks on the per-case fixed-pattern LU kernel); only
  complex64 or multi-device ZIP batches raise ``NotImplementedError``;
* ``numpy.linalg.LinAlgError`` from the inverse of a singular Y_dd
  (dense.py:151, uncaught in the reference too).

Setup (dense.py:150-152): radial feeders get K = -inv(Y_dd) and W = K src on
the device (``tpf_dense_setup_tree_c128``: column j of K is one tree-LU
solve, O(b^2) in all instead of the O(b^3) host inverse; equal to LAPACK's
to rounding); meshed networks (no zero-fill tree elimination) use LAPACK on
the host exactly as the reference.  The
iteration, the residual post-check and the converged mask run in libtpf.so.  ``workers`` is accepted and ignored (results are bitwise
independent of any partitioning, like the reference's, test_dense.py:96-102).
"""

from __future__ import annotations

import threading
from collections import OrderedDict

import numpy as np
import torch

from . import _capi
from ._device import (ModelContract, complex_strides, engine_dtype, host_csr, host_empty, host_loads,
                      device_workspace_slot, stream_scratch,
                      loads_to_device, ptr, require_cuda, residual_and_summary, resolve_devices, run_sliced,
                      stream_ptr)
from ._types import LoadMatrix, SolveOptions, VoltageBatch

__all__ = ["batch_solve_dense", "DenseOperator"]

_KW_CACHE: "OrderedDict[bytes, tuple[np.ndarray, np.ndarray]]" = OrderedDict()
_KW_CACHE_MAX = 8
_KW_LOCK = threading.Lock()


# radial feeders from this size: K, W built on the device (below it the host
# inverse is cheaper than the device setup and runs single-threaded in
# OpenBLAS; from about b = 100 the threaded inverse also leaves OpenBLAS's
# workers spinning, which starves the host threads staging a pageable caller
# array, tools/e2e_pageable2.py)
DEVICE_SETUP_MIN_B = 64


def device_kw(contract: ModelContract, device) -> tuple[torch.Tensor, torch.Tensor] | None:
    """K = -inv(Y_dd), W = K src on ``device`` from the tree LU of a radial
    feeder (``tpf_dense_setup_tree_c128``), or None when Y_dd has no zero-fill
    tree elimination (meshed networks: host LAPACK).  Memoised with the host
    entries (same cache, so clearing it re-times the setup)."""
    from .sparse import tree_direct
    dev = torch.device(device)
    key = contract.fingerprint() + b"|device:" + str(dev.index).encode()
    with _KW_LOCK:
        hit = _KW_CACHE.get(key)
        if hit is not None:
            _KW_CACHE.move_to_end(key)
            return hit
    t = tree_direct(contract.y_dd, contract.src)
    if t is None:
        return None
    b = contract.b

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    lvl = up(t.level_info[:t.levels + 1].astype(np.int32))
    info = up(t.node_info.astype(np.int32))
    coef = up(t.node_coef.astype(np.complex128))
    src = up(contract.src.astype(np.complex128))
    K = torch.empty((b, b), dtype=torch.complex128, device=dev)
    W = torch.empty(b, dtype=torch.complex128, device=dev)
    _capi.call("tpf_dense_setup_tree_c128", b, int(t.levels), lvl.data_ptr(), info.data_ptr(), coef.data_ptr(),
               src.data_ptr(), K.data_ptr(), W.data_ptr(), stream_ptr(dev))
    torch.cuda.current_stream(dev).synchronize()  # the inputs above are freed on return
    with _KW_LOCK:
        _KW_CACHE[key] = (K, W)
        while len(_KW_CACHE) > _KW_CACHE_MAX:
            _KW_CACHE.popitem(last=False)
    return K, W


def operator_kw(contract: ModelContract, device, setup: str = "auto"):
    """(K, W) for ``device``: device tensors from ``device_kw`` (``setup``
    "device", or "auto" with b >= DEVICE_SETUP_MIN_B, on radial feeders), else
    the host LAPACK arrays of ``dense_kw``."""
    if setup not in ("auto", "host", "device"):
        raise ValueError(f"setup must be 'auto', 'host' or 'device', not {setup!r}")
    if setup == "device" or (setup == "auto" and contract.b >= DEVICE_SETUP_MIN_B):
        kw = device_kw(contract, device)
        if kw is not None:
            return kw
    return dense_kw(contract)


def dense_kw(contract: ModelContract) -> tuple[np.ndarray, np.ndarray]:
    """K = -inv(Y_dd), W = K src (dense.py:150-152), memoised on the model's content.

    The key is a digest of Y_dd and src, so a changed model never hits a stale
    entry; a hit returns the very arrays LAPACK produced the first time (same
    bits).  Repeated batches on one feeder (the benchmark cells, bench.py:114-117)
    then skip the O(b^3) host inverse.
    """
    key = contract.fingerprint()
    with _KW_LOCK:
        hit = _KW_CACHE.get(key)
        if hit is not None:
            _KW_CACHE.move_to_end(key)
            return hit
    K = np.ascontiguousarray(-np.linalg.inv(contract.y_dd.toarray()))  # dense.py:151
    W = np.ascontiguousarray(K @ contract.src)                          # dense.py:152
    K.setflags(write=False)
    W.setflags(write=False)
    with _KW_LOCK:
        _KW_CACHE[key] = (K, W)
        while len(_KW_CACHE) > _KW_CACHE_MAX:
            _KW_CACHE.popitem(last=False)
    return K, W


class DenseOperator:
    """K = -inv(Y_dd) and W = K src resident on one device (dense.py:150-152).

    ``solve(S)`` runs the per-case-freeze fixed point on device tensors; it is
    what ``batch_solve_dense`` and ``bench.py`` call.
    """

    def __init__(self, model, device=None, dtype=None, setup: str = "auto"):
        self.device = require_cuda(device)
        self.contract = ModelContract.of(model)
        self.dtype = engine_dtype(dtype)
        b = self.contract.b
        K, W = operator_kw(self.contract, self.device, setup)
        self.setup = "device" if torch.is_tensor(K) else "host"
        # K, W in the engine's dtype (c64: rounded from the float64 inverse)
        tdt = torch.complex64 if self.dtype == np.complex64 else torch.complex128
        if torch.is_tensor(K):
            self.K = K.to(tdt)
            self.W = W.to(tdt)
        else:
            self.K = torch.from_numpy(np.array(K, dtype=self.dtype)).to(self.device)
            self.W = torch.from_numpy(np.array(W, dtype=self.dtype)).to(self.device)
        self.large = b > _capi.load().tpf_dense_max_nodes()
        self.v_flat = complex(abs(self.contract.v_s))
        self._ws: dict = {}  # per-stream scratch (_device.stream_scratch)

    @property
    def b(self) -> int:
        return self.contract.b

    def workspace(self, tau: int) -> torch.Tensor:
        lib = _capi.load()
        n = (lib.tpf_dense_large_workspace_bytes(tau, self.b) if self.large
             else lib.tpf_dense_workspace_bytes(self.b))
        return stream_scratch(self._ws, self.device, int(n))

    def solve(self, S: torch.Tensor, opts: SolveOptions = SolveOptions(), V: torch.Tensor | None = None,
              iters: torch.Tensor | None = None, kernel: str | None = None):
        """Run the iteration on a device b x tau complex128 tensor (any strides).

        Returns ``(V, iters)``; V is b x tau C-contiguous unless given.
        """
        b, tau = S.shape
        if b != self.b:
            raise ValueError(f"load matrix has {b} rows, model has {self.b}")
        tdt = torch.complex64 if self.dtype == np.complex64 else torch.complex128
        if S.dtype != tdt:
            raise ValueError(f"loads are {S.dtype}, the operator computes in {tdt}")
        if V is None:
            V = torch.empty((b, tau), dtype=tdt, device=self.device)
        if iters is None:
            iters = torch.empty(tau, dtype=torch.int32, device=self.device)
        if self.dtype == np.complex64:  # the c64 twin (include/tpf.h)
            ws = stream_scratch(self._ws, self.device, int(_capi.load().tpf_dense_c64_workspace_bytes(tau, b)))
            sn, sc = complex_strides(S)
            vn, vc = complex_strides(V)
            _capi.call("tpf_dense_fpi_c64", tau, b, S.data_ptr(), sn, sc, self.K.data_ptr(), self.W.data_ptr(),
                       self.v_flat.real, self.v_flat.imag, float(opts.tolerance), int(opts.max_iterations),
                       V.data_ptr(), vn, vc, iters.data_ptr(), ws.data_ptr(), ws.numel(),
                       stream_ptr(self.device))
            return V, iters
        ws = self.workspace(tau)
        sn, sc = complex_strides(S)
        vn, vc = complex_strides(V)
        fn = "tpf_dense_fpi_large_c128" if self.large else "tpf_dense_fpi_c128"
        if kernel is not None and not self.large:
            fn = {"ws": "tpf_dense_ws_fpi_c128", "pairs": "tpf_dense_pairs_fpi_c128"}[kernel]
        _capi.call(fn, tau, b, S.data_ptr(), sn, sc, self.K.data_ptr(), self.W.data_ptr(),
                   self.v_flat.real, self.v_flat.imag, float(opts.tolerance), int(opts.max_iterations),
                   V.data_ptr(), vn, vc, iters.data_ptr(), ws.data_ptr(), ws.numel(),
                   stream_ptr(self.device))
        return V, iters


def as_load_matrix(loads, dtype=None) -> LoadMatrix:
    """``loads`` as a LoadMatrix (complex128, dense.py:57-78).  A 2-D complex64
    array given to the complex64 twin is kept as is (no round trip through
    complex128 on the host)."""
    if isinstance(loads, LoadMatrix):
        return loads
    raw = getattr(loads, "values", loads)
    if (isinstance(raw, np.ndarray) and raw.dtype == np.complex64 and raw.ndim == 2
            and engine_dtype(dtype) == np.complex64):
        lm = object.__new__(LoadMatrix)
        object.__setattr__(lm, "values", raw)
        object.__setattr__(lm, "dims", (raw.shape[1],))
        return lm
    return LoadMatrix(np.asarray(raw))


def batch_solve_dense(model, loads: LoadMatrix, opts: SolveOptions = SolveOptions(),
                      workers: int = 1, *, device=None, devices=None, return_on_device: bool = False,
                      chunk_cases: int = 0, dtype=None) -> VoltageBatch:
    """GPU ``batch_solve_dense`` (dense.py:129-205); see module docstring.

    Host (numpy) loads go through the native chunked H2D/solve/D2H pipeline
    (``tpf_dense_solve_host_c128``) and come back as numpy arrays; with
    ``devices=[...]`` the cases are split into contiguous slices, one pipeline
    per device, run concurrently (bitwise the same result).  With
    ``return_on_device=True`` the loads are copied once and the result stays
    on the device as torch tensors.  ``dtype=numpy.complex64`` runs the c64
    twin (FP32, b <= 104, one device; pass a tolerance >= ~1e-6).
    """
    del workers  # accepted for signature compatibility; partitioning never changes bits
    loads = as_load_matrix(loads, dtype)
    if loads.n_demand != model.n_demand:
        raise ValueError(f"load matrix has {loads.n_demand} rows, model has {model.n_demand}")
    if not model.zip.is_constant_power:
        if engine_dtype(dtype) != np.complex128 or (devices is not None and len(devices) > 1):
            raise NotImplementedError("ZIP loads run in complex128 on one device")
        return solve_zip(model, loads, opts, devices[0] if devices else device, return_on_device)
    dt = engine_dtype(dtype)
    if not return_on_device and dt == np.complex128:
        return _solve_host_pipeline(model, loads, opts, resolve_devices(device, devices), chunk_cases)
    if devices is not None and len(devices) > 1:
        raise ValueError("return_on_device=True and dtype=complex64 run on a single device")
    op = DenseOperator(model, devices[0] if devices else device, dtype=dt)
    S = loads_to_device(loads.values, op.device, dt)
    V, iters = op.solve(S, opts)
    resid, mask, summ = residual_and_summary(op.contract, S, V, iters, opts.residual_tolerance, op.device)
    return finish(V, iters, resid, mask, summ, return_on_device)


# ZIP route by feeder size (tools/zip_route_probe.py, one B200): the thread-per-case
# kernel wins up to ~b = 350 (b=100: 108 vs 210 ms at tau=525,600; b=300: 92 vs
# 100 ms), the one-case-per-SM tree kernel above (b=500: 72 vs 84 ms; b=5000:
# 149 vs 558 ms).
ZIP_CHAIN_MAX_B = 384


def _zip_start(c: ModelContract, opts: SolveOptions, dev):
    """fpi_solve's start (fpi.py:141-145): ``opts.initial_voltage`` (b values,
    ValueError on a length mismatch) as a device vector in original node
    order, or None for the flat start |v_s| + 0j.  The reference's ZIP route
    (dense.py:214-230) goes through fpi_solve case by case, so it honours the
    option, unlike the constant-power batch paths."""
    if opts.initial_voltage is None:
        return None
    v = np.asarray(opts.initial_voltage, dtype=complex).ravel().copy()
    if v.shape[0] != c.b:
        raise ValueError("initial voltage length mismatch")
    return torch.from_numpy(np.ascontiguousarray(v, dtype=np.complex128)).to(dev)


def _ptr_or_null(t) -> int:
    return 0 if t is None else t.data_ptr()


def solve_zip(model, loads: LoadMatrix, opts: SolveOptions, device=None, return_on_device: bool = False):
    """ZIP loads: the reference's per-case route (dense.py:214-230 -> fpi_solve,
    fpi.py:107-206), one GPU launch per batch, each case factorizing its own
    B = Y_dd + diag(alpha_z s*) and iterating with fpi_solve's stopping rules
    and start (``opts.initial_voltage`` honoured, fpi.py:141-145).  Routing:
    radial feeders up to ZIP_CHAIN_MAX_B nodes and radial feeders the tree
    kernel does not take -> ``tpf_sparse_zip_chain_c128`` (one thread per
    case); larger radial feeders -> ``tpf_sparse_tree_zip_fpi_c128`` (one case
    per SM, on-chip tree LU); meshed or non-symmetric networks ->
    ``tpf_sparse_zip_lu_c128`` (per-case LU on a fixed fill pattern).  Only
    complex64 and multi-device ZIP batches raise NotImplementedError."""
    from ._types import SingularSystemError
    from .sparse import factorize_ydd, tree_ell, tree_schedule
    c = ModelContract.of(model)
    _zip_start(c, opts, "cpu")  # validate before any device work
    y = c.y_dd
    b = c.b
    if (y != y.T).nnz != 0:  # non-symmetric values: the general per-case LU
        return _solve_zip_lu(model, c, loads, opts, device, return_on_device)
    if b <= ZIP_CHAIN_MAX_B:  # small feeders: one thread per case beats one case per SM
        return _solve_zip_chain(model, c, loads, opts, device, return_on_device)
    tree = tree_schedule(factorize_ydd(y, count=False), c.src) if b <= 5120 else None
    ell = tree_ell(tree, c) if tree is not None else None
    if tree is None or ell is None:
        return _solve_zip_chain(model, c, loads, opts, device, return_on_device)
    dev = require_cuda(device)
    v0 = _zip_start(c, opts, dev)
    order = tree.node_info.reshape(b, 4)[:, 0]
    z = model.zip
    alpha = np.ascontiguousarray(np.concatenate([np.asarray(z.alpha_z, float)[order],
                                                 np.asarray(z.alpha_i, float)[order],
                                                 np.asarray(z.alpha_p, float)[order]]))
    ydiag = np.ascontiguousarray(y.diagonal()[order].astype(np.complex128))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    g = dict(level_info=t(tree.level_info), node_info=t(tree.node_info), node_coef=t(tree.node_coef),
             alpha=t(alpha), ydiag=t(ydiag), ell_col=t(ell[1]), ell_val=t(ell[2]))
    S = loads_to_device(loads.values, dev)
    tau = S.shape[1]
    V = torch.empty((b, tau), dtype=torch.complex128, device=dev)
    iters = torch.empty(tau, dtype=torch.int32, device=dev)
    resid = torch.empty(tau, dtype=torch.float64, device=dev)
    met = torch.zeros(tau, dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _capi.load()
    ws = torch.empty(int(lib.tpf_sparse_tree_zip_workspace_bytes(tau, b)), dtype=torch.uint8, device=dev)
    sn, sc = complex_strides(S)
    v_flat = complex(abs(c.v_s))
    if tau:
        _capi.call("tpf_sparse_tree_zip_fpi_c128", tau, b, tree.levels, g["level_info"].data_ptr(),
                   g["node_info"].data_ptr(), g["node_coef"].data_ptr(), g["alpha"].data_ptr(),
                   g["ydiag"].data_ptr(), S.data_ptr(), sn, sc, v_flat.real, v_flat.imag, _ptr_or_null(v0),
                   float(opts.tolerance),
                   int(opts.max_iterations), V.data_ptr(), tau, 1, iters.data_ptr(), ell[0],
                   g["ell_col"].data_ptr(), g["ell_val"].data_ptr(), resid.data_ptr(), met.data_ptr(),
                   status.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr(dev))
    if int(status.item()) != 0:  # assemble_fpi's splu failure (fpi.py:119-126)
        raise SingularSystemError("iteration matrix B is singular for some case (zero pivot)")
    # fpi_solve: converged = step_met and residual < residual_tolerance (fpi.py:197-198)
    mask = (met != 0) & torch.isfinite(resid) & (resid < float(opts.residual_tolerance))
    n_max = int(iters.max().item()) if tau else 0
    if return_on_device:
        return VoltageBatch(values=V, iterations=n_max, converged_mask=mask, residuals=resid,
                            iterations_per_case=iters)
    return VoltageBatch(values=V.cpu().numpy(), iterations=n_max, converged_mask=mask.cpu().numpy(),
                        residuals=resid.cpu().numpy(), iterations_per_case=iters.cpu().numpy())


def _solve_zip_chain(model, c, loads, opts, device, return_on_device):
    """ZIP loads on radial feeders, one thread per case with the per-case tree
    LU and fpi_solve rules (``tpf_sparse_zip_chain_c128``).  Meshed networks
    go to the per-case LU kernel (``_solve_zip_lu``)."""
    from ._types import SingularSystemError
    from .sparse import tree_parents
    tp = tree_parents(c.y_dd)
    if tp is None:  # meshed: per-case LU on a fixed fill pattern
        return _solve_zip_lu(model, c, loads, opts, device, return_on_device)
    dev = require_cuda(device)
    order, parent = tp
    v0 = _zip_start(c, opts, dev)
    b = c.b
    y = c.y_dd.tocsr()
    e = np.zeros(b, dtype=np.complex128)
    has = parent >= 0
    e[has] = np.asarray(y[order[has], order[parent[has]]]).ravel()
    z = model.zip
    alpha = np.concatenate([np.asarray(z.alpha_z, float)[order], np.asarray(z.alpha_i, float)[order],
                            np.asarray(z.alpha_p, float)[order]])
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    g = dict(orig=t(order.astype(np.int32)), parent=t(parent.astype(np.int32)), e=t(e),
             ydiag=t(y.diagonal()[order].astype(np.complex128)), alpha=t(alpha), src=t(c.src[order]))
    S = loads_to_device(loads.values, dev)
    tau = S.shape[1]
    V = torch.empty((b, tau), dtype=torch.complex128, device=dev)
    iters = torch.empty(tau, dtype=torch.int32, device=dev)
    resid = torch.empty(tau, dtype=torch.float64, device=dev)
    met = torch.zeros(tau, dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _capi.load()
    chunk = max(1, min(tau, (1 << 30) // (64 * b)))  # scratch: 64 B per node and case, <= 1 GB
    ws = torch.empty(int(lib.tpf_sparse_zip_chain_workspace_bytes(chunk, b)), dtype=torch.uint8, device=dev)
    sn, sc = complex_strides(S)
    v_flat = complex(abs(c.v_s))
    for lo in range(0, tau, chunk):
        hi = min(tau, lo + chunk)
        _capi.call("tpf_sparse_zip_chain_c128", hi - lo, b, g["orig"].data_ptr(), g["parent"].data_ptr(),
                   g["e"].data_ptr(), g["ydiag"].data_ptr(), g["alpha"].data_ptr(), g["src"].data_ptr(),
                   S.data_ptr() + 16 * lo * sc, sn, sc, v_flat.real, v_flat.imag, _ptr_or_null(v0),
                   float(opts.tolerance), int(opts.max_iterations), V.data_ptr() + 16 * lo, tau, 1,
                   iters.data_ptr() + 4 * lo,
                   resid.data_ptr() + 8 * lo, met.data_ptr() + lo, status.data_ptr(), ws.data_ptr(), ws.numel(),
                   stream_ptr(dev))
    return _zip_outputs(V, iters, resid, met, status, opts, return_on_device)


def _solve_zip_dense(model, c, loads, opts, device, return_on_device):
    """ZIP loads on small meshed networks (b <= 64) with the pivoting of the
    reference's splu (fpi.py:119): one thread per case, dense LU of B with
    row partial pivoting (``tpf_sparse_zip_dense_c128``)."""
    dev = require_cuda(device)
    v0 = _zip_start(c, opts, dev)
    b = c.b
    z = model.zip
    alpha = np.concatenate([np.asarray(z.alpha_z, float), np.asarray(z.alpha_i, float), np.asarray(z.alpha_p, float)])
    rp, ci, yv = host_csr(c)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    g = dict(yd=t(np.asarray(c.y_dd.toarray(), np.complex128)), alpha=t(alpha), src=t(np.asarray(c.src, np.complex128)),
             rp=t(rp), ci=t(ci), yv=t(yv))
    S = loads_to_device(loads.values, dev)
    tau = S.shape[1]
    V = torch.empty((b, tau), dtype=torch.complex128, device=dev)
    iters = torch.empty(tau, dtype=torch.int32, device=dev)
    resid = torch.empty(tau, dtype=torch.float64, device=dev)
    met = torch.zeros(tau, dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _capi.load()
    chunk = max(1, min(tau, (1 << 30) // (16 * (b * b + b) + 4 * b)))  # scratch <= 1 GB
    ws = torch.empty(int(lib.tpf_sparse_zip_dense_workspace_bytes(chunk, b)), dtype=torch.uint8, device=dev)
    sn, sc = complex_strides(S)
    v_flat = complex(abs(c.v_s))
    for lo in range(0, tau, chunk):
        hi = min(tau, lo + chunk)
        _capi.call("tpf_sparse_zip_dense_c128", hi - lo, b, g["yd"].data_ptr(), g["alpha"].data_ptr(),
                   g["src"].data_ptr(), g["rp"].data_ptr(), g["ci"].data_ptr(), g["yv"].data_ptr(),
                   S.data_ptr() + 16 * lo * sc, sn, sc, v_flat.real, v_flat.imag, _ptr_or_null(v0),
                   float(opts.tolerance), int(opts.max_iterations), V.data_ptr() + 16 * lo, tau, 1,
                   iters.data_ptr() + 4 * lo, resid.data_ptr() + 8 * lo, met.data_ptr() + lo, status.data_ptr(),
                   ws.data_ptr(), ws.numel(), stream_ptr(dev))
    return _zip_outputs(V, iters, resid, met, status, opts, return_on_device)


def _solve_zip_lu(model, c, loads, opts, device, return_on_device):
    """ZIP loads on meshed (or non-symmetric) networks: the reference's per-case
    SuperLU route (dense.py:214-230 -> fpi.py:107-206).  Up to b = 64 with
    splu's row pivoting (``_solve_zip_dense``); larger networks as one thread
    per case factorizing B = Y_dd + diag(alpha_z s*) on a fixed minimum-degree
    fill pattern without pivoting (``tpf_sparse_zip_lu_c128``).  A zero pivot
    raises SingularSystemError, as splu does for a singular B."""
    if c.b <= _capi.load().tpf_sparse_zip_dense_max_nodes():
        return _solve_zip_dense(model, c, loads, opts, device, return_on_device)
    from .sparse import zip_lu_schedule
    dev = require_cuda(device)
    sch = zip_lu_schedule(c.y_dd)
    v0 = _zip_start(c, opts, dev)
    order = sch.orig.astype(np.int64)
    b = c.b
    z = model.zip
    alpha = np.concatenate([np.asarray(z.alpha_z, float)[order], np.asarray(z.alpha_i, float)[order],
                            np.asarray(z.alpha_p, float)[order]])
    rp, ci, yv = host_csr(c)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    g = dict(orig=t(sch.orig), kinfo=t(sch.kinfo), idx=t(sch.idx), base=t(sch.base), alpha=t(alpha),
             src=t(np.asarray(c.src, np.complex128)[order]), rp=t(rp), ci=t(ci), yv=t(yv))
    S = loads_to_device(loads.values, dev)
    tau = S.shape[1]
    V = torch.empty((b, tau), dtype=torch.complex128, device=dev)
    iters = torch.empty(tau, dtype=torch.int32, device=dev)
    resid = torch.empty(tau, dtype=torch.float64, device=dev)
    met = torch.zeros(tau, dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _capi.load()
    per_case = 16 * (sch.nslot + b)
    chunk = max(1, min(tau, (1 << 30) // per_case))  # scratch <= 1 GB
    ws = torch.empty(int(lib.tpf_sparse_zip_lu_workspace_bytes(chunk, b, sch.nslot)), dtype=torch.uint8,
                     device=dev)
    sn, sc = complex_strides(S)
    v_flat = complex(abs(c.v_s))
    for lo in range(0, tau, chunk):
        hi = min(tau, lo + chunk)
        _capi.call("tpf_sparse_zip_lu_c128", hi - lo, b, sch.nslot, g["orig"].data_ptr(), g["kinfo"].data_ptr(),
                   g["idx"].data_ptr(), g["base"].data_ptr(), g["alpha"].data_ptr(), g["src"].data_ptr(),
                   g["rp"].data_ptr(), g["ci"].data_ptr(), g["yv"].data_ptr(), S.data_ptr() + 16 * lo * sc, sn,
                   sc, v_flat.real, v_flat.imag, _ptr_or_null(v0), float(opts.tolerance), int(opts.max_iterations),
                   V.data_ptr() + 16 * lo, tau, 1, iters.data_ptr() + 4 * lo, resid.data_ptr() + 8 * lo,
                   met.data_ptr() + lo, status.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr(dev))
    return _zip_outputs(V, iters, resid, met, status, opts, return_on_device)


def _zip_outputs(V, iters, resid, met, status, opts, return_on_device):
    from ._types import SingularSystemError
    if int(status.item()) != 0:  # assemble_fpi's splu failure (fpi.py:119-126)
        raise SingularSystemError("iteration matrix B is singular for some case (zero pivot)")
    # fpi_solve: converged = step_met and residual < residual_tolerance (fpi.py:197-198)
    mask = (met != 0) & torch.isfinite(resid) & (resid < float(opts.residual_tolerance))
    n_max = int(iters.max().item()) if iters.numel() else 0
    if return_on_device:
        return VoltageBatch(values=V, iterations=n_max, converged_mask=mask, residuals=resid,
                            iterations_per_case=iters)
    return VoltageBatch(values=V.cpu().numpy(), iterations=n_max, converged_mask=mask.cpu().numpy(),
                        residuals=resid.cpu().numpy(), iterations_per_case=iters.cpu().numpy())


def finish(V, iters, resid, mask, summ, on_device: bool) -> VoltageBatch:
    if on_device:
        summ_h = summ.cpu().numpy()
        return VoltageBatch(values=V, iterations=int(summ_h[0]), converged_mask=mask.bool(),
                            residuals=resid, iterations_per_case=iters)
    # D2H into page-locked blocks of torch's caching host allocator (a pageable
    # destination halves the PCIe rate); one synchronisation for all five
    host = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in (V, iters, resid, mask, summ)]
    for h, x in zip(host, (V, iters, resid, mask, summ)):
        h.copy_(x, non_blocking=True)
    torch.cuda.current_stream(V.device).synchronize()
    Vh, ih, rh, mh, sh = (h.numpy() for h in host)
    return VoltageBatch(values=Vh, iterations=int(sh[0]), converged_mask=mh.astype(bool),
                        residuals=rh, iterations_per_case=ih)


def _solve_host_pipeline(model, loads: LoadMatrix, opts: SolveOptions, devs, chunk_cases: int):
    c = ModelContract.of(model)
    rp, ci, yv = host_csr(c)
    S, sn, sc = host_loads(loads.values)
    b, tau = S.shape
    V = host_empty((b, tau), np.complex128)  # C-contiguous like dense.py:201
    iters = host_empty((tau,), np.int32)
    resid = host_empty((tau,), np.float64)
    mask = host_empty((tau,), np.uint8)
    v_flat = complex(abs(c.v_s))
    lib = _capi.load()

    def call(dev, lo, hi, slot):
        n = hi - lo
        summ = np.zeros(2, dtype=np.int32)
        if n == 0:
            return summ
        ws = device_workspace_slot(dev, lib.tpf_dense_solve_host_workspace_bytes(n, b, int(chunk_cases), yv.size),
                                   slot)
        K, W = operator_kw(c, dev)  # host LAPACK arrays, or device tensors on dev (radial, large b)
        kp = K.data_ptr() if torch.is_tensor(K) else ptr(K)
        wp = W.data_ptr() if torch.is_tensor(W) else ptr(W)
        torch.cuda.current_stream(dev).synchronize()  # the pipeline runs on its own streams
        _capi.call("tpf_dense_solve_host_c128", n, b, ptr(S) + 16 * lo * sc, sn, sc, kp, wp, ptr(rp),
                   ptr(ci), ptr(yv), ptr(c.src), v_flat.real, v_flat.imag, float(opts.tolerance),
                   int(opts.max_iterations), float(opts.residual_tolerance), ptr(V) + 16 * lo, tau, 1,
                   ptr(iters) + 4 * lo, ptr(resid) + 8 * lo, ptr(mask) + lo, ptr(summ), int(chunk_cases),
                   dev.index, ws.data_ptr(), ws.numel())
        return summ

    parts = run_sliced(devs, tau, call, (S,)) if len(devs) > 1 else [call(devs[0], 0, tau, 0)]
    return VoltageBatch(values=V, iterations=max(int(p[0]) for p in parts), converged_mask=mask.astype(bool),
                        residuals=resid, iterations_per_case=iters)
