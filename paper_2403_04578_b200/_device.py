"""Host <-> device plumbing shared by the dense and sparse solvers (PyTorch is
used for device memory and streams only; all arithmetic runs in libtpf.so)."""

from __future__ import annotations

from dataclasses import dataclass

import hashlib
import threading

import numpy as np
import torch
from scipy import sparse

from . import _capi


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the TPF engine needs a CUDA device (sm_100a); there is no CPU fallback")
    _capi.load()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    return torch.device("cuda", dev.index if dev.index is not None else torch.cuda.current_device())


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


@dataclass
class ModelContract:
    """The four things the hot path reads from a network model."""

    b: int
    y_dd: sparse.csr_matrix
    src: np.ndarray
    v_s: complex
    constant_power: bool

    @classmethod
    def of(cls, model) -> "ModelContract":
        y = sparse.csr_matrix(model.admittance.y_dd, dtype=complex)
        y.sort_indices()
        return cls(b=int(model.n_demand), y_dd=y,
                   src=np.ascontiguousarray(np.asarray(model.source_injection(), dtype=complex)),
                   v_s=complex(model.slack.v_s),
                   constant_power=bool(model.zip.is_constant_power))

    def fingerprint(self) -> bytes:
        """Digest of everything the solve reads (Y_dd pattern and values, src, v_s)."""
        h = hashlib.blake2b(digest_size=20)
        y = self.y_dd
        for a in (np.asarray(y.shape, dtype=np.int64), y.indptr, y.indices, y.data, self.src,
                  np.asarray([self.v_s], dtype=complex)):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.digest()

    def row_order(self) -> np.ndarray:
        """A depth-first order of Y_dd's graph (every component): the residual
        kernel visits rows in it, so a row's neighbours were read moments
        before and still sit in L1 (C2: 0.50 -> 0.42 ms, tools/resid_order_probe.py)."""
        from scipy.sparse import csgraph
        y = self.y_dd
        pat = sparse.csr_matrix((np.ones(y.indices.size), y.indices, y.indptr), shape=y.shape)
        seen = np.zeros(self.b, dtype=bool)
        parts = []
        for r in range(self.b):
            if not seen[r]:
                part = csgraph.depth_first_order(pat, r, directed=False, return_predecessors=False)
                seen[part] = True
                parts.append(part)
        return np.concatenate(parts).astype(np.int32) if parts else np.zeros(0, dtype=np.int32)

    def csr_on(self, device: torch.device):
        """Y_dd (CSR), src and the residual's row order on ``device``."""
        rp = torch.from_numpy(self.y_dd.indptr.astype(np.int32)).to(device)
        ci = torch.from_numpy(self.y_dd.indices.astype(np.int32)).to(device)
        val = torch.from_numpy(np.ascontiguousarray(self.y_dd.data)).to(device)
        src = torch.from_numpy(self.src).to(device)
        order = torch.from_numpy(self.row_order()).to(device)
        return rp, ci, val, src, order


def complex_strides(t: torch.Tensor) -> tuple[int, int]:
    """(node_stride, case_stride) in complex elements of a b x tau tensor."""
    return int(t.stride(0)), int(t.stride(1))


def loads_to_device(values: np.ndarray, device: torch.device, dtype=np.complex128) -> torch.Tensor:
    """Copy a b x tau complex load matrix to the device keeping its C/F order
    (a tensor already there is used as is)."""
    if isinstance(values, torch.Tensor):
        tdt = torch.complex64 if np.dtype(dtype) == np.complex64 else torch.complex128
        return values.to(device=device, dtype=tdt)
    arr = np.asarray(values, dtype=dtype)
    if not (arr.flags.c_contiguous or arr.flags.f_contiguous):
        arr = np.ascontiguousarray(arr)
    host = torch.from_numpy(arr)
    out = torch.empty_strided(host.shape, host.stride(), dtype=host.dtype, device=device)
    out.copy_(host)
    return out


def residual_and_summary(contract: ModelContract, S: torch.Tensor, V: torch.Tensor,
                         iters: torch.Tensor, residual_tol: float, device: torch.device,
                         csr=None, out=None, have_resid: bool = False):
    """Residual post-check and converged mask on the device (dense.py:198-199).

    ``csr`` (from ``contract.csr_on``) and ``out`` = (resid, mask, summ) may be
    passed in to reuse device buffers: then the call only enqueues kernels.
    ``have_resid``: ``out[0]`` already holds the residuals (a solver that fuses
    the post-check, ``SparseOperator.solve(..., resid=)``); only the summary runs.
    """
    tau = V.shape[1]
    if out is None:
        resid = torch.empty(tau, dtype=torch.float64, device=device)
        mask = torch.empty(tau, dtype=torch.uint8, device=device)
        summ = torch.empty(2, dtype=torch.int32, device=device)
    else:
        resid, mask, summ = out
    st = stream_ptr(device)
    sn, sc = complex_strides(S)
    vn, vc = complex_strides(V)
    if not have_resid:
        rp, ci, val, src, order = csr if csr is not None else contract.csr_on(device)
        if V.dtype == torch.complex64:
            _capi.call("tpf_residual_c64", tau, contract.b, S.data_ptr(), sn, sc, V.data_ptr(), vn, vc,
                       rp.data_ptr(), ci.data_ptr(), val.data_ptr(), src.data_ptr(), resid.data_ptr(), st)
        else:
            _capi.call("tpf_residual_order_c128", tau, contract.b, S.data_ptr(), sn, sc, V.data_ptr(), vn, vc,
                       rp.data_ptr(), ci.data_ptr(), val.data_ptr(), src.data_ptr(), order.data_ptr(),
                       resid.data_ptr(), st)
    _capi.call("tpf_batch_summary", tau, iters.data_ptr(), resid.data_ptr(), float(residual_tol),
               mask.data_ptr(), summ.data_ptr(), st)
    return resid, mask, summ


def engine_dtype(dtype) -> np.dtype:
    """complex128 (default, the reference's arithmetic) or complex64 (the c64 twins)."""
    dt = np.dtype(np.complex128 if dtype is None else dtype)
    if dt not in (np.dtype(np.complex128), np.dtype(np.complex64)):
        raise ValueError(f"dtype must be complex128 or complex64, got {dt}")
    return dt


def host_empty(shape, dtype) -> np.ndarray:
    """Page-locked host array from torch's caching host allocator (DMA-able, reused)."""
    tdt = {np.complex128: torch.complex128, np.float64: torch.float64, np.int32: torch.int32,
           np.uint8: torch.uint8}[np.dtype(dtype).type]
    return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()


def host_loads(values) -> tuple[np.ndarray, int, int]:
    """The load matrix as C- or F-contiguous complex128 plus its complex strides."""
    arr = np.asarray(values, dtype=np.complex128)
    if not (arr.flags.c_contiguous or arr.flags.f_contiguous):
        arr = np.ascontiguousarray(arr)
    return arr, arr.strides[0] // 16, arr.strides[1] // 16


def host_csr(contract: ModelContract):
    y = contract.y_dd
    return (np.ascontiguousarray(y.indptr, dtype=np.int32), np.ascontiguousarray(y.indices, dtype=np.int32),
            np.ascontiguousarray(y.data, dtype=np.complex128))


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# Host-pipeline scratch, one grow-only buffer per (device, slot) and per
# calling THREAD: the native pipelines release the GIL, so two Python threads
# solving on one device must never carve the same arena.  Thread-
# local storage also drops a thread's buffers when the thread ends.
_WS_TLS = threading.local()


def resolve_devices(device=None, devices=None) -> list[torch.device]:
    """The CUDA devices of one call: ``devices`` (a list) wins over ``device``."""
    if devices is None:
        return [require_cuda(device)]
    devs = [require_cuda(d) for d in devices]
    if not devs:
        raise ValueError("devices must name at least one CUDA device")
    return devs


def case_slices(tau: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous, near-equal case ranges [lo, hi) (SURVEY 8(e) partitioning)."""
    base, extra = divmod(tau, parts)
    out, lo = [], 0
    for k in range(parts):
        hi = lo + base + (1 if k < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


class _PinScope:
    """Page-lock host arrays for the duration of a multi-device call, so the
    per-device pipelines (which would otherwise each register the same span)
    all see page-locked memory and never unregister under each other."""

    def __init__(self, *arrays):
        self.arrays = [a for a in arrays if a is not None and a.nbytes > 0]
        self.done = []

    def __enter__(self):
        lib = _capi.load()
        for a in self.arrays:
            if lib.tpf_host_pin(a.ctypes.data, a.nbytes) == 1:  # 0: already page-locked or not pinnable
                self.done.append(a.ctypes.data)
        return self

    def __exit__(self, *exc):
        lib = _capi.load()
        for p in self.done:
            lib.tpf_host_unpin(p)
        return False


def run_sliced(devices: list[torch.device], tau: int, call, arrays) -> list:
    """Run ``call(device, lo, hi, slot)`` for contiguous case slices, one per
    device entry, concurrently (the C pipelines release the GIL).  ``arrays``
    are the host buffers the calls read/write (page-locked for the call)."""
    import threading
    slices = case_slices(tau, len(devices))
    results: list = [None] * len(devices)
    errors: list = []

    def work(k):
        lo, hi = slices[k]
        try:
            with torch.cuda.device(devices[k]):
                results[k] = call(devices[k], lo, hi, k)
        except BaseException as exc:  # re-raised in the caller's thread
            errors.append(exc)

    with _PinScope(*arrays):
        threads = [threading.Thread(target=work, args=(k,)) for k in range(1, len(devices))]
        for t in threads:
            t.start()
        work(0)
        for t in threads:
            t.join()
    if errors:
        raise errors[0]
    return results


_STREAM_WS_LOCK = threading.Lock()


def stream_scratch(cache: dict, device: torch.device, nbytes: int) -> torch.Tensor:
    """Grow-only device scratch of an operator, one buffer per CUDA stream:
    solves queued on different streams (threads, or one thread alternating
    streams) never share scratch, and a buffer is reused only by work that its
    stream orders after the previous use.  A grown buffer replaces the old one
    on the same stream (torch's allocator keeps the freed block for that
    stream's later work)."""
    key = (str(device), torch.cuda.current_stream(device).cuda_stream)
    with _STREAM_WS_LOCK:
        ws = cache.get(key)
        if ws is None or ws.numel() < nbytes:
            cache.pop(key, None)
            ws = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
            cache[key] = ws
    return ws


def device_workspace_slot(device: torch.device, nbytes: int, slot: int) -> torch.Tensor:
    """Grow-only scratch for one host-pipeline call: one buffer per (calling
    thread, device, slot), so concurrent calls (the per-device threads of
    ``run_sliced`` or independent caller threads on the same GPU) never share
    scratch.  A grown buffer replaces the old one only after the caller's
    previous call on it has returned (the pipelines synchronise their streams
    before returning), so no native stream still uses the freed block."""
    cache = getattr(_WS_TLS, "ws", None)
    if cache is None:
        cache = _WS_TLS.ws = {}
    key = (device, slot)
    ws = cache.get(key)
    if ws is None or ws.numel() < nbytes:
        cache.pop(key, None)
        ws = torch.empty(int(nbytes), dtype=torch.uint8, device=device)
        cache[key] = ws
    return ws
