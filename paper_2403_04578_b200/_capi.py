"""ctypes binding of the C ABI in include/tpf.h (libtpf.so, built in-tree).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every solver call raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtpf.so")

TPF_OK = 0
TPF_ERR_INVALID = 1
TPF_ERR_CUDA = 2
TPF_ERR_UNSUPPORTED = 3
TPF_ERR_SINGULAR = 4
TPF_ERR_MEMORY = 5

_c_i32, _c_i64, _c_dbl, _c_ptr, _c_sz = (ctypes.c_int32, ctypes.c_int64, ctypes.c_double,
                                         ctypes.c_void_p, ctypes.c_size_t)
_c_flt = ctypes.c_float

# name -> (restype, argtypes); must match include/tpf.h exactly
SIGNATURES = {
    "tpf_version": (ctypes.c_int, []),
    "tpf_last_error": (ctypes.c_char_p, []),
    "tpf_gen_loads_workspace_bytes": (_c_sz, []),
    "tpf_gen_loads_c128": (ctypes.c_int, [_c_i64, _c_i32, _c_ptr, _c_dbl, _c_dbl, ctypes.c_uint64, _c_i64, _c_dbl,
                                          _c_ptr, _c_i64, _c_i64, _c_ptr, _c_sz, _c_ptr]),
    "tpf_dense_max_nodes": (ctypes.c_int, []),
    "tpf_dense_setup_tree_c128": (ctypes.c_int, [_c_i32, _c_i32, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr,
                                                _c_ptr]),
    "tpf_dense_workspace_bytes": (_c_sz, [_c_i32]),
    "tpf_dense_fpi_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_dbl, _c_dbl, _c_dbl, _c_i32,
        _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_sz, _c_ptr]),
    "tpf_dense_ws_fpi_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_dbl, _c_dbl, _c_dbl, _c_i32,
        _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_sz, _c_ptr]),
    "tpf_dense_pairs_fpi_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_dbl, _c_dbl, _c_dbl, _c_i32,
        _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_sz, _c_ptr]),
    "tpf_dense_large_workspace_bytes": (_c_sz, [_c_i64, _c_i32]),
    "tpf_dense_fpi_large_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_dbl, _c_dbl, _c_dbl, _c_i32,
        _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_sz, _c_ptr]),
    "tpf_residual_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr,
        _c_ptr, _c_ptr, _c_ptr]),
    "tpf_residual_order_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr,
        _c_ptr, _c_ptr, _c_ptr, _c_ptr]),
    "tpf_batch_summary": (ctypes.c_int, [_c_i64, _c_ptr, _c_ptr, _c_dbl, _c_ptr, _c_ptr, _c_ptr]),
    "tpf_sparse_fpi_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_i64, _c_i64,
        _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr,
        _c_ptr, _c_dbl, _c_dbl, _c_dbl, _c_i32,
        _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_sz, _c_ptr]),
    "tpf_sparse_workspace_bytes": (_c_sz, [_c_i64, _c_i32]),
    "tpf_dense_solve_host_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr,
        _c_dbl, _c_dbl, _c_dbl, _c_i32, _c_dbl, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr,
        _c_ptr, _c_i64, _c_i32, _c_ptr, _c_sz]),
    "tpf_sparse_solve_host_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr,
        _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr,
        _c_dbl, _c_dbl, _c_dbl, _c_i32, _c_dbl, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr,
        _c_ptr, _c_i64, _c_i32, _c_ptr, _c_sz]),
    "tpf_dense_solve_host_workspace_bytes": (_c_sz, [_c_i64, _c_i32, _c_i64, _c_i64]),
    "tpf_sparse_solve_host_workspace_bytes": (_c_sz, [_c_i64, _c_i32, _c_i64, _c_i64, _c_i64, _c_i64]),
    "tpf_sparse_tree_max_slots": (ctypes.c_int, []),
    "tpf_sparse_tree_fpi_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_i32, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_i64, _c_i64, _c_dbl, _c_dbl, _c_dbl,
        _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_sz, _c_ptr]),
    "tpf_sparse_tree_fpi_resid_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_i32, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_i64, _c_i64, _c_dbl, _c_dbl, _c_dbl,
        _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_i32, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_sz, _c_ptr]),
    "tpf_sparse_tree_max_ell_width": (ctypes.c_int, []),
    "tpf_sparse_subtree_warps": (ctypes.c_int, []),
    "tpf_sparse_subtree_smem_bytes": (_c_sz, [_c_i32, _c_i32, _c_i32, _c_i32, _c_i32]),
    "tpf_sparse_subtree_workspace_bytes": (_c_sz, [_c_i64, _c_i32]),
    "tpf_sparse_subtree_solve_host_workspace_bytes": (_c_sz, [_c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i64,
                                                              _c_i64]),
    "tpf_sparse_subtree_solve_host_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr,
        _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_dbl, _c_dbl, _c_dbl, _c_i32, _c_dbl, _c_ptr,
        _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_i64, _c_i32, _c_ptr, _c_sz]),
    "tpf_sparse_subtree_fpi_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr,
        _c_ptr, _c_i64, _c_i64, _c_dbl, _c_dbl, _c_dbl, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr,
        _c_sz, _c_ptr]),
    "tpf_sparse_tree_zip_workspace_bytes": (_c_sz, [_c_i64, _c_i32]),
    "tpf_sparse_zip_chain_workspace_bytes": (_c_sz, [_c_i64, _c_i32]),
    "tpf_sparse_zip_chain_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_i64, _c_i64, _c_dbl, _c_dbl, _c_ptr,
        _c_dbl, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_sz, _c_ptr]),
    "tpf_sparse_zip_lu_workspace_bytes": (_c_sz, [_c_i64, _c_i32, _c_i32]),
    "tpf_sparse_zip_lu_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_i32, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_i64,
        _c_i64, _c_dbl, _c_dbl, _c_ptr, _c_dbl, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr,
        _c_sz, _c_ptr]),
    "tpf_sparse_zip_dense_max_nodes": (ctypes.c_int, []),
    "tpf_sparse_zip_dense_workspace_bytes": (_c_sz, [_c_i64, _c_i32]),
    "tpf_sparse_zip_dense_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_i64, _c_i64, _c_dbl, _c_dbl, _c_ptr,
        _c_dbl, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_sz, _c_ptr]),
    "tpf_sparse_tree_zip_fpi_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_i32, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_i64, _c_i64, _c_dbl, _c_dbl, _c_ptr,
        _c_dbl, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_i32, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_sz,
        _c_ptr]),
    "tpf_sparse_tree_ell_width": (ctypes.c_int, [_c_i32, _c_ptr]),
    "tpf_sparse_tree_build_ell": (ctypes.c_int, [_c_i32, _c_i32, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr]),
    "tpf_sparse_tree_solve_host_workspace_bytes": (_c_sz, [_c_i64, _c_i32, _c_i64, _c_i64]),
    "tpf_sparse_tree_solve_host_c128": (ctypes.c_int, [
        _c_i64, _c_i32, _c_i32, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr,
        _c_ptr, _c_dbl, _c_dbl, _c_dbl, _c_i32, _c_dbl, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr,
        _c_ptr, _c_i64, _c_i32, _c_ptr, _c_sz]),
    "tpf_dense_c64_max_nodes": (ctypes.c_int, []),
    "tpf_dense_c64_workspace_bytes": (_c_sz, [_c_i64, _c_i32]),
    "tpf_dense_fpi_c64": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_flt, _c_flt, _c_flt, _c_i32, _c_ptr, _c_i64,
        _c_i64, _c_ptr, _c_ptr, _c_sz, _c_ptr]),
    "tpf_sparse_c64_workspace_bytes": (_c_sz, [_c_i64, _c_i32]),
    "tpf_sparse_fpi_c64": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr,
        _c_ptr, _c_flt, _c_flt, _c_flt, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_sz, _c_ptr]),
    "tpf_residual_c64": (ctypes.c_int, [
        _c_i64, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr,
        _c_ptr]),
    "tpf_loads_csv_scan": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int32),
                                          ctypes.POINTER(ctypes.c_int64)]),
    "tpf_loads_csv_read": (ctypes.c_int, [ctypes.c_char_p, _c_i32, _c_i64, _c_ptr, ctypes.POINTER(ctypes.c_int64),
                                          _c_i32]),
    "tpf_write_pairs_csv": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, _c_i32, _c_i64, _c_ptr, _c_ptr, _c_i64,
                                           _c_i64, _c_ptr, _c_i32]),
    "tpf_voltage_stats_workspace_bytes": (_c_sz, [_c_i64, _c_i32]),
    "tpf_voltage_stats_c128": (ctypes.c_int, [_c_i64, _c_i32, _c_ptr, _c_i64, _c_i64, _c_ptr, _c_ptr, _c_ptr,
                                               _c_i32, _c_ptr, _c_sz, _c_ptr]),
    "tpf_host_pin": (ctypes.c_int, [_c_ptr, _c_sz]),
    "tpf_host_unpin": (ctypes.c_int, [_c_ptr]),
    "tpf_probe_fp64_tflops": (ctypes.c_int, [ctypes.POINTER(_c_dbl), ctypes.POINTER(_c_dbl)]),
}

_lib = None


class EngineError(RuntimeError):
    """A CUDA-side failure reported through tpf_last_error()."""


def load() -> ctypes.CDLL:
    """Load libtpf.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA engine first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    lib = load()
    return [n for n in SIGNATURES if hasattr(lib, n)]


def check(rc: int) -> None:
    if rc == TPF_OK:
        return
    msg = load().tpf_last_error().decode(errors="replace")
    if rc == TPF_ERR_INVALID:
        raise ValueError(msg)
    if rc == TPF_ERR_SINGULAR:
        from ._types import SingularSystemError
        raise SingularSystemError(msg)
    if rc == TPF_ERR_MEMORY:
        from ._types import MemoryGuardError
        raise MemoryGuardError(msg)
    if rc == TPF_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise EngineError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
