"""Sparse Tensor Power Flow on the GPU -- drop-in for ``tpflow.batch_solve_sparse``.

Reference: pkg/src/tpflow/sparse.py:167-207.  The reference stacks tau blocks
``-diag(1/s_j*) Y_dd`` into one (b tau)^2 block-diagonal matrix and factorizes
it with SuperLU (sparse.py:115-164, 70-97).  Multiplying block row i by
``-s_ij*`` shows every block is the same equation

    Y_dd v'_j = -(s_j* ./ conj(v_j) + src)          (zero-load rows included)

so this engine factorizes ``Y_dd`` ONCE on the host (SuperLU; for radial
feeders in leaf-first order, which gives an LU with no fill and no pivoting,
SURVEY.md A.6) and runs batched forward/backward sweeps for all tau cases per
iteration in libtpf.so.  ``factorization_count()`` therefore still grows by
exactly one per batch (test_sparse.py:164-168).

``max_nnz``: the reference refuses batches whose block matrix would exceed
``max_nnz`` nonzeros (sparse.py:131-136).  Here no block matrix exists; the
guard is honoured only when the caller passes ``max_nnz`` explicitly (same
``MemoryGuardError`` message), otherwise the batch is solved whatever its
size, in tau chunks that fit device memory.
"""

from __future__ import annotations

import threading
from collections import deque
from dataclasses import dataclass

import numpy as np
import torch
from scipy import sparse
from scipy.sparse.linalg import splu

from . import _capi
from ._device import (ModelContract, complex_strides, stream_scratch, engine_dtype, host_csr, host_empty, host_loads,
                      device_workspace_slot,
                      loads_to_device, ptr, require_cuda, residual_and_summary, resolve_devices, run_sliced,
                      stream_ptr)
from ._types import LoadMatrix, MemoryGuardError, SingularSystemError, SolveOptions, VoltageBatch
from .dense import as_load_matrix, finish

__all__ = ["batch_solve_sparse", "factorization_count", "factorize_ydd", "TreeLU",
           "TreeSchedule", "tree_schedule", "SparseOperator", "DEFAULT_MAX_BLOCK_NNZ"]

# sparse.py:44
DEFAULT_MAX_BLOCK_NNZ = 50_000_000

_factorizations = 0
_lock = threading.Lock()


def factorization_count() -> int:
    """Monotone count of Y_dd factorizations (sparse.py:50-52)."""
    return _factorizations


def leaf_first_order(y: sparse.csr_matrix) -> np.ndarray | None:
    """Decreasing-depth order of the graph of Y_dd if it is a forest, else None.

    Eliminating a tree leaf-first creates no fill.
    """
    b = y.shape[0]
    g = sparse.csr_matrix(abs(y) + abs(y).T)
    g.setdiag(0)
    g.eliminate_zeros()
    if g.nnz // 2 > b - 1:
        return None
    depth = np.full(b, -1, dtype=np.int64)
    for root in range(b):
        if depth[root] >= 0:
            continue
        depth[root] = 0
        queue = deque([root])
        edges = 0
        nodes = 0
        while queue:
            u = queue.popleft()
            nodes += 1
            for v in g.indices[g.indptr[u]:g.indptr[u + 1]]:
                edges += 1
                if depth[v] < 0:
                    depth[v] = depth[u] + 1
                    queue.append(v)
        if edges // 2 != nodes - 1:
            return None
    return np.argsort(-depth, kind="stable")


def tree_parents(y) -> tuple[np.ndarray, np.ndarray] | None:
    """Leaf-first order of a forest-shaped Y_dd and each position's parent
    position (-1 at roots), or None if Y_dd has a cycle."""
    y = sparse.csr_matrix(y)
    order = leaf_first_order(y)
    if order is None:
        return None
    b = y.shape[0]
    g = sparse.csr_matrix(abs(y) + abs(y).T)
    g.setdiag(0)
    g.eliminate_zeros()
    pos = np.empty(b, dtype=np.int64)
    pos[order] = np.arange(b)
    parent = np.full(b, -1, dtype=np.int64)
    for k, v in enumerate(order):  # the neighbour eliminated after v is its parent (at most one: a forest)
        nb = g.indices[g.indptr[v]:g.indptr[v + 1]]
        later = [int(pos[u]) for u in nb if pos[u] > k]
        if len(later) > 1:
            return None
        if later:
            parent[k] = later[0]
    return order, parent


@dataclass
class ZipLUSchedule:
    """Fixed-pattern LU schedule of a meshed Y_dd for per-case factorization
    (``tpf_sparse_zip_lu_c128``): minimum-degree elimination order over the
    symmetrised pattern, no pivoting.  Step k eliminates node ``orig[k]``; its
    later neighbours (fill included) sit at positions ``idx[off:off+m]``,
    followed by their L slots, U slots and the m x m update targets; slot k
    (< b) is the pivot of step k."""

    b: int
    nslot: int
    orig: np.ndarray   # int32 [b]
    kinfo: np.ndarray  # int32 [b, 2]: m_k, offset into idx
    idx: np.ndarray    # int32
    base: np.ndarray   # complex128 [nslot]: Y_dd at the factor slots (0 at fill)

    @property
    def fill(self) -> int:
        return self.nslot - self.b


def zip_lu_schedule(y) -> ZipLUSchedule:
    """Greedy minimum-degree order (ties: lowest node index) and the symbolic
    elimination of Y_dd's symmetrised pattern."""
    import heapq
    y = sparse.csr_matrix(y)
    b = y.shape[0]
    g = sparse.csr_matrix(abs(y) + abs(y).T)
    g.setdiag(0)
    g.eliminate_zeros()
    adj = [set(g.indices[g.indptr[v]:g.indptr[v + 1]].tolist()) for v in range(b)]
    heap = [(len(adj[v]), v) for v in range(b)]
    heapq.heapify(heap)
    done = np.zeros(b, dtype=bool)
    order, nbrs = [], []
    while heap:
        d, v = heapq.heappop(heap)
        if done[v] or d != len(adj[v]):
            continue  # stale entry
        done[v] = True
        nb = adj[v]
        order.append(v)
        nbrs.append(list(nb))
        for u in nb:
            adj[u].discard(v)
            adj[u] |= nb - {u}
            heapq.heappush(heap, (len(adj[u]), u))
        adj[v] = set()
    order = np.asarray(order, dtype=np.int64)
    pos = np.empty(b, dtype=np.int64)
    pos[order] = np.arange(b)
    later = [sorted(int(pos[u]) for u in nb) for nb in nbrs]
    slot = {}
    nslot = b
    for k, lk in enumerate(later):
        for q in lk:
            slot[(q, k)] = nslot  # L
            slot[(k, q)] = nslot + 1  # U
            nslot += 2
    kinfo = np.zeros((b, 2), dtype=np.int32)
    idx = []
    for k, lk in enumerate(later):
        kinfo[k] = (len(lk), len(idx))
        idx += lk
        idx += [slot[(q, k)] for q in lk]
        idx += [slot[(k, q)] for q in lk]
        idx += [(q if q == r else slot[(q, r)]) for q in lk for r in lk]
    base = np.zeros(nslot, dtype=np.complex128)
    c = y.tocoo()
    for r, col, v in zip(c.row, c.col, c.data):
        pr, pc = int(pos[r]), int(pos[col])
        base[pr if pr == pc else slot[(pr, pc)]] += v
    return ZipLUSchedule(b=b, nslot=nslot, orig=order.astype(np.int32), kinfo=kinfo,
                         idx=np.asarray(idx, dtype=np.int32), base=base)


def zip_lu_solve_host(s: ZipLUSchedule, diag_add: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """Host restatement of the kernel's factorization + solve (schedule tests):
    (Y_dd + diag(diag_add)) x = rhs, original node order."""
    F = s.base.copy()
    F[:s.b] += np.asarray(diag_add)[s.orig]
    for k in range(s.b):
        m, off = s.kinfo[k]
        pos, ls, us, tg = (s.idx[off:off + m], s.idx[off + m:off + 2 * m], s.idx[off + 2 * m:off + 3 * m],
                           s.idx[off + 3 * m:off + 3 * m + m * m].reshape(m, m))
        F[k] = 1.0 / F[k]
        for i in range(m):
            F[ls[i]] *= F[k]
            F[tg[i]] -= F[ls[i]] * F[us]
    z = np.asarray(rhs, dtype=np.complex128)[s.orig].copy()
    for k in range(s.b):
        m, off = s.kinfo[k]
        z[s.idx[off:off + m]] -= F[s.idx[off + m:off + 2 * m]] * z[k]
    for k in range(s.b - 1, -1, -1):
        m, off = s.kinfo[k]
        z[k] = (z[k] - np.dot(F[s.idx[off + 2 * m:off + 3 * m]], z[s.idx[off:off + m]])) * F[k]
    out = np.empty_like(z)
    out[s.orig] = z
    return out


@dataclass
class TreeLU:
    """Pr (Y_dd[o][:, o]) Pc = L U in the arrays libtpf's sparse kernel reads."""

    b: int
    l_ptr: np.ndarray
    l_col: np.ndarray
    l_val: np.ndarray
    u_ptr: np.ndarray
    u_col: np.ndarray
    u_val: np.ndarray
    u_diag_inv: np.ndarray
    perm: np.ndarray  # [row_src (b) | col_dst (b)], int32
    ordering: str

    @property
    def nnz(self) -> int:
        return int(self.l_col.size + self.u_col.size + self.b)


def factorize_ydd(y_dd, count: bool = True) -> TreeLU:
    """One LU of Y_dd; raises SingularSystemError like sparse.py:82-94.

    ``count=False``: a structural helper factorization (the ZIP path's level
    schedule), not a batch factorization; ``factorization_count`` is unchanged.
    """
    global _factorizations
    y = sparse.csr_matrix(y_dd, dtype=complex)
    b = y.shape[0]
    if y.shape[0] != y.shape[1]:
        raise ValueError("factorize requires a square matrix")
    order = leaf_first_order(y)
    try:
        if order is not None:
            yp = y[order][:, order].tocsc()
            lu = splu(yp, permc_spec="NATURAL", diag_pivot_thresh=0.0,
                      options=dict(SymmetricMode=True))
            kind = "leaf-first"
        else:
            order = np.arange(b)
            lu = splu(y.tocsc())
            kind = "colamd"
    except RuntimeError as exc:
        empty_rows = np.where(np.diff(y.indptr) == 0)[0]
        empty_cols = np.where(np.diff(y.tocsc().indptr) == 0)[0]
        where = []
        if empty_rows.size:
            where.append(f"empty rows {empty_rows[:8].tolist()}")
        if empty_cols.size:
            where.append(f"empty columns {empty_cols[:8].tolist()}")
        detail = f" ({'; '.join(where)})" if where else ""
        raise SingularSystemError(f"sparse factorization failed: {exc}{detail}") from exc
    if count:
        with _lock:
            _factorizations += 1
    L = sparse.csr_matrix(lu.L)
    U = sparse.csr_matrix(lu.U)
    Ls = sparse.tril(L, k=-1, format="csr")
    Us = sparse.triu(U, k=1, format="csr")
    Ls.sort_indices()
    Us.sort_indices()
    diag = U.diagonal()
    if np.any(diag == 0):
        raise SingularSystemError("sparse factorization failed: zero pivot on the diagonal of U")
    perm_r_inv = np.empty(b, dtype=np.int64)
    perm_r_inv[lu.perm_r] = np.arange(b)
    order_inv = np.empty(b, dtype=np.int64)
    order_inv[order] = np.arange(b)
    row_src = order[perm_r_inv]            # forward row k reads node row_src[k]
    col_dst = lu.perm_c[order_inv]         # node i is solution index col_dst[i]
    return TreeLU(
        b=b,
        l_ptr=Ls.indptr.astype(np.int32), l_col=Ls.indices.astype(np.int32),
        l_val=np.ascontiguousarray(Ls.data.astype(complex)),
        u_ptr=Us.indptr.astype(np.int32), u_col=Us.indices.astype(np.int32),
        u_val=np.ascontiguousarray(Us.data.astype(complex)),
        u_diag_inv=np.ascontiguousarray(1.0 / diag),
        perm=np.concatenate([row_src, col_dst]).astype(np.int32),
        ordering=kind)


TREE_THREADS = 512      # CTA size of tpf_sparse_tree_fpi_c128
TREE_MAX_SLOTS = 16     # TMEM slots per thread (include/tpf.h)
TREE_LEVEL_SLOTS = 6    # slots of one depth level held in registers at a time
TREE_MAX_ROOTS = 512    # root-level nodes (source injections kept in shared memory)
TREE_CHUNK = 65536      # cases per compact chunk on long node-major batches (SparseOperator)
TREE_MAX_NODES = 220 * 1024 // 44  # 5,120: sweep vector, child products, child ranges, parents: 44 B per node
SUBTREE_MIN_B = 0       # radial feeders from this size run the warp-per-subtree kernel (tpf_sparse_subtree_fpi_c128)


def _subtree_layout_ok(S: torch.Tensor, V: torch.Tensor) -> bool:
    """The subtree kernel moves whole case columns by TMA: S and V each
    node-major (case stride 1) or case-major (node stride 1), 16-byte aligned."""
    b, tau = S.shape
    sn, sc = S.stride()
    vn, vc = V.stride()
    aligned = S.data_ptr() % 16 == 0 and V.data_ptr() % 16 == 0
    s_ok = (sc == 1 and sn >= tau) or (sn == 1 and sc >= b)
    v_ok = (vc == 1 and vn >= tau) or (vn == 1 and vc >= b)
    return aligned and s_ok and v_ok and tau < (1 << 30)


@dataclass
class TreeSchedule:
    """Depth-level layout of a zero-fill tree LU for the on-chip tree kernel.

    Nodes are renumbered level by level (root level first); within a level,
    children of the same parent are contiguous.  ``level_info`` = level
    offsets (levels+1) followed by per-level first TMEM slot (levels+1);
    ``node_info`` = int32[4 per node] {original node, parent, first child,
    child count}; ``node_coef`` = complex, four planes of b (level order):
    e = Y[parent, m], g = U[m, parent] / U[m, m], 1/U[m, m], src[original node].
    """

    b: int
    levels: int
    level_info: np.ndarray
    node_info: np.ndarray
    node_coef: np.ndarray
    slots: int


def tree_levels(f: TreeLU, src: np.ndarray) -> TreeSchedule | None:
    """Depth-level layout of a zero-fill tree elimination of a symmetric Y_dd,
    or None.  No kernel limits: ``tree_schedule`` (one-case-per-SM level
    kernel) and ``subtree_schedule`` (warp-per-subtree kernel) apply theirs.
    ``level_info``'s slot starts are those of the level kernel's 512 threads."""
    b = f.b
    if f.ordering != "leaf-first":
        return None
    row_src = f.perm[:b].astype(np.int64)
    col_dst = f.perm[b:].astype(np.int64)
    if not np.array_equal(col_dst[row_src], np.arange(b)):
        return None  # not a symmetric permutation
    ucount = np.diff(f.u_ptr)
    if ucount.max(initial=0) > 1:
        return None
    parent = np.full(b, -1, dtype=np.int64)
    upar = np.zeros(b, dtype=complex)
    has = ucount == 1
    parent[has] = f.u_col[f.u_ptr[:-1][has]]
    upar[has] = f.u_val[f.u_ptr[:-1][has]]
    if np.any(parent[has] <= np.nonzero(has)[0]):
        return None  # parents must be eliminated after their children
    # L[parent, k]: the entry of row parent(k), column k
    lval = np.zeros(b, dtype=complex)
    nchild = np.diff(f.l_ptr)
    rows = np.repeat(np.arange(b), nchild)
    if np.any(parent[f.l_col] != rows):
        return None  # L holds something other than child edges
    lval[f.l_col] = f.l_val
    depth = np.zeros(b, dtype=np.int64)
    for k in range(b - 1, -1, -1):
        if parent[k] >= 0:
            depth[k] = depth[parent[k]] + 1
    levels = int(depth.max(initial=0)) + 1
    pos_in_level = np.zeros(b, dtype=np.int64)
    level_nodes = [np.nonzero(depth == 0)[0]]
    pos_in_level[level_nodes[0]] = np.arange(level_nodes[0].size)
    # level by level (level 0 first) so children sort by parent position, then by k
    for d in range(1, levels):
        cand = np.nonzero(depth == d)[0]
        key = pos_in_level[parent[cand]]
        level_nodes.append(cand[np.lexsort((cand, key))])
        pos_in_level[level_nodes[-1]] = np.arange(cand.size)
    order = np.concatenate(level_nodes)
    m_of_k = np.empty(b, dtype=np.int64)
    m_of_k[order] = np.arange(b)
    sizes = np.array([x.size for x in level_nodes])
    offs = np.concatenate([[0], np.cumsum(sizes)])
    slots_per = -(-sizes // TREE_THREADS)
    j0 = np.concatenate([[0], np.cumsum(slots_per)])
    pm = np.where(parent[order] >= 0, m_of_k[np.maximum(parent[order], 0)], -1)
    cnt = np.zeros(b, dtype=np.int64)
    kids = pm >= 0
    np.add.at(cnt, pm[kids], 1)
    first_seen = np.full(b, b, dtype=np.int64)
    np.minimum.at(first_seen, pm[kids], np.nonzero(kids)[0])
    first = np.where(cnt > 0, first_seen, 0)
    # contiguity of children
    if np.any(cnt > 0):
        ok = np.all(pm[first[cnt > 0] + cnt[cnt > 0] - 1] == np.nonzero(cnt > 0)[0])
        if not ok:
            return None
    info = np.stack([row_src[order], pm, first, cnt], axis=1).astype(np.int32)
    # scaled sweeps use e_m = Y[parent, m] = L[parent, m] U[m, m]; symmetric Y needs U[m, p] == e_m
    e = lval[order] / f.u_diag_inv[order]
    if not np.allclose(upar[order], e, rtol=1e-12, atol=0.0):
        return None
    src_o = np.asarray(src)[row_src[order]]
    if np.any(src_o[offs[1]:] != 0):
        return None  # source injection only at the root level (nodes next to the slack)
    g = upar[order] * f.u_diag_inv[order]  # U[m, parent] / U[m, m] = L[parent, m] for symmetric Y
    coef = np.stack([e, g, f.u_diag_inv[order], src_o], axis=1).astype(complex)
    return TreeSchedule(b=b, levels=levels,
                        level_info=np.concatenate([offs, j0]).astype(np.int32),
                        node_info=np.ascontiguousarray(info.ravel()),
                        node_coef=np.ascontiguousarray(coef.T.ravel()), slots=int(j0[-1]))


def tree_direct(y_dd, src: np.ndarray) -> TreeSchedule | None:
    """The zero-fill tree elimination of a symmetric radial Y_dd computed
    directly, without SuperLU (the dense setup, ``dense.device_kw``): BFS
    levels from one root per component (a node next to the slack where there
    is one), leaves first U_pp -= e_m g_m with e_m = Y[m, parent], g_m = e_m /
    U_mm.  The same layout as ``tree_levels``; the values equal the SuperLU
    factors' to rounding.  None unless Y_dd's graph is a forest with
    symmetric values."""
    y = y_dd if sparse.isspmatrix_csr(y_dd) and y_dd.dtype == complex else sparse.csr_matrix(y_dd, dtype=complex)
    b = y.shape[0]
    if b < 1 or y.shape[1] != b:
        return None
    if not y.has_sorted_indices:
        y = y.sorted_indices()
    rp, ci, yv = y.indptr.astype(np.int64), y.indices.astype(np.int64), y.data
    rows = np.repeat(np.arange(b), np.diff(rp))
    off = ci != rows
    srcv = np.asarray(src)
    # level-synchronous BFS (numpy), roots: the nodes next to the slack, then
    # one node of any component still unreached
    parent = np.full(b, -1, dtype=np.int64)
    depth = np.full(b, -1, dtype=np.int64)
    frontier = np.nonzero(srcv != 0)[0]
    roots = list(frontier)
    depth[frontier] = 0
    while True:
        while frontier.size:
            lens = rp[frontier + 1] - rp[frontier]
            total = int(lens.sum())
            start = np.repeat(rp[frontier] - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens)
            k = start + np.arange(total)
            nb, fr = ci[k], np.repeat(frontier, lens)
            keep = (nb != fr) & (nb != parent[fr])
            nb, fr = nb[keep], fr[keep]
            if np.any(depth[nb] >= 0) or np.unique(nb).size != nb.size:
                return None  # a cycle: not a forest
            parent[nb] = fr
            depth[nb] = depth[fr] + 1
            frontier = nb
        rest = np.nonzero(depth < 0)[0]
        if rest.size == 0:
            break
        frontier = rest[:1]
        roots.append(int(rest[0]))
        depth[frontier] = 0
    ncomp = len(roots)
    if int(off.sum()) != 2 * (b - ncomp):
        return None
    levels = int(depth.max()) + 1
    # e_m = Y[m, parent(m)], and Y[parent(m), m] must be the same value
    e = np.zeros(b, dtype=complex)
    fwd = off & (ci == parent[rows])
    e[rows[fwd]] = yv[fwd]
    bwd = off & (rows == parent[ci])
    if int(fwd.sum()) != b - ncomp or not np.array_equal(yv[bwd], e[ci[bwd]]):
        return None
    # leaves first
    U = y.diagonal().astype(complex)
    g = np.zeros(b, dtype=complex)
    for lv in range(levels - 1, 0, -1):
        nodes = np.nonzero(depth == lv)[0]
        g[nodes] = e[nodes] / U[nodes]
        np.subtract.at(U, parent[nodes], e[nodes] * g[nodes])
    if np.any(U == 0) or not np.all(np.isfinite(U)):
        return None
    uinv = 1.0 / U
    # level order: roots, then each level's children contiguous by parent position
    pos_in_level = np.zeros(b, dtype=np.int64)
    level_nodes = [np.sort(np.nonzero(depth == 0)[0])]
    pos_in_level[level_nodes[0]] = np.arange(level_nodes[0].size)
    for lv in range(1, levels):
        cand = np.nonzero(depth == lv)[0]
        level_nodes.append(cand[np.lexsort((cand, pos_in_level[parent[cand]]))])
        pos_in_level[level_nodes[-1]] = np.arange(cand.size)
    order = np.concatenate(level_nodes)
    m_of = np.empty(b, dtype=np.int64)
    m_of[order] = np.arange(b)
    sizes = np.array([x.size for x in level_nodes])
    offs = np.concatenate([[0], np.cumsum(sizes)])
    slots_per = -(-sizes // TREE_THREADS)
    j0 = np.concatenate([[0], np.cumsum(slots_per)])
    pm = np.where(parent[order] >= 0, m_of[np.maximum(parent[order], 0)], -1)
    cnt = np.zeros(b, dtype=np.int64)
    kids = pm >= 0
    np.add.at(cnt, pm[kids], 1)
    first_seen = np.full(b, b, dtype=np.int64)
    np.minimum.at(first_seen, pm[kids], np.nonzero(kids)[0])
    first = np.where(cnt > 0, first_seen, 0)
    info = np.stack([order, pm, first, cnt], axis=1).astype(np.int32)
    coef = np.stack([e[order], g[order], uinv[order], srcv[order].astype(complex)], axis=1)
    return TreeSchedule(b=b, levels=levels, level_info=np.concatenate([offs, j0]).astype(np.int32),
                        node_info=np.ascontiguousarray(info.ravel()),
                        node_coef=np.ascontiguousarray(coef.T.ravel()), slots=int(j0[-1]))


def radial_levels(contract, count: bool = True) -> TreeSchedule | None:
    """The batch factorization of a radial feeder: ``tree_direct`` (counted
    by ``factorization_count`` like a SuperLU factorization), or None for
    meshed networks (SuperLU, ``factorize_ydd``)."""
    global _factorizations
    t = tree_direct(contract.y_dd, contract.src)
    if t is not None and count:
        with _lock:
            _factorizations += 1
    return t


def tree_limits(t: TreeSchedule | None) -> TreeSchedule | None:
    """``t`` if it is within the level kernel's limits (tpf_sparse_tree_fpi_c128), else None."""
    if t is None or t.b > TREE_MAX_NODES:
        return None
    offs = t.level_info[:t.levels + 1]
    sizes = np.diff(offs)
    if t.slots > TREE_MAX_SLOTS or np.any(-(-sizes // TREE_THREADS) > TREE_LEVEL_SLOTS) \
            or sizes[0] > TREE_MAX_ROOTS:
        return None
    return t


def tree_schedule(f: TreeLU, src: np.ndarray) -> TreeSchedule | None:
    """``tree_levels`` within the level kernel's limits (tpf_sparse_tree_fpi_c128), else None."""
    return tree_limits(tree_levels(f, src)) if f.b <= TREE_MAX_NODES else None


def tree_ell(t: TreeSchedule, contract) -> tuple[int, np.ndarray, np.ndarray] | None:
    """Level-ordered ELL rows of Y_dd for the fused residual (tpf_sparse_tree_build_ell), or None."""
    lib = _capi.load()
    rp, ci, yv = host_csr(contract)
    w = int(lib.tpf_sparse_tree_ell_width(t.b, ptr(rp)))
    if w < 1 or w > int(lib.tpf_sparse_tree_max_ell_width()):
        return None
    col = np.empty(w * t.b, dtype=np.int32)
    val = np.empty(w * t.b, dtype=np.complex128)
    if lib.tpf_sparse_tree_build_ell(t.b, w, ptr(t.node_info), ptr(rp), ptr(ci), ptr(yv), ptr(col), ptr(val)) != 0:
        return None  # rows beyond diagonal + tree edges: the separate residual kernel
    return w, col, val


def tree_solve_host(t: TreeSchedule, rhs: np.ndarray) -> np.ndarray:
    """Numpy emulation of the tree kernel's two sweeps (host-logic tests only)."""
    b = t.b
    info = t.node_info.reshape(b, 4)
    coef = t.node_coef.reshape(4, b).T
    offs = t.level_info[:t.levels + 1]
    T = np.zeros(b, dtype=complex)
    for d in range(t.levels - 1, -1, -1):
        for m in range(offs[d], offs[d + 1]):
            z = rhs[info[m, 0]]
            for c in range(info[m, 2], info[m, 2] + info[m, 3]):
                z -= coef[c, 1] * T[c]
            T[m] = z
    for d in range(t.levels):
        for m in range(offs[d], offs[d + 1]):
            w = T[m] * coef[m, 2]
            if info[m, 1] >= 0:
                w -= coef[m, 1] * T[info[m, 1]]
            T[m] = w
    x = np.empty(b, dtype=complex)
    x[info[:, 0]] = T
    return x


def lu_solve_host(f: TreeLU, rhs: np.ndarray) -> np.ndarray:
    """Numpy emulation of the kernel's sweep order (host-logic tests only)."""
    b = f.b
    z = np.zeros(b, dtype=complex)
    for k in range(b):
        acc = rhs[f.perm[k]]
        for p in range(f.l_ptr[k], f.l_ptr[k + 1]):
            acc -= f.l_val[p] * z[f.l_col[p]]
        z[k] = acc
    for k in range(b - 1, -1, -1):
        acc = z[k]
        for p in range(f.u_ptr[k], f.u_ptr[k + 1]):
            acc -= f.u_val[p] * z[f.u_col[p]]
        z[k] = acc * f.u_diag_inv[k]
    return z[f.perm[b:]]


class SparseOperator:
    """One factorization of Y_dd resident on a device; ``solve`` iterates."""

    def __init__(self, model, device=None, use_tree: bool = True, dtype=None, kernel: str = "auto"):
        """``kernel``: "auto" (warp-per-subtree kernel where its schedule fits and
        b >= SUBTREE_MIN_B, else the level kernel on radial feeders, else the
        general CSR kernel), or "subtree" / "tree" / "general" to force one
        (A/B tests; a forced radial kernel that does not fit falls back)."""
        self.device = require_cuda(device)
        self.contract = ModelContract.of(model)
        self.dtype = engine_dtype(dtype)
        c64 = self.dtype == np.complex64
        d = self.device
        def t(a):  # never hand a 0-element (null) buffer to the C ABI
            a = np.ascontiguousarray(a)
            if a.size == 0:
                a = np.zeros(1, dtype=a.dtype)
            return torch.from_numpy(a).to(d)
        self._t = t
        use_tree = use_tree and not c64 and kernel != "general"  # the c64 twin is the general CSR kernel
        # one factorization: the tree elimination of a radial feeder, else SuperLU
        levels = radial_levels(self.contract) if use_tree else None
        self.lu = None if levels is not None else factorize_ydd(self.contract.y_dd)
        self._dev = None
        self.v_flat = complex(abs(self.contract.v_s))
        self._ws: dict = {}  # per-stream scratch (_device.stream_scratch)
        self._csr = None
        self._chunk = None
        if levels is None and use_tree:
            levels = tree_levels(self.lu, self.contract.src)
        self.tree = None
        self.sub = None
        if levels is not None and kernel in ("auto", "subtree") and \
                (kernel == "subtree" or self.contract.b >= SUBTREE_MIN_B):
            from .subtree import subtree_schedule
            rp, ci, yv = host_csr(self.contract)
            self.sub = subtree_schedule(levels, rp, ci, yv)
        if self.sub is not None:
            sb = self.sub
            self.sub_dev = dict(pinfo=t(sb.pinfo), kids=torch.from_numpy(sb.kids.view(np.int16).copy()).to(d),
                                slotinfo=t(sb.slotinfo), coef=t(sb.coef), ell_col=t(sb.ell_col),
                                ell_val=t(sb.ell_val))
        if levels is not None:
            # the level kernel: radial feeders without a subtree schedule, and
            # the fallback for S / V layouts the subtree kernel's TMA cannot move
            self.tree = tree_limits(levels)
        if self.tree is not None:
            self.tree_dev = dict(level_info=t(self.tree.level_info), node_info=t(self.tree.node_info),
                                 node_coef=t(self.tree.node_coef))
            ell = tree_ell(self.tree, self.contract)
            if ell is not None:  # residual post-check fused into the tree kernel
                self.tree_dev.update(ell_w=ell[0], ell_col=t(ell[1]), ell_val=t(ell[2]))

    @property
    def b(self) -> int:
        return self.contract.b

    @property
    def dev(self) -> dict:
        """The general CSR kernel's LU arrays on the device (built on first use:
        radial feeders factor as a tree and need them only for layouts the
        tree kernels cannot take)."""
        if self._dev is None:
            if self.lu is None:
                self.lu = factorize_ydd(self.contract.y_dd, count=False)  # the same matrix, factored again
            f, t = self.lu, self._t
            cx = (lambda a: np.asarray(a).astype(np.complex64)) if self.dtype == np.complex64 else (lambda a: a)
            self._dev = dict(l_ptr=t(f.l_ptr), l_col=t(f.l_col), l_val=t(cx(f.l_val)), u_ptr=t(f.u_ptr),
                             u_col=t(f.u_col), u_val=t(cx(f.u_val)), u_diag_inv=t(cx(f.u_diag_inv)),
                             perm=t(f.perm), src=t(cx(self.contract.src)))
        return self._dev

    @property
    def kernel(self) -> str:
        if self.sub is not None:
            return "sparse_subtree_kernel"
        return "sparse_tree_kernel" if self.tree is not None else "sparse_fpi_kernel"

    def csr(self):
        """Y_dd CSR + source injection on the device (original node order), cached."""
        if self._csr is None:
            self._csr = self.contract.csr_on(self.device)
        return self._csr

    def solve(self, S: torch.Tensor, opts: SolveOptions = SolveOptions(), V=None, iters=None, resid=None):
        """Iterate a device b x tau load tensor; returns ``(V, iters)``.

        With ``resid`` (float64[tau] device tensor) the residual post-check
        (fpi.py:221-240) is also written: fused into the tree kernel's retire
        step, or by ``tpf_residual_c128`` after the general kernel.
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
        if self.sub is not None and _subtree_layout_ok(S, V):
            # node-major batches are solved in case-major chunks (scratch in the workspace)
            need = (int(_capi.load().tpf_sparse_subtree_workspace_bytes(tau, b))
                    if S.stride(1) == 1 or V.stride(1) == 1 else 256)
            ws = stream_scratch(self._ws, self.device, need)
            sb, g = self.sub, self.sub_dev
            sn, sc = complex_strides(S)
            vn, vc = complex_strides(V)
            _capi.call("tpf_sparse_subtree_fpi_c128", tau, b, sb.NS, sb.NT, sb.RMAX, sb.RW, int(sb.kids.size),
                       g["pinfo"].data_ptr(), g["slotinfo"].data_ptr(), g["kids"].data_ptr(), g["coef"].data_ptr(),
                       g["ell_col"].data_ptr(), g["ell_val"].data_ptr(), S.data_ptr(), sn, sc,
                       self.v_flat.real, self.v_flat.imag, float(opts.tolerance), int(opts.max_iterations),
                       V.data_ptr(), vn, vc, iters.data_ptr(), 0 if resid is None else resid.data_ptr(),
                       ws.data_ptr(), ws.numel(), stream_ptr(self.device))
            return V, iters
        if self.tree is not None:
            ws = stream_scratch(self._ws, self.device, 256)
            if tau > TREE_CHUNK and S.stride(1) == 1 and V.stride(1) == 1:
                return self._solve_tree_chunked(S, opts, V, iters, resid)
            sn, sc = complex_strides(S)
            vn, vc = complex_strides(V)
            g = self.tree_dev
            head = (tau, b, self.tree.levels, g["level_info"].data_ptr(), g["node_info"].data_ptr(),
                    g["node_coef"].data_ptr(), S.data_ptr(), sn, sc, self.v_flat.real, self.v_flat.imag,
                    float(opts.tolerance), int(opts.max_iterations), V.data_ptr(), vn, vc, iters.data_ptr())
            tail = (ws.data_ptr(), ws.numel(), stream_ptr(self.device))
            if resid is not None and "ell_w" in g:
                _capi.call("tpf_sparse_tree_fpi_resid_c128", *head, g["ell_w"], g["ell_col"].data_ptr(),
                           g["ell_val"].data_ptr(), resid.data_ptr(), *tail)
                return V, iters
            _capi.call("tpf_sparse_tree_fpi_c128", *head, *tail)
            if resid is not None:
                self._residual(S, V, resid)
            return V, iters
        c64 = self.dtype == np.complex64
        lib = _capi.load()
        need = int(lib.tpf_sparse_c64_workspace_bytes(tau, b) if c64 else lib.tpf_sparse_workspace_bytes(tau, b))
        ws = stream_scratch(self._ws, self.device, need)
        sn, sc = complex_strides(S)
        vn, vc = complex_strides(V)
        g = self.dev
        _capi.call("tpf_sparse_fpi_c64" if c64 else "tpf_sparse_fpi_c128", tau, b, S.data_ptr(), sn, sc,
                   g["l_ptr"].data_ptr(), g["l_col"].data_ptr(), g["l_val"].data_ptr(),
                   g["u_ptr"].data_ptr(), g["u_col"].data_ptr(), g["u_val"].data_ptr(),
                   g["u_diag_inv"].data_ptr(), g["perm"].data_ptr(), g["src"].data_ptr(),
                   self.v_flat.real, self.v_flat.imag, float(opts.tolerance), int(opts.max_iterations),
                   V.data_ptr(), vn, vc, iters.data_ptr(), ws.data_ptr(), ws.numel(),
                   stream_ptr(self.device))
        if resid is not None:
            self._residual(S, V, resid)
        return V, iters

    def _solve_tree_chunked(self, S, opts, V, iters, resid):
        """Node-major batches longer than TREE_CHUNK cases: the tree kernel's
        one-case-per-SM accesses stride a whole row of S / V per node; past a
        few MB per row they miss the TLB (C3, 8.4 MB rows: 127 vs 105 us per
        case per SM).  Each chunk is copied into compact buffers (rows of
        TREE_CHUNK cases), solved, and copied back (tools/c3_chunk_probe.py:
        450 -> 400 ms at full C3, copies included).  Bits are unchanged: every
        case's arithmetic is independent of its position."""
        b, tau = S.shape
        ch = TREE_CHUNK
        if self._chunk is None or self._chunk[0].shape != (b, ch) or self._chunk[0].dtype != S.dtype:
            self._chunk = (torch.empty((b, ch), dtype=S.dtype, device=self.device),
                           torch.empty((b, ch), dtype=S.dtype, device=self.device))
        sc_buf, vc_buf = self._chunk
        for lo in range(0, tau, ch):
            hi = min(tau, lo + ch)
            n = hi - lo
            sc_buf[:, :n].copy_(S[:, lo:hi])
            self.solve(sc_buf[:, :n], opts, V=vc_buf[:, :n], iters=iters[lo:hi],
                       resid=None if resid is None else resid[lo:hi])
            V[:, lo:hi].copy_(vc_buf[:, :n])
        return V, iters

    def _residual(self, S, V, resid):
        rp, ci, val, src, order = self.csr()
        sn, sc = complex_strides(S)
        vn, vc = complex_strides(V)
        if V.dtype == torch.complex64:
            _capi.call("tpf_residual_c64", S.shape[1], self.b, S.data_ptr(), sn, sc, V.data_ptr(), vn, vc,
                       rp.data_ptr(), ci.data_ptr(), val.data_ptr(), src.data_ptr(), resid.data_ptr(),
                       stream_ptr(self.device))
        else:
            _capi.call("tpf_residual_order_c128", S.shape[1], self.b, S.data_ptr(), sn, sc, V.data_ptr(), vn, vc,
                       rp.data_ptr(), ci.data_ptr(), val.data_ptr(), src.data_ptr(), order.data_ptr(),
                       resid.data_ptr(), stream_ptr(self.device))


def batch_solve_sparse(model, loads: LoadMatrix, opts: SolveOptions = SolveOptions(),
                       max_nnz: int | None = None, *, device=None, devices=None,
                       return_on_device: bool = False, chunk_cases: int = 0,
                       use_tree: bool = True, dtype=None) -> VoltageBatch:
    """GPU ``batch_solve_sparse`` (sparse.py:167-207); see module docstring.

    ``devices=[...]``: contiguous case slices solved concurrently, one host
    pipeline per device, after the one host factorization (bitwise the same
    result as one device).  ``dtype=numpy.complex64`` runs the c64 twin (FP32
    general CSR kernel, one device; pass a tolerance >= ~1e-6).
    """
    loads = as_load_matrix(loads, dtype)
    if not model.zip.is_constant_power:
        raise ValueError("the sparse batch path supports constant-power loads only")
    if loads.n_demand != model.n_demand:
        raise ValueError(f"load matrix has {loads.n_demand} rows, model has {model.n_demand}")
    if max_nnz is not None:
        total = int(model.admittance.y_dd.nnz) * loads.tau
        if total > max_nnz:
            raise MemoryGuardError(
                f"block system would hold {total} nonzeros (> {max_nnz}); "
                "chunk the batch over cases and solve the chunks separately")
    dt = engine_dtype(dtype)
    if not return_on_device and dt == np.complex128:
        return _solve_host_pipeline(model, loads, opts, resolve_devices(device, devices), chunk_cases, use_tree)
    if devices is not None and len(devices) > 1:
        raise ValueError("return_on_device=True and dtype=complex64 run on a single device")
    op = SparseOperator(model, devices[0] if devices else device, use_tree=use_tree, dtype=dt)
    S = loads_to_device(loads.values, op.device, dt)
    resid = torch.empty(S.shape[1], dtype=torch.float64, device=op.device)
    V, iters = op.solve(S, opts, resid=resid)
    out = (resid, torch.empty(S.shape[1], dtype=torch.uint8, device=op.device),
           torch.empty(2, dtype=torch.int32, device=op.device))
    resid, mask, summ = residual_and_summary(op.contract, S, V, iters, opts.residual_tolerance, op.device,
                                             out=out, have_resid=True)
    return finish(V, iters, resid, mask, summ, return_on_device)


def _nonempty(a):
    a = np.ascontiguousarray(a)
    return a if a.size else np.zeros(1, dtype=a.dtype)


def _batch_lu(contract, use_tree: bool):
    """The batch's factorization of Y_dd and its kernel schedule, once per
    batch like the reference's (sparse.py:186), so ``factorization_count``
    counts factorizations that ran: radial feeders by their tree elimination
    (``tree_direct``, no fill), meshed networks by SuperLU.  Nothing is
    memoised: the host setup is part of every call, as it is of the
    reference's."""
    levels = radial_levels(contract) if use_tree else None  # a radial feeder: its tree elimination
    f = None
    if levels is None:
        f = factorize_ydd(contract.y_dd)
        levels = tree_levels(f, contract.src) if use_tree else None
    sub = None
    if levels is not None and contract.b >= SUBTREE_MIN_B:
        from .subtree import subtree_schedule
        sub = subtree_schedule(levels, *host_csr(contract))
    tree = tree_limits(levels) if levels is not None and sub is None else None
    if f is None and sub is None and tree is None:
        f = factorize_ydd(contract.y_dd, count=False)  # the general kernel's LU of the same matrix
    return f, tree, sub


def _solve_host_pipeline(model, loads: LoadMatrix, opts: SolveOptions, devs, chunk_cases: int,
                         use_tree: bool = True):
    c = ModelContract.of(model)
    f, tree, sub = _batch_lu(c, use_tree)  # one factorization per batch, shared by every device
    rp, ci, yv = host_csr(c)
    S, sn, sc = host_loads(loads.values)
    b, tau = S.shape
    V = host_empty((b, tau), np.complex128)
    iters = host_empty((tau,), np.int32)
    resid = host_empty((tau,), np.float64)
    mask = host_empty((tau,), np.uint8)
    v_flat = complex(abs(c.v_s))
    arrs = [] if f is None else [_nonempty(x) for x in (f.l_ptr, f.l_col, f.l_val, f.u_ptr, f.u_col, f.u_val,
                                                        f.u_diag_inv, f.perm)]
    lib = _capi.load()

    def call(dev, lo, hi, slot):
        n = hi - lo
        summ = np.zeros(2, dtype=np.int32)
        if n == 0:
            return summ
        outs = (ptr(V) + 16 * lo, tau, 1, ptr(iters) + 4 * lo, ptr(resid) + 8 * lo, ptr(mask) + lo, ptr(summ),
                int(chunk_cases), dev.index)
        s_lo = ptr(S) + 16 * lo * sc
        if sub is not None:
            ws = device_workspace_slot(dev, lib.tpf_sparse_subtree_solve_host_workspace_bytes(
                n, b, sub.NS, sub.NT, sub.RW, int(sub.kids.size), int(chunk_cases), yv.size), slot)
            torch.cuda.current_stream(dev).synchronize()
            _capi.call("tpf_sparse_subtree_solve_host_c128", n, b, sub.NS, sub.NT, sub.RMAX, sub.RW,
                       int(sub.kids.size), ptr(sub.pinfo), ptr(sub.slotinfo), ptr(sub.kids), ptr(sub.coef),
                       ptr(sub.ell_col), ptr(sub.ell_val), s_lo, sn, sc, ptr(rp), ptr(ci), ptr(yv), ptr(c.src),
                       v_flat.real, v_flat.imag, float(opts.tolerance), int(opts.max_iterations),
                       float(opts.residual_tolerance), *outs, ws.data_ptr(), ws.numel())
            return summ
        if tree is not None:
            ws = device_workspace_slot(
                dev, lib.tpf_sparse_tree_solve_host_workspace_bytes(n, b, int(chunk_cases), yv.size), slot)
            torch.cuda.current_stream(dev).synchronize()
            _capi.call("tpf_sparse_tree_solve_host_c128", n, b, tree.levels, ptr(tree.level_info),
                       ptr(tree.node_info), ptr(tree.node_coef), s_lo, sn, sc, ptr(rp), ptr(ci), ptr(yv),
                       ptr(c.src), v_flat.real, v_flat.imag, float(opts.tolerance), int(opts.max_iterations),
                       float(opts.residual_tolerance), *outs, ws.data_ptr(), ws.numel())
            return summ
        ws = device_workspace_slot(dev, lib.tpf_sparse_solve_host_workspace_bytes(
            n, b, int(chunk_cases), yv.size, f.l_col.size, f.u_col.size), slot)
        torch.cuda.current_stream(dev).synchronize()  # the pipeline runs on its own streams
        _capi.call("tpf_sparse_solve_host_c128", n, b, s_lo, sn, sc, *[ptr(x) for x in arrs],
                   ptr(rp), ptr(ci), ptr(yv), ptr(c.src), v_flat.real, v_flat.imag, float(opts.tolerance),
                   int(opts.max_iterations), float(opts.residual_tolerance), *outs, ws.data_ptr(), ws.numel())
        return summ

    parts = run_sliced(devs, tau, call, (S,)) if len(devs) > 1 else [call(devs[0], 0, tau, 0)]
    return VoltageBatch(values=V, iterations=max(int(p[0]) for p in parts), converged_mask=mask.astype(bool),
                        residuals=resid, iterations_per_case=iters)
