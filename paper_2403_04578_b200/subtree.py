"""Warp-per-subtree schedule for the radial sparse kernel (``tpf_sparse_subtree_fpi_c128``).

The sparse fixed point (sparse.py:186-197 restated as ``Y_dd v' = -(s*/conj(v)
+ src)``, one LU of Y_dd for every case) on a radial feeder is an up-sweep
(children before parents) and a down-sweep (parents before children) of the
tree LU per iteration (``tree_levels``).  The level kernel synchronises the
whole CTA at every depth level (14 barriers per iteration at C3).  This
schedule cuts the tree at depth ``D``:

* the nodes of depth < D form the *top* (21 nodes at C3), swept redundantly
  by every warp on its own private copy;
* every node of depth D roots a *subtree*; subtrees are packed onto the W
  warps of the CTA (largest first, balancing the per-warp slot count), so a
  warp sweeps its subtrees with ``__syncwarp`` only.

One iteration is then: every warp's subtree up-sweep, ONE CTA barrier (the
subtree roots' child sums, double-buffered by iteration parity in
``Proot``), the top up- and down-sweep (per warp, redundant), the warp's
subtree down-sweep.  The step test of iteration k is AND-reduced at the
barrier of iteration k + 1.

Slots: thread ``lane`` of warp ``w`` owns, in slot ``j`` (0 <= j < NSL), the
node at position ``p = (w * NSL + j) * 32 + lane`` (or nothing).  Within a
warp the slots are in up-sweep order: leaves below depth D (all independent),
internal nodes by decreasing depth, the depth-D roots, then the top slots
(depth D-1 first).  ``sync`` bit j marks a group change between slots j and
j + 1 (a ``__syncwarp``).  Arithmetic per node is that of the level kernel
(same coefficients, same child order), so both kernels give the same bits.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["SubtreeSchedule", "subtree_schedule", "subtree_solve_host", "SUB_WARPS", "SUB_NSL"]

SUB_WARPS = 12                       # CTA = 384 threads, 3 warps per TMEM lane quadrant
SUB_NSL = (6, 9, 12, 15, 18, 21)     # slots per thread the kernel is compiled for (V+S: 8 TMEM columns each)
SUB_SMEM_MAX = 227 * 1024
PARENT_NONE = -32768


@dataclass
class SubtreeSchedule:
    b: int
    W: int
    NSL: int          # slots per thread (compiled value)
    NS: int           # subtree slots per warp (padded); top slots are NS..NSL-1
    NT: int           # top slots
    D: int            # cut depth
    RMAX: int         # root slots per warp (Proot stride)
    RW: int           # residual row width (ELL)
    P: int            # positions = W * NSL * 32
    meta: np.ndarray  # int32 [2W]: first depth-D slot per warp, sync mask per warp
    pinfo: np.ndarray  # int32 [P, 2]
    kids: np.ndarray   # uint16 [nk]
    coef: np.ndarray   # complex128 [3, P]: g, 1/U[m,m], src
    ell_col: np.ndarray  # int32 [RW, P] original column indices (CSR order), -1 padding
    ell_val: np.ndarray  # complex128 [RW, P]
    m_at: np.ndarray     # int32 [P]: level-order node at each position (-1 empty), host tests
    smem_bytes: int


def _pack(lo16: int, hi16: int) -> int:
    v = (lo16 & 0xFFFF) | ((hi16 & 0xFFFF) << 16)
    return v - (1 << 32) if v >= (1 << 31) else v


def subtree_schedule(t, rp: np.ndarray, ci: np.ndarray, yv: np.ndarray, W: int = SUB_WARPS):
    """Build the schedule from a ``tree_levels`` layout and Y_dd in CSR
    (original order, for the fused residual), or None if the feeder does not
    fit the kernel (slots, shared memory, 16-bit codes)."""
    b, L = t.b, t.levels
    if L < 2 or b >= 0xFFFF:
        return None
    offs = t.level_info[:L + 1].astype(np.int64)
    info = t.node_info.reshape(b, 4).astype(np.int64)
    orig, pm, first, cnt = info[:, 0], info[:, 1], info[:, 2], info[:, 3]
    coef4 = t.node_coef.reshape(4, b)
    depth = np.repeat(np.arange(L), np.diff(offs))
    leaf = cnt == 0
    sizes = np.diff(offs)

    best = None
    for D in range(1, L):
        root_of = np.arange(b)
        for _ in range(L):
            root_of = np.where(depth[root_of] > D, pm[np.maximum(root_of, 0)], root_of)
        # group index per node of depth >= D, in up order: 0 = leaves below D,
        # 1.. = internal depth L-2 .. D+1, last = depth D
        ng = 1 + max(0, L - 2 - D) + 1
        grp = np.full(b, -1, dtype=np.int64)
        sub = depth >= D
        grp[sub & leaf & (depth > D)] = 0
        inner = sub & ~leaf & (depth > D)
        grp[inner] = 1 + (L - 2 - depth[inner])
        grp[depth == D] = ng - 1
        roots = np.arange(offs[D], offs[D + 1])
        cnts = np.zeros((roots.size, ng), dtype=np.int64)
        np.add.at(cnts, (root_of[sub] - offs[D], grp[sub]), 1)
        order = np.argsort(-cnts.sum(1), kind="stable")
        load = np.zeros((W, ng), dtype=np.int64)
        owner = np.empty(roots.size, dtype=np.int64)
        for r in order:
            trial = load + cnts[r]
            slots = (-(-trial // 32)).sum(1)
            w = int(np.lexsort((trial.sum(1), slots))[0])
            load[w] += cnts[r]
            owner[r] = w
        ns = int((-(-load // 32)).sum(1).max())
        nt = int((-(-sizes[:D] // 32)).sum())
        rmax = int((-(-load[:, ng - 1] // 32)).max())
        key = (ns + nt, nt)
        if best is None or key < best[0]:
            best = (key, D, ns, nt, rmax, root_of, grp, owner, ng)
    (_, D, ns, nt, rmax, root_of, grp, owner, ng) = best
    nsl = next((n for n in SUB_NSL if n >= ns + nt), None)
    if nsl is None:
        return None
    NS = nsl - nt
    P = W * nsl * 32
    if P > 0x8000 or W * rmax * 32 > 0x4000:
        return None

    pos = np.full(b, -1, dtype=np.int64)     # subtree nodes: absolute position
    qidx = np.full(b, -1, dtype=np.int64)    # top nodes: top index q
    rho = np.full(b, -1, dtype=np.int64)     # subtree roots: Proot index
    m_at = np.full(P, -1, dtype=np.int64)
    meta = np.zeros(2 * W, dtype=np.int64)
    warp_of = np.where(depth >= D, owner[np.clip(root_of - offs[D], 0, owner.size - 1)], -1)
    for w in range(W):
        j = 0
        mask = 0
        for gidx in range(ng):
            nodes = np.nonzero((depth >= D) & (warp_of == w) & (grp == gidx))[0]
            if nodes.size == 0:
                continue
            if gidx == ng - 1:
                meta[w] = j
            for k, m in enumerate(nodes):  # nodes are in level order (sorted m)
                p = (w * nsl + j + k // 32) * 32 + k % 32
                pos[m] = p
                m_at[p] = m
                if gidx == ng - 1:
                    rho[m] = (w * rmax + k // 32) * 32 + k % 32
            j += -(-nodes.size // 32)
            mask |= 1 << (j - 1)
        assert j <= NS
        meta[W + w] = mask
    # top: depth D-1 first (up order), slots NS.., top index q = (slot - NS) * 32 + lane
    tj = 0
    tmask = 0
    for d in range(D - 1, -1, -1):
        nodes = np.arange(offs[d], offs[d + 1])
        for k, m in enumerate(nodes):
            q = (tj + k // 32) * 32 + k % 32
            qidx[m] = q
        tj += -(-nodes.size // 32)
        tmask |= 1 << (NS + tj - 1)
    assert tj == nt
    for w in range(W):
        meta[W + w] |= tmask
        for m in range(offs[D]):
            p = (w * nsl + NS) * 32 + qidx[m]
            m_at[p] = m

    # child lists (shared by the W copies of a top node) and per-position info
    kid_first = np.zeros(b, dtype=np.int64)
    kid_list = []
    for m in range(b):
        kid_first[m] = len(kid_list)
        for c in range(first[m], first[m] + cnt[m]):
            if depth[c] < D:
                kid_list.append(0x8000 + qidx[c])
            elif depth[c] == D:
                kid_list.append(0xC000 + rho[c])
            else:
                kid_list.append(pos[c])
    kids = np.asarray(kid_list if kid_list else [0], dtype=np.uint16)
    if len(kid_list) >= 0xFFFF or cnt.max(initial=0) > 255:
        return None
    # residual rows: Y_dd CSR (original order) per position
    rlen_node = np.diff(rp)[orig]
    RW = int(rlen_node.max(initial=1))
    if RW > 16:
        return None
    pinfo = np.zeros((P, 2), dtype=np.int64)
    coef = np.zeros((3, P), dtype=np.complex128)
    ell_col = np.full((RW, P), -1, dtype=np.int32)
    ell_val = np.zeros((RW, P), dtype=np.complex128)
    for p in range(P):
        m = m_at[p]
        if m < 0:
            pinfo[p] = (0, _pack(0, 0xFFFF))
            continue
        w = p // (nsl * 32)
        if pm[m] < 0:
            pc = PARENT_NONE
        elif depth[pm[m]] < D:
            pc = -1 - int(qidx[pm[m]])
        else:
            pc = int(pos[pm[m]])
        is_top_copy = depth[m] < D
        rl = int(rlen_node[m]) if (not is_top_copy or w == 0) else 0
        pinfo[p, 0] = _pack(pc, int(kid_first[m]))
        pinfo[p, 1] = _pack(int(cnt[m]) | (rl << 8), int(orig[m]))
        coef[0, p] = coef4[1, m]
        coef[1, p] = coef4[2, m]
        coef[2, p] = coef4[3, m]
        i = int(orig[m])
        lo, hi = int(rp[i]), int(rp[i + 1])
        ell_col[:hi - lo, p] = ci[lo:hi]
        ell_val[:hi - lo, p] = yv[lo:hi]
    xcap = max(P, -(-b // 256) * 256)
    smem = xcap * 16 + P * 8 + kids.size * 2 + 2 * W * rmax * 32 * 16 + 1024
    smem = (smem + 15) // 16 * 16
    if smem > SUB_SMEM_MAX:
        return None
    return SubtreeSchedule(b=b, W=W, NSL=nsl, NS=NS, NT=nt, D=D, RMAX=rmax, RW=RW, P=P,
                           meta=meta.astype(np.int32), pinfo=pinfo.astype(np.int32), kids=kids,
                           coef=coef, ell_col=ell_col, ell_val=ell_val, m_at=m_at.astype(np.int32),
                           smem_bytes=int(smem))


def subtree_solve_host(s: SubtreeSchedule, rhs: np.ndarray) -> np.ndarray:
    """Numpy emulation of one solve ``Y_dd x = rhs`` in the kernel's order and
    storage (positions, private top copies, Proot, child codes); host tests
    compare it bit for bit with ``sparse.tree_solve_host``."""
    W, NSL, NS = s.W, s.NSL, s.NS
    P = s.P
    X = np.zeros(P, dtype=complex)
    Proot = np.zeros(W * s.RMAX * 32, dtype=complex)
    Z = np.zeros(P, dtype=complex)
    pinfo = s.pinfo.astype(np.int64) & 0xFFFFFFFF
    parent = ((pinfo[:, 0] & 0xFFFF) ^ 0x8000) - 0x8000
    kfirst = pinfo[:, 0] >> 16
    kcnt = pinfo[:, 1] & 0xFF
    orig = pinfo[:, 1] >> 16
    g, uinv = s.coef[0], s.coef[1]

    def child_val(w, code):
        if code >= 0xC000:
            return Proot[code - 0xC000]
        if code >= 0x8000:
            return X[(w * NSL + NS) * 32 + code - 0x8000]
        return X[code]

    def up(w, j):
        for lane in range(32):
            p = (w * NSL + j) * 32 + lane
            if orig[p] == 0xFFFF:
                continue
            z = rhs[orig[p]]
            for k in range(kcnt[p]):
                z = z - child_val(w, int(s.kids[kfirst[p] + k]))
            Z[p] = z
            X[p] = g[p] * z
            if j >= s.meta[w] and j < NS and parent[p] != -32768 and parent[p] < 0:
                Proot[(w * s.RMAX + j - s.meta[w]) * 32 + lane] = X[p]

    def down(w, j):
        for lane in range(32):
            p = (w * NSL + j) * 32 + lane
            if orig[p] == 0xFFFF:
                continue
            x = Z[p] * uinv[p]
            pc = parent[p]
            if pc != -32768:
                wp = X[(w * NSL + NS) * 32 + (-1 - pc)] if pc < 0 else X[pc]
                x = x - g[p] * wp
            X[p] = x

    for w in range(W):
        for j in range(NS):
            up(w, j)
    out = np.empty(s.b, dtype=complex)
    for w in range(W):
        for j in range(NS, NSL):
            up(w, j)
        for j in range(NSL - 1, -1, -1):
            down(w, j)
        for j in range(NSL):
            for lane in range(32):
                p = (w * NSL + j) * 32 + lane
                if orig[p] != 0xFFFF:
                    out[orig[p]] = X[p]
    return out
