"""Warp-per-subtree schedule for the radial sparse kernel (``tpf_sparse_subtree_fpi_c128``).

The sparse fixed point (sparse.py:186-197 restated as ``Y_dd v' = -(s*/conj(v)
+ src)``, one LU of Y_dd for every case) on a radial feeder is an up-sweep
(children before parents) and a down-sweep (parents before children) of the
tree LU per iteration (``sparse.tree_levels`` / ``sparse.tree_direct``).  The
level kernel synchronises the whole CTA at every depth level (14 barriers per
iteration at C3).  This schedule cuts the tree at depth ``D``:

* the nodes of depth < D form the *top* (21 nodes at C3), swept redundantly
  by every warp on its own private copy (shared memory);
* every node of depth D roots a *subtree*; subtrees are packed onto the W
  warps of the CTA (largest first onto the least loaded warp), and each
  warp's nodes are list-scheduled into *slots* of 32 mutually independent
  nodes by Hu's rule (a node goes to the first slot after all of its
  children's; the deepest ready nodes first), so a warp sweeps its subtrees
  with one ``__syncwarp`` per step and no CTA barrier; consecutive slots with
  no parent-child pair between them are marked and swept two at a time.
  The cut depth is the one with the fewest slots (subtree + top); a cut whose
  Hu lower bound max_w max(ceil(n_w / 32), height_w) cannot win is skipped.

One iteration is then: every warp's subtree up-sweep, ONE CTA barrier (the
subtree roots' child products cross warps through ``Proot``, double-buffered
by iteration parity; the barrier also AND-reduces the previous iteration's
step test), the top up- and down-sweep (per warp, redundant), the warp's
subtree down-sweep.

Slots: thread ``lane`` of warp ``w`` owns, in slot ``j`` (0 <= j < NSL), the
node at position ``p = (w * NSL + j) * 32 + lane`` (or nothing).  Slots
``0 .. NS-1`` are subtree slots (iterate and load in Tensor Memory, plus
z / U_mm for slots with an internal node; leaf-only slots recompute it),
slots ``NS ..`` the top (depth D-1 first).  Arithmetic per node is that of
the level kernel (same coefficients, same child order), so both kernels give
the same bits.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np

__all__ = ["SubtreeSchedule", "subtree_schedule", "subtree_solve_host", "SUB_WARPS", "SUB_MAX_NS"]

SUB_WARPS = 12           # CTA = 384 threads, 3 warps per TMEM lane quadrant
SUB_TMEM_COLS = 168      # TMEM columns per warp (3 column groups of 168 <= 512)
SUB_MAX_NS = 20          # subtree slots per thread (V, S: 8 TMEM columns; y: 4 more unless leaves only)
SUB_KMAX = 15            # children per node (4-bit count)
SUB_RWMAX = 8            # Y_dd row width of the fused residual (diagonal + parent + children)
SUB_SMEM_MAX = 227 * 1024


@dataclass
class SubtreeSchedule:
    b: int
    W: int
    NS: int           # subtree slots per thread
    NT: int           # top slots
    NSL: int          # NS + NT
    D: int            # cut depth
    RMAX: int         # root slots per warp (Proot stride)
    RW: int           # residual row width (ELL)
    P: int            # positions = W * NSL * 32
    NY: int           # TMEM y slots per thread (slots holding an internal node)
    slotinfo: np.ndarray  # int32 [W, NS]: kmax (4 bits) | pair-with-next (bit 4) | y slot + 1 (bits 5-9)
    #                       | widest residual row (bits 10-13)
    pinfo: np.ndarray  # int32 [P, 2]
    kids: np.ndarray   # uint16 [nk] X indices of children
    coef: np.ndarray   # complex128 [3, P]: g, 1/U[m,m], src
    ell_col: np.ndarray  # int32 [P / 32, RW, 32] original column indices (CSR order); padding: X's zero entry
    ell_val: np.ndarray  # complex128 [P / 32, RW, 32] (padding 0)
    m_at: np.ndarray     # int32 [P]: level-order node at each position (-1 empty)
    smem_bytes: int

    @property
    def kmax(self) -> np.ndarray:
        return self.slotinfo & 0xF

    @property
    def xcap(self) -> int:
        return max(self.P, -(-self.b // 256) * 256)

    @property
    def RR(self) -> int:
        return self.W * self.RMAX * 32


def _pack(lo16: int, hi16: int) -> int:
    v = (lo16 & 0xFFFF) | ((hi16 & 0xFFFF) << 16)
    return v - (1 << 32) if v >= (1 << 31) else v


def _superslots(nodes: np.ndarray, kids_of, parent, prio, width: int = 32) -> list[list[int]]:
    """List-schedule ``nodes`` (a union of subtrees; the up-sweep DAG is an
    in-forest, child -> parent) into slots of ``width`` mutually
    independent nodes: at each step the ready nodes (all children in earlier
    slots) farthest from their root go first (Hu's rule, optimal for
    unit tasks on an in-forest)."""
    nodes = [int(m) for m in nodes]
    member = set(nodes)
    left = {m: len(kids_of(m)) for m in nodes}
    ready = [(-prio[m], m) for m in nodes if left[m] == 0]
    heapq.heapify(ready)
    slots: list[list[int]] = []
    while ready:
        cur = [heapq.heappop(ready)[1] for _ in range(min(width, len(ready)))]
        slots.append(sorted(cur))
        for m in cur:
            p = int(parent[m])
            if p >= 0 and p in member:
                left[p] -= 1
                if left[p] == 0:
                    heapq.heappush(ready, (-prio[p], p))
    assert sum(len(x) for x in slots) == len(nodes)
    return slots


def subtree_schedule(t, rp: np.ndarray, ci: np.ndarray, yv: np.ndarray, W: int = SUB_WARPS):
    """Build the schedule from a ``tree_levels`` layout and Y_dd in CSR
    (original order, for the fused residual), or None if the feeder does not
    fit the kernel (TMEM slots, shared memory, 16-bit codes)."""
    b, L = t.b, t.levels
    if L < 2 or b >= 0xFFFF:
        return None
    offs = t.level_info[:L + 1].astype(np.int64)
    info = t.node_info.reshape(b, 4).astype(np.int64)
    orig, pm, first, cnt = info[:, 0], info[:, 1], info[:, 2], info[:, 3]
    if cnt.max(initial=0) > SUB_KMAX:
        return None
    coef4 = t.node_coef.reshape(4, b)
    depth = np.repeat(np.arange(L), np.diff(offs))
    sizes = np.diff(offs)

    def kids_of(m):
        return range(first[m], first[m] + cnt[m])

    # per cut depth D: subtrees packed onto warps (largest first onto the least
    # loaded); the Hu schedule is built only for the cuts whose lower bound
    # max_w max(ceil(n_w / 32), height_w) could still win
    cands = []
    for D in range(1, L):
        root_of = np.arange(b)
        for _ in range(L):
            root_of = np.where(depth[root_of] > D, pm[np.maximum(root_of, 0)], root_of)
        roots = np.arange(offs[D], offs[D + 1])
        sub = depth >= D
        size = np.bincount(root_of[sub] - offs[D], minlength=roots.size)
        height = np.zeros(roots.size, dtype=np.int64)
        np.maximum.at(height, root_of[sub] - offs[D], depth[sub] - D + 1)
        owner = np.empty(roots.size, dtype=np.int64)
        heap = [(0, w) for w in range(W)]  # (load, warp): the least loaded, lowest index first
        for r in np.argsort(-size, kind="stable").tolist():
            ld, w = heapq.heappop(heap)
            owner[r] = w
            heapq.heappush(heap, (ld + int(size[r]), w))
        load = np.bincount(owner, weights=size, minlength=W).astype(np.int64)
        warp_of = np.full(b, -1, dtype=np.int64)
        warp_of[sub] = owner[root_of[sub] - offs[D]]
        hw = np.zeros(W, dtype=np.int64)
        np.maximum.at(hw, owner, height)
        lb = max(int(np.max(np.maximum(-(-load // 32), hw))), 1)
        nt = int((-(-sizes[:D] // 32)).sum())
        pen = 12 * W * nt * 32 * 3 * 16 > 48 * 1024
        cands.append(((lb > SUB_MAX_NS, lb + nt + pen, nt), D, nt, pen, warp_of))
    cands.sort(key=lambda x: x[0])
    best = None
    for lbkey, D, nt, pen, warp_of in cands:
        if best is not None and (lbkey > best[0] or (lbkey == best[0] and D > best[1])):
            continue  # this cut cannot beat the best schedule found
        sslots = [_superslots(np.nonzero(warp_of == w)[0], kids_of, pm, depth, width=32) for w in range(W)]
        ns = max(max(len(x) for x in sslots), 1)
        rmax = int(max(-(-np.count_nonzero((warp_of == w) & (depth == D)) // 32) for w in range(W)))
        key = (ns > SUB_MAX_NS, ns + nt + pen, nt)
        if best is None or key < best[0] or (key == best[0] and D < best[1]):
            best = (key, D, ns, nt, max(rmax, 1), warp_of, sslots)
    (_, D, NS, NT, RMAX, warp_of, sslots) = best
    if NS > SUB_MAX_NS:
        return None
    NSL = NS + NT
    P = W * NSL * 32
    xcap = max(P, -(-b // 256) * 256)
    RR = W * RMAX * 32
    if xcap + 2 * RR + 1 >= 0xFFFF or RR >= 1 << 12:
        return None

    pos = np.full(b, -1, dtype=np.int64)     # subtree nodes: absolute position
    qidx = np.full(b, -1, dtype=np.int64)    # top nodes: top index q
    rho = np.full(b, -1, dtype=np.int64)     # subtree roots: Proot index
    m_at = np.full(P, -1, dtype=np.int64)
    slotinfo = np.zeros((W, NS), dtype=np.int64)
    rlen = np.diff(rp).astype(np.int64)
    ny = 0
    for w in range(W):
        if not sslots[w]:
            continue
        nodes_w = np.concatenate([np.asarray(x, dtype=np.int64) for x in sslots[w]])
        slot_w = np.repeat(np.arange(len(sslots[w])), [len(x) for x in sslots[w]])
        lane_w = np.concatenate([np.arange(len(x)) for x in sslots[w]])
        pw = (w * NSL + slot_w) * 32 + lane_w
        pos[nodes_w] = pw
        m_at[pw] = nodes_w
        rt = nodes_w[depth[nodes_w] == D]  # subtree roots, in slot order
        rho[rt] = (w * RMAX + np.arange(rt.size) // 32) * 32 + np.arange(rt.size) % 32
        km = np.zeros(len(sslots[w]), dtype=np.int64)
        np.maximum.at(km, slot_w, cnt[nodes_w])
        rwm = np.zeros(len(sslots[w]), dtype=np.int64)
        np.maximum.at(rwm, slot_w, rlen[orig[nodes_w]])  # widest residual row of the slot
        has_y = km > 0  # some internal node: z / U_mm kept in TMEM (leaf-only slots recompute it)
        ys = np.where(has_y, np.cumsum(has_y), 0)
        slotinfo[w, :len(sslots[w])] = km | (ys << 5) | (rwm << 10)
        # slots k, k+1 independent (no node of k has its parent in k + 1): swept as a pair
        par = pm[nodes_w]
        dep = (par >= 0) & (pos[np.maximum(par, 0)] // 32 == (w * NSL + slot_w + 1)) & (depth[np.maximum(par, 0)] >= D)
        blocked = np.zeros(len(sslots[w]), dtype=bool)
        blocked[slot_w[dep]] = True
        pairable = ~blocked[:-1]
        slotinfo[w, :len(sslots[w]) - 1] |= np.where(pairable, 1 << 4, 0)
        ny = max(ny, int(has_y.sum()))
    if 8 * NS + 4 * ny > SUB_TMEM_COLS or ny >= 31:
        return None
    tj = 0
    for d in range(D - 1, -1, -1):  # top: depth D-1 first (up order), index q = (slot - NS) * 32 + lane
        k = np.arange(offs[d + 1] - offs[d])
        qidx[offs[d]:offs[d + 1]] = (tj + k // 32) * 32 + k % 32
        tj += -(-k.size // 32)
    assert tj == NT
    top = np.arange(offs[D])
    for w in range(W):
        m_at[(w * NSL + NS) * 32 + qidx[top]] = top

    # X index space of the kernel: positions [0, xcap), Proot parity 0 at
    # [xcap, xcap + RR), parity 1 at [xcap + RR, xcap + 2 RR) (the kernel adds
    # RR on odd iterations), a zero entry at xcap + 2 RR.  Child lists and
    # parents are X indices; a top node's copy in warp w points into w's copy.
    def xidx(c, w):
        return np.where(depth[c] < D, (w * NSL + NS) * 32 + qidx[c],
                        np.where(depth[c] == D, xcap + rho[c], pos[c]))

    pp = np.arange(P)
    mp = m_at
    valid = mp >= 0
    mv = np.maximum(mp, 0)
    wp = pp // (NSL * 32)
    nk = np.where(valid, cnt[mv], 0)
    # one child list per position, in position order (each top node once per warp)
    kid_first_pos = np.concatenate([[0], np.cumsum(nk)[:-1]])
    tot = int(nk.sum())
    owner = np.repeat(pp, nk)
    child = np.repeat(first[mv], nk) + (np.arange(tot) - np.repeat(kid_first_pos, nk))
    kid_list = xidx(child, wp[owner]) if tot else np.zeros(0, dtype=np.int64)
    kid_first_pos = np.where(nk > 0, kid_first_pos, 0)
    # SUB_KMAX padding entries: the kernel's branch-free child sum reads up to the
    # slot's largest child count from every lane's list start
    if tot + SUB_KMAX >= 0xFFFF:
        return None
    kids = np.concatenate([kid_list, np.full(SUB_KMAX, xcap + 2 * RR)]).astype(np.uint16)
    RW = int(rlen[orig].max(initial=1))
    if RW > SUB_RWMAX:
        return None

    def pack(lo16, hi16):
        v = (np.asarray(lo16, dtype=np.int64) & 0xFFFF) | ((np.asarray(hi16, dtype=np.int64) & 0xFFFF) << 16)
        return np.where(v >= (1 << 31), v - (1 << 32), v)

    pmv = pm[mv]
    pc = np.where(pmv < 0, 0xFFFF, np.where(depth[np.maximum(pmv, 0)] < D, xidx(np.maximum(pmv, 0), wp),
                                             pos[np.maximum(pmv, 0)]))
    root = np.where(depth[mv] == D, rho[mv] + 1, 0)
    pinfo = np.zeros((P, 2), dtype=np.int64)
    pinfo[:, 0] = np.where(valid, pack(pc, kid_first_pos), pack(0xFFFF, 0))
    pinfo[:, 1] = np.where(valid, pack(cnt[mv] | (root << 4), orig[mv]), pack(0, 0xFFFF))
    coef = np.zeros((3, P), dtype=np.complex128)
    coef[:, valid] = coef4[1:4, mp[valid]]
    # ELL rows blocked by slot: entry r of position p at [p // 32, r, p % 32];
    # padding points at X's zero entry with value 0.  Residual rows: subtree
    # nodes and warp 0's top copies.
    ell_col = np.full((P // 32, RW, 32), xcap + 2 * RR, dtype=np.int32)
    ell_val = np.zeros((P // 32, RW, 32), dtype=np.complex128)
    rowp = pp[valid & ((depth[mv] >= D) | (wp == 0))]
    ri = orig[mp[rowp]]
    ln = rlen[ri]
    tot = int(ln.sum())
    rpos = np.repeat(rowp, ln)
    rr = np.arange(tot) - np.repeat(np.concatenate([[0], np.cumsum(ln)[:-1]]), ln)
    src_k = np.repeat(rp[ri].astype(np.int64), ln) + rr
    ell_col[rpos // 32, rr, rpos % 32] = ci[src_k]
    ell_val[rpos // 32, rr, rpos % 32] = yv[src_k]
    top_priv = 3 * W * NT * 32 * 16 + 3 * NT * 32 * 16
    smem = (xcap + 2 * RR + 1) * 16 + top_priv + P * 8 + W * NS * 4 + kids.size * 2 + 1024
    smem = (smem + 15) // 16 * 16
    if smem > SUB_SMEM_MAX:
        return None
    return SubtreeSchedule(b=b, W=W, NS=NS, NT=NT, NSL=NSL, D=D, RMAX=RMAX, RW=RW, P=P, NY=ny,
                           slotinfo=slotinfo.astype(np.int32), pinfo=pinfo.astype(np.int32), kids=kids,
                           coef=coef, ell_col=ell_col, ell_val=ell_val, m_at=m_at.astype(np.int32),
                           smem_bytes=int(smem))


def subtree_solve_host(s: SubtreeSchedule, rhs: np.ndarray) -> np.ndarray:
    """Numpy emulation of one solve ``Y_dd x = rhs`` in the kernel's order and
    storage (X index space with Proot and private top copies, child lists,
    parents, slots); host tests compare it bit for bit with
    ``sparse.tree_solve_host``."""
    W, NSL, NS = s.W, s.NSL, s.NS
    xcap, RR = s.xcap, s.RR
    X = np.zeros(xcap + 2 * RR + 1, dtype=complex)
    Y = np.zeros(s.P, dtype=complex)
    pinfo = s.pinfo.astype(np.int64) & 0xFFFFFFFF
    parent = pinfo[:, 0] & 0xFFFF
    kfirst = pinfo[:, 0] >> 16
    kcnt = pinfo[:, 1] & 0xF
    root = (pinfo[:, 1] >> 4) & 0xFFF
    orig = pinfo[:, 1] >> 16
    g, uinv = s.coef[0], s.coef[1]
    shift = RR  # emulate an odd iteration

    def up(w, j):
        for lane in range(32):
            p = (w * NSL + j) * 32 + lane
            if orig[p] == 0xFFFF:
                continue
            z = rhs[orig[p]]
            for k in range(kcnt[p]):
                idx = int(s.kids[kfirst[p] + k])
                z = z - X[idx + (shift if idx >= xcap else 0)]
            X[p] = g[p] * z
            if root[p]:
                X[xcap + shift + root[p] - 1] = X[p]
            Y[p] = z * uinv[p]

    def down(w, j):
        for lane in range(32):
            p = (w * NSL + j) * 32 + lane
            if orig[p] == 0xFFFF:
                continue
            x = Y[p]
            if parent[p] != 0xFFFF:
                x = x - g[p] * X[parent[p]]
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
