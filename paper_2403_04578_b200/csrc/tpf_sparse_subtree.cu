// Sparse Tensor Power Flow for radial feeders, warp-per-subtree (the
// schedule is built on the host: paper_2403_04578_b200/subtree.py).
//
// One fixed-point iteration of the reference's sparse path (sparse.py:186-197,
// restated as Y_dd v' = -(s* ./ conj(v) + src) with one LU of Y_dd for all
// cases) on a tree-structured Y_dd is an up-sweep and a down-sweep of the
// tree LU:
//     up:   z_m = r_m - sum_c P_c,   P_m = g_m z_m,    r_m = -(s_m*/conj(v_m) + src_m)
//     down: w_m = z_m / U_mm - g_m w_parent,  v'_m = w_m
// (g_m = U[m,parent] / U[m,m]; the arithmetic and the child order of the level
// kernel tpf_sparse_tree.cu, so both give the same bits).
//
// The level kernel synchronises the whole CTA at every depth level.  Here the
// tree is cut at depth D: each node of depth D roots a subtree, the subtrees
// are packed onto the 12 warps of the CTA, and a warp sweeps its subtrees with
// __syncwarp only; the few nodes above the cut (the "top") are swept by every
// warp on its own private copy.  Per iteration there is ONE CTA barrier
// (between the subtree up-sweeps and the top), which also AND-reduces the
// previous iteration's step test.  The subtree roots' child products cross
// warps through Proot, double-buffered by iteration parity.
//
// One case per CTA (one CTA per SM), persistent over cases.  Per thread and
// slot: the iterate v and the load s in Tensor Memory (8 columns per slot),
// plus z / U_mm (4 columns) for slots that hold an internal node (leaf-only
// slots recompute it in the down-sweep with the same operations); the slot
// loops are rolled.  Shared memory: the sweep exchange vector X (by
// position), the per-position structure, the child lists, Proot and the
// warps' private top copies.  Per case the loads arrive by TMA (2-D tensor
// copy of one column of the node-major S, or a 1-D bulk copy of a case-major
// column) into X in original node order, the next case's column is
// prefetched into L2 by TMA while this one iterates, and V leaves the same way
// (TMA store from X).  The residual post-check (fpi.py:221-240) is fused: the
// final V is in X in original node order, Y_dd's rows come as ELL blocks per
// slot (see the residual below).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <cstdlib>
#include <cstring>

#include "tpf_common.cuh"
#include "tpf_internal.h"

namespace tpf {
namespace {

constexpr int kSubWarps = 12;

#ifdef TPF_PHASE_TIMING
// debug build only (tools/build_timing.sh): thread 0 of every CTA accumulates
// cycles per phase: {load, subtree up, barrier wait, top, subtree down,
// retire + store, residual, end barrier + claim, cases, iterations, total}
__device__ long long g_sub_cyc[148 * 12];
#define SUB_T(v) const long long v = clock64()
#define SUB_ACC(i, t0) \
  if (tid == 0) tc[i] += clock64() - (t0)
#else
#define SUB_T(v)
#define SUB_ACC(i, t0)
#endif
constexpr int kSubThreads = 32 * kSubWarps;
constexpr int kMaxRW = 7;   // residual row width (diagonal + parent + children)
constexpr int kSubKmax = 8;  // children per node (paper_2403_04578_b200/subtree.py SUB_KMAX)

struct SubArgs {
  int64_t tau;
  int b, NS, NT, NSL, RMAX, RW, P, xcap, nkids;
  int mode;      // S: 0 node-major (2-D TMA), 1 case-major (1-D bulk)
  int vmode;     // V: the same choices
  int nbox, boxrows;
  const double2* S;
  int64_t s_case;  // mode 1: case stride (complex elements)
  double2* V;
  int64_t v_case;
  const int2* pinfo;       // [P]
  const int32_t* slotinfo; // [W][NS]
  const uint16_t* kids;    // [nkids]
  const double2* coef;     // [3][P]: g, 1/U[m,m], src
  const int32_t* ell_col;  // [RW][P]
  const double2* ell_val;  // [RW][P]
  int32_t* iters;
  double* resid;           // or null
  unsigned long long* counter;
  double2 v_flat;
  double tol2;
  int max_iter;
};

// ---- TMA / bulk-copy helpers (sm_90+ async proxy) ----
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_prefetch(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ double2 cmul_s(double2 a, double2 x) {
  return make_double2(__fma_rn(a.x, x.x, -(a.y * x.y)), __fma_rn(a.x, x.y, a.y * x.x));
}
__device__ __forceinline__ double2 cfma_sub_s(double2 acc, double2 a, double2 x) {  // acc - a*x
  return make_double2(__fma_rn(-a.x, x.x, __fma_rn(a.y, x.y, acc.x)), __fma_rn(-a.x, x.y, __fma_rn(-a.y, x.x, acc.y)));
}

// TMEM access without a compiler memory clobber: Tensor Memory is not
// addressable by ordinary loads/stores, so independent global / shared loads
// may be scheduled across these (program order among the volatile asm
// statements themselves is kept).
__device__ __forceinline__ void tld2(uint32_t taddr, D2& o) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(o.r[0]), "=r"(o.r[1]), "=r"(o.r[2]), "=r"(o.r[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tst2(uint32_t taddr, double2 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
               "r"(__double2loint(v.x)), "r"(__double2hiint(v.x)), "r"(__double2loint(v.y)), "r"(__double2hiint(v.y)));
}
__device__ __forceinline__ void twait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;"); }
__device__ __forceinline__ void twait_st() { asm volatile("tcgen05.wait::st.sync.aligned;"); }

// shared memory through 32-bit addresses (no generic-to-shared conversion per access)
__device__ __forceinline__ double2 lds2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts2(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int lds_s32(uint32_t a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int2 lds_i2(uint32_t a) {
  int2 v;
  asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
  return v;
}

__device__ __forceinline__ double2 rhs_of(double2 v, const double2 sl, const double2 src) {
  // r_m = -(s*/conj(v) + src) on the guarded v (fpi.py:39-41), s*/conj(v) = conj(s) v / |v|^2
  double m2 = __fma_rn(v.x, v.x, v.y * v.y);
  if (m2 < kZeroGuard2) {
    v = make_double2(kZeroGuard, 0.0);
    m2 = kZeroGuard * kZeroGuard;
  }
  const double r = rcp_nr(m2);
  return make_double2(-(__fma_rn(sl.x, v.x, sl.y * v.y) * r + src.x),
                      -(__fma_rn(sl.x, v.y, -(sl.y * v.x)) * r + src.y));
}

__global__ void __launch_bounds__(kSubThreads, 1)
    sparse_subtree_kernel(const __grid_constant__ SubArgs a, const __grid_constant__ CUtensorMap tmS,
                          const __grid_constant__ CUtensorMap tmV) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int RR = kSubWarps * a.RMAX * 32;
  const int P = a.P, NS = a.NS, NT = a.NT, xcap = a.xcap;
  const int NTOP = kSubWarps * NT * 32;
  double2* X = reinterpret_cast<double2*>(smem_raw);  // [xcap | Proot parity 0 | parity 1 | zero]
  double2* TV = X + xcap + 2 * RR + 1;                 // top copies: iterate, load, z / U_mm
  double2* TS = TV + NTOP;
  double2* TY = TS + NTOP;
  double2* TC = TY + NTOP;                             // top coefficients, shared: g, 1/U, src [3][NT * 32]
  int2* PI = reinterpret_cast<int2*>(TC + 3 * NT * 32);  // [P]
  int32_t* SI = reinterpret_cast<int32_t*>(PI + P);   // [W][NS]
  uint16_t* KD = reinterpret_cast<uint16_t*>(SI + kSubWarps * NS);  // [nkids]
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ int s_case, s_next;
  __shared__ double s_red[kSubWarps];
  __shared__ uint32_t s_tmem;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < P; i += kSubThreads) PI[i] = __ldg(a.pinfo + i);
  for (int i = tid; i < kSubWarps * NS; i += kSubThreads) SI[i] = __ldg(a.slotinfo + i);
  for (int i = tid; i < a.nkids; i += kSubThreads) KD[i] = __ldg(a.kids + i);
  if (tid == 0) X[xcap + 2 * RR] = make_double2(0.0, 0.0);
  for (int i = tid; i < NT * 32; i += kSubThreads) {  // warp 0's top copy: the same for every warp
    const int p = NS * 32 + i;
    TC[i] = __ldg(a.coef + p);
    TC[NT * 32 + i] = __ldg(a.coef + P + p);
    TC[2 * NT * 32 + i] = __ldg(a.coef + 2 * P + p);
  }
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  // TMEM per warp (lane quadrant warp % 4, column group warp / 4 of 168 columns):
  // iterate V at 4 j, load S at 4 (NS + j), z / U_mm of y-slot y at 4 (2 NS + y)
  const uint32_t tm = s_tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * 168);
  const uint32_t tV = tm, tS = tm + 4 * NS, tY = tm + 8 * NS;
  const int base = warp * a.NSL * 32 + lane;  // position of slot j: base + 32 j
  const int topbase = (warp * a.NSL + NS) * 32;
  const int tpriv = warp * NT * 32 + lane;    // top copy of slot t: tpriv + 32 t
  const double2* cg = a.coef;
  const double2* cu = a.coef + P;
  const uint32_t in_bytes =
      a.mode == 0 ? uint32_t(a.nbox) * uint32_t(a.boxrows) * 16u : uint32_t(a.b) * 16u;
  uint32_t xs = smem_u32(X), pi_s = smem_u32(PI), kd_s = smem_u32(KD), si_s = smem_u32(SI + warp * NS);
  // opaque to the compiler: kept in registers instead of being rematerialised
  // (S2R SR_CgaCtaId + address arithmetic) at every shared-memory access
  asm volatile("" : "+r"(xs), "+r"(pi_s), "+r"(kd_s), "+r"(si_s));
  const uint32_t tv_s = xs + 16u * uint32_t(xcap + 2 * RR + 1), ts_s = tv_s + 16u * NTOP, ty_s = ts_s + 16u * NTOP,
                 tc_s = ty_s + 16u * NTOP;
  auto SIW = [&](const int j) { return lds_s32(si_s + 4 * j); };
  const uint32_t zero_idx = uint32_t(xcap + 2 * RR);

  auto claim = [&]() {
    const unsigned long long c = atomicAdd(a.counter, 1ull);
    return c < (unsigned long long)a.tau ? int(c) : -1;
  };
  if (tid == 0) {
    s_case = claim();
    s_next = s_case >= 0 ? claim() : -1;
  }
  __syncthreads();
  uint32_t phase = 0;
#ifdef TPF_PHASE_TIMING
  long long tc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_begin = clock64();
#endif

  for (;;) {
    SUB_T(t_load);
    const int cs = s_case, nx = s_next;
    if (cs < 0) break;
    // ---- S of case cs into X (original node order); L2 prefetch of case nx ----
    if (tid == 0) {
      mbar_expect_tx(&s_bar, in_bytes);
      if (a.mode == 0) {
        for (int k = 0; k < a.nbox; ++k) tma_load_2d(X + k * a.boxrows, &tmS, 2 * cs, k * a.boxrows, &s_bar);
        if (nx >= 0)
          for (int k = 0; k < a.nbox; ++k) tma_prefetch_2d(&tmS, 2 * nx, k * a.boxrows);
      } else {
        bulk_load(X, a.S + int64_t(cs) * a.s_case, in_bytes, &s_bar);
        if (nx >= 0) bulk_prefetch(a.S + int64_t(nx) * a.s_case, in_bytes);
      }
    }
    mbar_wait(&s_bar, phase);
    phase ^= 1u;
    for (int j = 0; j < NS; ++j) {
      const uint32_t o = uint32_t(lds_i2(pi_s + 8 * (base + 32 * j)).y) >> 16;
      tst2(tS + 4 * j, o != 0xFFFFu ? lds2(xs + 16 * o) : make_double2(0.0, 0.0));
      tst2(tV + 4 * j, a.v_flat);  // flat start (dense.py:155)
    }
    for (int t = 0; t < NT; ++t) {
      const uint32_t o = uint32_t(lds_i2(pi_s + 8 * (topbase + 32 * t + lane)).y) >> 16;
      sts2(ts_s + 16 * (tpriv + 32 * t), o != 0xFFFFu ? lds2(xs + 16 * o) : make_double2(0.0, 0.0));
      sts2(tv_s + 16 * (tpriv + 32 * t), a.v_flat);
    }
    twait_st();
    __syncthreads();  // X is free for the sweeps
    SUB_ACC(0, t_load);
#ifdef TPF_PHASE_TIMING
    if (tid == 0) tc[8] += 1;
#endif

    int it = 0;
    bool small = false;
    for (;;) {
      SUB_T(t_up);
      const int shift = (it & 1) ? RR : 0;  // Proot parity
      // ---- subtree up-sweep: z_m = r_m - sum_c X[c], X[m] = g_m z_m, y_m = z_m / U_mm ----
      {
        auto up_one = [&](const int j, const D2& vv, const D2& ss, const int2 pi, const int si, const double2 g,
                          const double2 u) {
          double2 z = rhs_of(vv.get(), ss.get(), make_double2(0.0, 0.0));
          const int km = si & 0xF;
          const uint32_t kf = uint32_t(pi.x) >> 16, kc = uint32_t(pi.y) & 0xF;
#pragma unroll 4
          for (int k = 0; k < km; ++k) {  // branch-free: lanes past their own count read the zero slot
            const uint32_t e = lds_u16(kd_s + 2 * (kf + k));
            const double2 c = lds2(xs + 16 * (uint32_t(k) < kc ? e : zero_idx));
            z.x -= c.x;
            z.y -= c.y;
          }
          const double2 P_m = cmul_s(g, z);
          sts2(xs + 16 * (base + 32 * j), P_m);
          const int root = (pi.y >> 4) & 0xFFF;
          if (root) sts2(xs + 16 * (xcap + shift + root - 1), P_m);  // subtree root: to the top via Proot
          const int ys = (si >> 5) & 0x1F;
          if (ys) tst2(tY + 4 * (ys - 1), cmul_s(z, u));  // leaf-only slots recompute it later
        };
        // one step = one slot, or two independent slots; the coefficients of the
        // next step are loaded one step ahead (two register sets, loop body
        // unrolled twice so the sets alternate without moves)
        auto up_step = [&](int& j, double2& g0, double2& u0, double2& g1, double2& u1, double2& gn0, double2& un0,
                           double2& gn1, double2& un1) {
          const int p0 = base + 32 * j;
          const int si0 = SIW(j);
          const bool pair = (si0 >> 4 & 1) && j + 1 < NS;
          const int jn = j + (pair ? 2 : 1);
          if (jn < NS) {
            gn0 = __ldg(cg + base + 32 * jn);
            un0 = __ldg(cu + base + 32 * jn);
            gn1 = __ldg(cg + base + 32 * (jn + 1));
            un1 = __ldg(cu + base + 32 * (jn + 1));
          }
          if (pair) {
            D2 v0, s0, v1, s1;
            tld2(tV + 4 * j, v0);
            tld2(tS + 4 * j, s0);
            tld2(tV + 4 * (j + 1), v1);
            tld2(tS + 4 * (j + 1), s1);
            const int2 pi0 = lds_i2(pi_s + 8 * p0), pi1 = lds_i2(pi_s + 8 * (p0 + 32));
            const int si1 = SIW(j + 1);
            twait_ld();
            up_one(j, v0, s0, pi0, si0, g0, u0);
            up_one(j + 1, v1, s1, pi1, si1, g1, u1);
          } else {
            D2 v0, s0;
            tld2(tV + 4 * j, v0);
            tld2(tS + 4 * j, s0);
            const int2 pi0 = lds_i2(pi_s + 8 * p0);
            twait_ld();
            up_one(j, v0, s0, pi0, si0, g0, u0);
          }
          __syncwarp();
          j = jn;
        };
        double2 ga0 = __ldg(cg + base), ua0 = __ldg(cu + base), ga1 = __ldg(cg + base + 32), ua1 = __ldg(cu + base + 32);
        double2 gb0, ub0, gb1, ub1;
        int j = 0;
        while (j < NS) {
          up_step(j, ga0, ua0, ga1, ua1, gb0, ub0, gb1, ub1);
          if (j >= NS) break;
          up_step(j, gb0, ub0, gb1, ub1, ga0, ua0, ga1, ua1);
        }
      }
      SUB_ACC(1, t_up);
      SUB_T(t_bar);
      // the previous iteration's step test, AND over the CTA (false at it = 0); the
      // subtree roots' products are visible after this barrier
      const int conv = __syncthreads_and(small);
      SUB_ACC(2, t_bar);
      if (conv) break;
      SUB_T(t_top);
      // ---- top (every warp on its own copy): up-sweep, then down-sweep ----
      small = true;
      for (int t = 0; t < NT; ++t) {
        const int p = topbase + 32 * t + lane, q = tpriv + 32 * t;
        const int2 pi = lds_i2(pi_s + 8 * p);
        if ((uint32_t(pi.y) >> 16) != 0xFFFFu) {
          const int pc = pi.x & 0xFFFF, tq = 32 * t + lane;
          const double2 src = pc == 0xFFFF ? lds2(tc_s + 16 * (2 * NT * 32 + tq)) : make_double2(0.0, 0.0);  // next to the slack
          double2 z = rhs_of(lds2(tv_s + 16 * q), lds2(ts_s + 16 * q), src);
          const uint32_t kf = uint32_t(pi.x) >> 16, kc = uint32_t(pi.y) & 0xF;
          // children in groups of 4, their loads issued together (past the count: the zero slot)
          for (uint32_t k0 = 0; k0 < kc; k0 += 4) {
            double2 c[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              uint32_t idx = lds_u16(kd_s + 2 * (kf + k0 + u));
              if (idx >= uint32_t(xcap)) idx += shift;  // a subtree root: Proot
              c[u] = lds2(xs + 16 * (k0 + u < kc ? idx : zero_idx));
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              z.x -= c[u].x;
              z.y -= c[u].y;
            }
          }
          sts2(xs + 16 * p, cmul_s(lds2(tc_s + 16 * tq), z));
          sts2(ty_s + 16 * q, cmul_s(z, lds2(tc_s + 16 * (NT * 32 + tq))));
        }
        __syncwarp();
      }
      for (int t = NT - 1; t >= 0; --t) {
        const int p = topbase + 32 * t + lane, q = tpriv + 32 * t;
        const int2 pi = lds_i2(pi_s + 8 * p);
        if ((uint32_t(pi.y) >> 16) != 0xFFFFu) {
          const int pc = pi.x & 0xFFFF;
          double2 w = lds2(ty_s + 16 * q);
          if (pc != 0xFFFF) w = cfma_sub_s(w, lds2(tc_s + 16 * (32 * t + lane)), lds2(xs + 16 * pc));
          sts2(xs + 16 * p, w);
          double2 v = lds2(tv_s + 16 * q);
          if (__fma_rn(v.x, v.x, v.y * v.y) < kZeroGuard2) v = make_double2(kZeroGuard, 0.0);
          const double dr = w.x - v.x, di = w.y - v.y;
          if (!(__fma_rn(dr, dr, di * di) < a.tol2)) small = false;  // NaN never passes
          sts2(tv_s + 16 * q, w);
        }
        __syncwarp();
      }
      SUB_ACC(3, t_top);
      SUB_T(t_down);
      // ---- subtree down-sweep: w_m = y_m - g_m w_parent, step test |w - v|^2 < tol^2 ----
      {
        auto down_one = [&](const int j, const D2& vv, const D2& ys_or_s, const int2 pi, const int si,
                            const double2 g, const double2 u) {
          double2 v = vv.get();
          // y_m from TMEM, or (leaf-only slot) recomputed: same operations, same bits
          double2 w = ((si >> 5) & 0x1F) ? ys_or_s.get() : cmul_s(rhs_of(v, ys_or_s.get(), make_double2(0.0, 0.0)), u);
          const uint32_t pc = uint32_t(pi.x) & 0xFFFF;
          if (pc != 0xFFFF) w = cfma_sub_s(w, g, lds2(xs + 16 * pc));
          sts2(xs + 16 * (base + 32 * j), w);
          if (__fma_rn(v.x, v.x, v.y * v.y) < kZeroGuard2) v = make_double2(kZeroGuard, 0.0);
          const double dr = w.x - v.x, di = w.y - v.y;
          if ((uint32_t(pi.y) >> 16) != 0xFFFFu && !(__fma_rn(dr, dr, di * di) < a.tol2)) small = false;
          tst2(tV + 4 * j, w);
        };
        auto down_step = [&](int& j, double2& g0, double2& u0, double2& g1, double2& u1, double2& gn0,
                             double2& un0, double2& gn1, double2& un1) {
          const int p0 = base + 32 * j;
          const int si0 = SIW(j);
          const bool pair = j >= 1 && (SIW(j - 1) >> 4 & 1);
          const int jn = j - (pair ? 2 : 1);
          if (jn >= 0) {
            gn0 = __ldg(cg + base + 32 * jn);
            un0 = __ldg(cu + base + 32 * jn);
            if (jn >= 1) {
              gn1 = __ldg(cg + base + 32 * (jn - 1));
              un1 = __ldg(cu + base + 32 * (jn - 1));
            }
          }
          if (pair) {
            const int si1 = SIW(j - 1);
            D2 v0, y0, v1, y1;
            tld2(tV + 4 * j, v0);
            tld2(((si0 >> 5) & 0x1F) ? tY + 4 * (((si0 >> 5) & 0x1F) - 1) : tS + 4 * j, y0);
            tld2(tV + 4 * (j - 1), v1);
            tld2(((si1 >> 5) & 0x1F) ? tY + 4 * (((si1 >> 5) & 0x1F) - 1) : tS + 4 * (j - 1), y1);
            const int2 pi0 = lds_i2(pi_s + 8 * p0), pi1 = lds_i2(pi_s + 8 * (p0 - 32));
            twait_ld();
            down_one(j, v0, y0, pi0, si0, g0, u0);
            down_one(j - 1, v1, y1, pi1, si1, g1, u1);
          } else {
            D2 v0, y0;
            tld2(tV + 4 * j, v0);
            tld2(((si0 >> 5) & 0x1F) ? tY + 4 * (((si0 >> 5) & 0x1F) - 1) : tS + 4 * j, y0);
            const int2 pi0 = lds_i2(pi_s + 8 * p0);
            twait_ld();
            down_one(j, v0, y0, pi0, si0, g0, u0);
          }
          __syncwarp();
          j = jn;
        };
        int j = NS - 1;
        double2 ga0 = __ldg(cg + base + 32 * j), ua0 = __ldg(cu + base + 32 * j);
        double2 ga1 = j >= 1 ? __ldg(cg + base + 32 * (j - 1)) : ga0;
        double2 ua1 = j >= 1 ? __ldg(cu + base + 32 * (j - 1)) : ua0;
        double2 gb0 = ga0, ub0 = ua0, gb1 = ga1, ub1 = ua1;
        while (j >= 0) {
          down_step(j, ga0, ua0, ga1, ua1, gb0, ub0, gb1, ub1);
          if (j < 0) break;
          down_step(j, gb0, ub0, gb1, ub1, ga0, ua0, ga1, ua1);
        }
      }
      twait_st();
      SUB_ACC(4, t_down);
      ++it;
      if (it == a.max_iter) break;
    }
#ifdef TPF_PHASE_TIMING
    if (tid == 0) tc[9] += it;
#endif
    SUB_T(t_ret);
    __syncthreads();  // every warp is done with X (the cap path leaves without a barrier)
    // ---- retire: V into X in original node order (top nodes: warp 0's copy) ----
    for (int j = 0; j < NS; ++j) {
      D2 vv;
      tld2(tV + 4 * j, vv);
      twait_ld();
      const uint32_t o = uint32_t(lds_i2(pi_s + 8 * (base + 32 * j)).y) >> 16;
      if (o != 0xFFFFu) sts2(xs + 16 * o, vv.get());
    }
    if (warp == 0) {
      for (int t = 0; t < NT; ++t) {
        const uint32_t o = uint32_t(lds_i2(pi_s + 8 * (topbase + 32 * t + lane)).y) >> 16;
        if (o != 0xFFFFu) sts2(xs + 16 * o, lds2(tv_s + 16 * (tpriv + 32 * t)));
      }
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      if (a.vmode == 0) {
        for (int k = 0; k < a.nbox; ++k) tma_store_2d(&tmV, 2 * cs, k * a.boxrows, X + k * a.boxrows);
      } else {
        bulk_store(a.V + int64_t(cs) * a.v_case, X, uint32_t(a.b) * 16u);
      }
      bulk_commit();
      a.iters[cs] = it;
    }
    SUB_ACC(5, t_ret);
    SUB_T(t_res);
    if (a.resid) {
      // residual_per_case (fpi.py:221-240): max_i |s_i + v_i conj(src_i + (Y_dd v)_i)|,
      // the operations of residual_kernel in the same order (Y_dd rows in CSR
      // order).  ELL block of slot j: entry r of the lane's row at
      // ((warp * NSL + j) * RW + r) * 32 + lane (one base, immediate offsets, coalesced);
      // rows narrower than the slot's widest are padded with the zero entry of X and
      // value 0 (adds +-0: the same magnitude, hence the same hypot).  The next
      // slot's row is loaded while this one is summed (two register sets).
      double worst = 0.0, thr = -1.0;
      const int nres = NS + (warp == 0 ? NT : 0);
      auto rw_of = [&](const int j) { return j < NS ? (SIW(j) >> 10) & 0xF : a.RW; };
      auto load_row = [&](const int j, const int rw, int (&c)[kMaxRW], double2 (&y)[kMaxRW]) {
        const size_t o = size_t((warp * a.NSL + j) * a.RW) * 32 + lane;
        const int32_t* cp = a.ell_col + o;
        const double2* vp = a.ell_val + o;
#pragma unroll
        for (int r = 0; r < kMaxRW; ++r) {  // every element assigned: no stale values kept live
          c[r] = r < rw ? __ldg(cp + 32 * r) : 0;
          y[r] = r < rw ? __ldg(vp + 32 * r) : make_double2(0.0, 0.0);
        }
      };
      auto row = [&](const int j, const int rw, const int (&c)[kMaxRW], const double2 (&y)[kMaxRW]) {
        const uint32_t o = uint32_t(lds_i2(pi_s + 8 * (base + 32 * j)).y) >> 16;
        double2 sl;
        if (j < NS) {
          D2 sd;
          tld2(tS + 4 * j, sd);
          twait_ld();
          sl = sd.get();
        } else {
          sl = lds2(ts_s + 16 * (tpriv + 32 * (j - NS)));
        }
        if (o == 0xFFFFu) return;  // no node at this position
        // src is zero below the cut: the loaded +0 and the literal +0 give the same bits
        const double2 si = j >= NS ? lds2(tc_s + 16 * (2 * NT * 32 + 32 * (j - NS) + lane)) : make_double2(0.0, 0.0);
        double ar = si.x, ai = si.y;
#pragma unroll
        for (int r = 0; r < kMaxRW; ++r)
          if (r < rw) {
            const double2 v = lds2(xs + 16 * uint32_t(c[r]));
            ar = __fma_rn(y[r].x, v.x, __fma_rn(-y[r].y, v.y, ar));
            ai = __fma_rn(y[r].x, v.y, __fma_rn(y[r].y, v.x, ai));
          }
        const double2 v = lds2(xs + 16 * o);
        const double mr = sl.x + (v.x * ar + v.y * ai);
        const double mi = sl.y + (v.y * ar - v.x * ai);
        // hypot only where it can raise the maximum: m2 <= thr = worst^2 (1 - 1e-13)
        // bounds |m| below worst by far more than the rounding of m2 and of hypot;
        // NaN and inf always take the hypot, so the max is that of every row
        const double m2 = __fma_rn(mr, mr, mi * mi);
        if (!(m2 <= thr)) {
          worst = nanmax(worst, hypot(mr, mi));
          thr = worst > 1e-150 ? worst * worst * (1.0 - 1e-13) : -1.0;
        }
      };
      int ca[kMaxRW], cb[kMaxRW];
      double2 ya[kMaxRW], yb[kMaxRW];
      int rwa = rw_of(0), rwb = 0;
      load_row(0, rwa, ca, ya);
      for (int j = 0; j < nres; j += 2) {
        if (j + 1 < nres) {
          rwb = rw_of(j + 1);
          load_row(j + 1, rwb, cb, yb);
        }
        row(j, rwa, ca, ya);
        if (j + 1 >= nres) break;
        if (j + 2 < nres) {
          rwa = rw_of(j + 2);
          load_row(j + 2, rwa, ca, ya);
        }
        row(j + 1, rwb, cb, yb);
      }
      for (int o = 16; o > 0; o >>= 1) worst = nanmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
      if (lane == 0) s_red[warp] = worst;
    }
    SUB_ACC(6, t_res);
    SUB_T(t_end);
    fence_async_smem();  // generic accesses to X before the next case's TMA load into it
    __syncthreads();     // X reads of the residual done; s_red complete
    if (tid == 0) {
      if (a.resid) {
        double w = 0.0;
        for (int k = 0; k < kSubWarps; ++k) w = nanmax(w, s_red[k]);
        a.resid[cs] = w;
      }
      bulk_wait_read0();  // the V store has read X
      s_case = nx;
      s_next = nx >= 0 ? claim() : -1;
    }
    __syncthreads();
    SUB_ACC(7, t_end);
  }
#ifdef TPF_PHASE_TIMING
  if (tid == 0 && blockIdx.x < 148) {
    tc[10] = clock64() - t_begin;
    for (int i = 0; i < 12; ++i) g_sub_cyc[blockIdx.x * 12 + i] = tc[i];
  }
#endif
  if (tid == 0) bulk_wait0();
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(s_tmem, 512);
}

// dst[c * ldd + r] = src[r * lds + c] for r < R, c < C (complex128), 32 x 32
// tiles through shared memory: coalesced on both sides.  Node-major S
// (b rows of cases) <-> case-major chunks (rows of b nodes) for the subtree
// kernel, whose per-case column is then one contiguous 16 b-byte block.
__global__ void __launch_bounds__(256) transpose_c128_kernel(const double2* __restrict__ src, int64_t lds,
                                                             double2* __restrict__ dst, int64_t ldd, int64_t R,
                                                             int64_t C) {
  __shared__ double2 tile[32][33];
  const int64_t c0 = int64_t(blockIdx.x) * 32, r0 = int64_t(blockIdx.y) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i, c = c0 + tx;
    if (r < R && c < C) tile[i][tx] = src[r * lds + c];
  }
  __syncthreads();
#pragma unroll
  for (int i = ty; i < 32; i += 8) {
    const int64_t c = c0 + i, r = r0 + tx;
    if (r < R && c < C) dst[c * ldd + r] = tile[tx][i];
  }
}

int transpose_c128(const double2* src, int64_t lds, double2* dst, int64_t ldd, int64_t R, int64_t C,
                   cudaStream_t st) {
  if (R <= 0 || C <= 0) return TPF_OK;
  const int64_t gx = (C + 31) / 32, gy = (R + 31) / 32;
  if (gx > 0x7fffffff || gy > 65535) return set_error(TPF_ERR_INVALID, "transpose_c128: matrix too large");
  transpose_c128_kernel<<<dim3(unsigned(gx), unsigned(gy)), dim3(32, 8), 0, st>>>(src, lds, dst, ldd, R, C);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? TPF_OK : set_cuda_error("launch(transpose_c128_kernel)", err);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// one column (case) of a node-major b x tau complex matrix = a box of 2 doubles x rows
int column_map(CUtensorMap* m, const void* base, int64_t tau, int b, int64_t node_stride, int boxrows) {
  auto fn = encode_fn();
  if (!fn) return set_error(TPF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cuuint64_t(2 * tau), cuuint64_t(b)};
  cuuint64_t strides[1] = {cuuint64_t(node_stride) * 16u};
  cuuint32_t box[2] = {2u, cuuint32_t(boxrows)};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(TPF_ERR_INVALID, "cuTensorMapEncodeTiled failed (alignment or strides)");
  return TPF_OK;
}

int sub_launch(const SubArgs& a, const CUtensorMap& ms, const CUtensorMap& mv, size_t smem, int grid,
               cudaStream_t st) {
  auto kern = sparse_subtree_kernel;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (err != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(subtree)", err);
  kern<<<unsigned(grid), kSubThreads, smem, st>>>(a, ms, mv);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(sparse_subtree_kernel)", err);
  return TPF_OK;
}

}  // namespace
}  // namespace tpf

using namespace tpf;

extern "C" int tpf_sparse_subtree_warps(void) { return kSubWarps; }

#ifdef TPF_PHASE_TIMING
extern "C" int tpf_debug_subtree_phase_cycles(long long* out) {
  return cudaMemcpyFromSymbol(out, g_sub_cyc, sizeof(g_sub_cyc)) == cudaSuccess ? 0 : 1;
}
#endif

constexpr int64_t kSubChunk = 65536;  // cases per case-major chunk of a node-major batch

extern "C" size_t tpf_sparse_subtree_workspace_bytes(int64_t tau, int32_t b) {
  const int64_t chunk = tau < kSubChunk ? tau : kSubChunk;
  return 256 + size_t(2) * size_t(chunk > 0 ? chunk : 0) * size_t(b > 0 ? b : 0) * 16;
}

extern "C" size_t tpf_sparse_subtree_smem_bytes(int32_t b, int32_t ns, int32_t nt, int32_t rmax, int32_t nkids) {
  const int64_t P = int64_t(kSubWarps) * (ns + nt) * 32;
  const int boxrows = b < 256 ? b : 256;
  const int64_t nbox = (b + boxrows - 1) / boxrows;
  const int64_t xcap = P > nbox * boxrows ? P : nbox * boxrows;
  return size_t(xcap + int64_t(2) * kSubWarps * rmax * 32 + 1) * 16 + size_t(3) * kSubWarps * nt * 32 * 16 +
         size_t(3) * nt * 32 * 16 +
         size_t(P) * 8 + size_t(kSubWarps) * ns * 4 + (size_t(nkids) * 2 + 15) / 16 * 16;
}

extern "C" int tpf_sparse_subtree_fpi_c128(int64_t tau, int32_t b, int32_t ns, int32_t nt, int32_t rmax, int32_t rw,
                                           int32_t nkids, const int32_t* pinfo, const int32_t* slotinfo,
                                           const uint16_t* kids, const double* coef, const int32_t* ell_col,
                                           const double* ell_val, const double* S, int64_t s_node_stride,
                                           int64_t s_case_stride, double v_flat_re, double v_flat_im, double tol,
                                           int32_t max_iter, double* V, int64_t v_node_stride, int64_t v_case_stride,
                                           int32_t* iters, double* resid, void* workspace, size_t workspace_bytes,
                                           void* stream) {
  if (tau < 0 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_sparse_subtree_fpi_c128: need tau >= 0, b >= 1");
  if (tau >= (int64_t(1) << 30)) return set_error(TPF_ERR_INVALID, "tau too large for one launch; shard it");
  if (!(tol > 0.0)) return set_error(TPF_ERR_INVALID, "tolerance must be positive");
  if (max_iter < 1) return set_error(TPF_ERR_INVALID, "max_iterations must be >= 1");
  if (tau == 0) return TPF_OK;
  if (!pinfo || !slotinfo || !kids || !coef || !ell_col || !ell_val || !S || !V || !iters || !workspace ||
      workspace_bytes < 256)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_subtree_fpi_c128: null pointer or small workspace");
  if (ns < 1 || nt < 1 || 8 * ns > 168 || rmax < 1 || rw < 1 || rw > kMaxRW || nkids < 1)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_subtree_fpi_c128: bad schedule");
  // S and V each node-major (case stride 1: the reference layout) or case-major (node stride 1)
  const bool s_nm = s_case_stride == 1 && s_node_stride >= tau, s_cm = s_node_stride == 1 && s_case_stride >= b;
  const bool v_nm = v_case_stride == 1 && v_node_stride >= tau, v_cm = v_node_stride == 1 && v_case_stride >= b;
  if (!(s_nm || s_cm) || !(v_nm || v_cm))
    return set_error(TPF_ERR_UNSUPPORTED, "tpf_sparse_subtree_fpi_c128: S / V must be node- or case-major");
  const int mode = s_cm ? 1 : 0, vmode = v_cm ? 1 : 0;
  SubArgs a;
  memset(&a, 0, sizeof a);
  a.tau = tau;
  a.b = b;
  a.NS = ns;
  a.NT = nt;
  a.NSL = ns + nt;
  a.RMAX = rmax;
  a.RW = rw;
  a.P = kSubWarps * a.NSL * 32;
  a.boxrows = b < 256 ? b : 256;
  a.nbox = (b + a.boxrows - 1) / a.boxrows;
  a.xcap = a.P > a.nbox * a.boxrows ? a.P : a.nbox * a.boxrows;
  a.nkids = nkids;
  a.mode = mode;
  a.vmode = vmode;
  a.S = reinterpret_cast<const double2*>(S);
  a.s_case = s_case_stride;
  a.V = reinterpret_cast<double2*>(V);
  a.v_case = v_case_stride;
  a.pinfo = reinterpret_cast<const int2*>(pinfo);
  a.slotinfo = slotinfo;
  a.kids = kids;
  a.coef = reinterpret_cast<const double2*>(coef);
  a.ell_col = ell_col;
  a.ell_val = reinterpret_cast<const double2*>(ell_val);
  a.iters = iters;
  a.resid = resid;
  a.counter = static_cast<unsigned long long*>(workspace);
  a.v_flat = make_double2(v_flat_re, v_flat_im);
  a.tol2 = tol * tol;
  a.max_iter = max_iter;
  const size_t smem = tpf_sparse_subtree_smem_bytes(b, ns, nt, rmax, nkids);
  if (smem > 227 * 1024) return set_error(TPF_ERR_UNSUPPORTED, "tpf_sparse_subtree_fpi_c128: schedule too large");
  CUtensorMap ms, mv;
  memset(&ms, 0, sizeof ms);
  memset(&mv, 0, sizeof mv);
  if (mode == 0) {
    const int rc = column_map(&ms, S, tau, b, s_node_stride, a.boxrows);
    if (rc != TPF_OK) return rc;
  }
  if (vmode == 0) {
    const int rc = column_map(&mv, V, tau, b, v_node_stride, a.boxrows);
    if (rc != TPF_OK) return rc;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // Node-major batches with a chunk workspace: each chunk is transposed into a
  // case-major scratch, solved there (1-D bulk copies: one 16 b-byte block per
  // case, one TLB page; a node-major column spans b rows of 16 tau bytes, one
  // 2 MB page each at C3) and transposed back.
  const int64_t chunk = tau < kSubChunk ? tau : kSubChunk;
  const size_t need = size_t(2) * size_t(chunk) * size_t(b) * 16;
  if ((mode == 0 || vmode == 0) && workspace_bytes >= 256 + need) {
    double2* Sc = reinterpret_cast<double2*>(static_cast<char*>(workspace) + 256);
    double2* Vc = Sc + size_t(chunk) * size_t(b);
    SubArgs c = a;
    c.mode = 1;
    c.vmode = 1;
    for (int64_t lo = 0; lo < tau; lo += chunk) {
      const int64_t n = tau - lo < chunk ? tau - lo : chunk;
      if (mode == 0) {
        const int rc = transpose_c128(reinterpret_cast<const double2*>(S) + lo, s_node_stride, Sc, b, b, n, st);
        if (rc != TPF_OK) return rc;
        c.S = Sc;
        c.s_case = b;
      } else {
        c.S = reinterpret_cast<const double2*>(S) + lo * s_case_stride;
      }
      if (vmode == 0) {
        c.V = Vc;
        c.v_case = b;
      } else {
        c.V = reinterpret_cast<double2*>(V) + lo * v_case_stride;
      }
      cudaError_t err = cudaMemsetAsync(workspace, 0, sizeof(unsigned long long), st);
      if (err != cudaSuccess) return set_cuda_error("cudaMemsetAsync(counter)", err);
      c.tau = n;
      c.iters = iters + lo;
      c.resid = resid ? resid + lo : nullptr;
      int rc = sub_launch(c, ms, mv, smem, int(n < sms ? n : sms), st);
      if (rc != TPF_OK) return rc;
      if (vmode == 0) {
        rc = transpose_c128(Vc, b, reinterpret_cast<double2*>(V) + lo, v_node_stride, n, b, st);
        if (rc != TPF_OK) return rc;
      }
    }
    return TPF_OK;
  }
  cudaError_t err = cudaMemsetAsync(workspace, 0, sizeof(unsigned long long), st);
  if (err != cudaSuccess) return set_cuda_error("cudaMemsetAsync(counter)", err);
  const int grid = int(tau < sms ? tau : sms);
  return sub_launch(a, ms, mv, smem, grid, st);
}
