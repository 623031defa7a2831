// Dense Tensor Power Flow, warp-specialised variant (b <= 104).
//
// Same update and semantics as tpf_dense.cu (dense.py:114-126, per-case
// freeze), reorganised so the FP64 tensor pipe of every SM sub-partition
// (SMSP) always has DMMA work queued:
//
//   * per SMSP one MMA warp and two elementwise (EW) warps, each EW warp
//     owning a group of 8 case slots (64 slots per SM);
//   * the MMA warp alternates between the two groups: while it runs the
//     complex GEMM V' = W + U K^T of group g (all 13 node blocks, M = 8
//     slots), the EW warp of the other group does everything else for its
//     slots: step test, retire/refill (continuous batching), zero-voltage
//     guard and U = S*/conj(V);
//   * hand-off through Tensor Memory of the SMSP's lane quadrant: per group
//     a 104-column buffer that holds U in DMMA A-fragment order (written by
//     the EW warp, read by the MMA warp) and then V' in C-fragment order
//     (written by the MMA warp, read by the EW warp), plus 104 columns with
//     the group's guarded iterate; S* stays in the EW warp's registers;
//   * mbarriers (32 arrivals, one per lane) order the hand-offs, with
//     tcgen05 fences around them;
//   * K^T stays in shared memory in B-fragment order (one LDS.128 per
//     fragment).
//
// Default variant (M3 = true): the complex GEMM is done with 3 real DMMAs per
// block-product (Gauss: P1 = Ur Kr, P2 = Ui Ki, P3 = (Ur+Ui)(Kr+Ki)), Kr+Ki
// staged in shared memory for the node blocks that fit, and the EW warp of a
// group computes the last node blocks of its own group's GEMM right after
// handing U over, so two DMMA streams feed each SMSP's FP64 tensor pipe.
// The EW arithmetic avoids FP64 instructions where it exactly can (every
// scalar FP64 instruction on the SMSP stalls the DMMA stream ~5-9 cycles):
// Newton reciprocal, integer-bracketed step test and zero guard.
// TPF_WS_4M=1 selects the 4-DMMA single-stream variant (bitwise equal to the
// pair/solo kernels), TPF_WS_SPLIT=2 the two-DMMA-warp 4M variant.
#include <climits>
#include <cstdlib>
#include <cstring>

#include "tpf_common.cuh"
#include "tpf_internal.h"

namespace tpf {
namespace ws {

// 12 warps: warps 0-3: MMA (SMSP w), 4-7: EW group 0, 8-11: EW group 1
// (the SPLIT=2 variant launches 16 warps: see ws_launch)
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kGroupCols = 208;  // 104 (U / V' hand-off) + 104 (guarded iterate)
// 3M variant: V' of node blocks [0, kM3Pass0) goes to a per-group scratch area
// after the two groups (columns 416 + 48 g), so the second pass can still read
// all of U from the hand-off buffer
constexpr int kM3Pass0 = 6;
constexpr uint32_t kScratchCol = 2 * kGroupCols;

struct Args {
  int64_t tau;
  int b, ks_count;
  const double* S;
  int64_t s_node, s_case;
  const double* K;
  const double* W;
  double v_flat_re, v_flat_im, tol2;
  int max_iter;
  double* V;
  int64_t v_node, v_case;
  int32_t* iters;
  unsigned long long* counter;
  // step-test bracket (3M variant): high words of |delta| bounds, see step_small
  int tol_hi_small, tol_hi_big;
  // the CTA's shared-memory image of K^T (B-fragment order), W and (3M) Kr + Ki,
  // W_re + W_im, built once per launch by ws_image_kernel and streamed into every
  // CTA by two cp.async.bulk copies: [0, stage_off) and [wsum_off, bytes)
  const unsigned char* img;
};

#ifdef TPF_PHASE_TIMING
// debug build only (tools/build_timing.sh): per-warp cycle accounting,
// [block][warp][8] = {wait U, gemm | U round, wait V', test, retire, rounds, total}
__device__ long long g_ws_cyc[148 * 12 * 8];
struct PhaseClock {
  long long c[8], t, t_start;
  __device__ __forceinline__ void start() {
    for (int i = 0; i < 8; ++i) c[i] = 0;
    t = t_start = clock64();
  }
  __device__ __forceinline__ void mark(int i) {
    const long long n = clock64();
    c[i] += n - t;
    t = n;
  }
  __device__ __forceinline__ void round() { ++c[6]; }
  __device__ __forceinline__ void flush() {
    c[7] = clock64() - t_start;
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0 && blockIdx.x < 148 && w < 12)
      for (int i = 0; i < 8; ++i) g_ws_cyc[(blockIdx.x * 12 + w) * 8 + i] = c[i];
  }
};
#else
struct PhaseClock {
  __device__ __forceinline__ void start() {}
  __device__ __forceinline__ void mark(int) {}
  __device__ __forceinline__ void round() {}
  __device__ __forceinline__ void flush() {}
};
#endif

__device__ __forceinline__ int claim(unsigned long long* counter) {
  const unsigned long long c = atomicAdd(counter, 1ull);
  return c < (unsigned long long)INT_MAX ? int(c) : INT_MAX;
}

__device__ __forceinline__ int abs_hi(double x) { return __double2hiint(x) & 0x7fffffff; }

// Step test of the 3M variant: |dr + i di|^2 < tol^2 is decided on the
// integer pipe when the high words of |dr|, |di| are clearly below 0.7 tol
// (true) or above tol (false) -- exact either way, see tpf_dense_ws_fpi_c128 --
// and by the FP64 test only for the rare values in between.  NaN/inf have the
// largest high words, so they never pass.
// v (guarded) has |v|^2 >= 1e-24 for sure when |re| or |im| >= 1.01e-12
__device__ __forceinline__ bool maybe_tiny(double x, double y) {
  return max(abs_hi(x), abs_hi(y)) <= 0x3d71c4a2;  // high word of 1.01e-12
}

struct Shared {
  uint64_t full_u[4][2];  // EW -> MMA: U of group g ready (or group finished)
  uint64_t full_v[4][2];  // MMA -> EW: V' of group g ready
  uint64_t ew_u[4][2];    // EW -> MMA (3M, NE > 0): the EW warp's share of the GEMM has read U
  int done[4][2];
  uint32_t tmem;
  uint64_t kbar;          // the K / W image has landed (bulk copy)
};

// Two k-steps (kp, kp+1) of the complex GEMM for all NB node blocks.  Per
// block the four real DMMAs run back to back (the two that accumulate onto
// the same fragment are two instructions = 32 pipe cycles apart, more than the
// ~27-cycle DMMA latency), so each K fragment is loaded once; KS is a
// template parameter so every fragment address is an immediate offset.
template <int NB, int KS>
__device__ __forceinline__ void kpair(double (&vr)[NB][2], double (&vi)[NB][2], const D4& af, const double2* kb,
                                      int kp) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int ks = kp + h;
    if (ks < KS) {
      const double ur = af.get(2 * h), ui = af.get(2 * h + 1);
      const double nui = neg_int(ui);
      const double2* k0 = kb + size_t(ks) * 32;
#pragma unroll
      for (int lb = 0; lb < NB; ++lb) {
        const double2 k = k0[size_t(lb) * KS * 32];
        dmma884(vr[lb][0], vr[lb][1], ur, k.x);
        dmma884(vi[lb][0], vi[lb][1], ur, k.y);
        dmma884(vr[lb][0], vr[lb][1], nui, k.y);
        dmma884(vi[lb][0], vi[lb][1], ui, k.x);
      }
    }
  }
}

// DMMA warp over node blocks [NB0, NB0 + NBW) of both slot groups of its SMSP.
template <int KS, int NB0, int NBW, int SPLIT>
__device__ __forceinline__ void mma_warp(const Args& a, Shared& sh, const double2* k_sm, const double* w_re,
                                         const double* w_im, int q, int lane, uint32_t tm) {
  constexpr int NB = NBW;
  uint32_t par[2] = {0u, 0u};
  bool alive[2] = {true, true};
  const int qq = lane & 3;
  for (int g = 0; alive[0] || alive[1]; g ^= 1) {
    if (!alive[g]) continue;
    mbar_wait(&sh.full_u[q][g], par[g]);
    par[g] ^= 1u;
    tmem_fence_after();
    if (sh.done[q][g]) {
      alive[g] = false;
      continue;
    }
    const uint32_t uv = tm + g * kGroupCols;
    double vr[NB][2], vi[NB][2];
#pragma unroll
    for (int lb = 0; lb < NB; ++lb) {
      const double2 wr = reinterpret_cast<const double2*>(w_re)[(8 * (NB0 + lb) + 2 * qq) / 2];
      const double2 wi = reinterpret_cast<const double2*>(w_im)[(8 * (NB0 + lb) + 2 * qq) / 2];
      vr[lb][0] = wr.x;
      vr[lb][1] = wr.y;
      vi[lb][0] = wi.x;
      vi[lb][1] = wi.y;
    }
    // A fragments (ur, ui) of two k-steps per TMEM load, ping-pong between two
    // register sets (compile-time indexed, so they stay in registers)
    D4 a0, a1;
    tmem_ld4d(uv, a0);
    tmem_wait_ld();
    const double2* kb = k_sm + size_t(NB0) * KS * 32 + lane;
#pragma unroll 1
    for (int kp = 0; kp < KS; kp += 4) {
      if (kp + 2 < KS) tmem_ld4d(uv + 4 * (kp + 2), a1);
      kpair<NB, KS>(vr, vi, a0, kb, kp);
      tmem_wait_ld();
      if (kp + 4 < KS) tmem_ld4d(uv + 4 * (kp + 4), a0);
      if (kp + 2 < KS) kpair<NB, KS>(vr, vi, a1, kb, kp + 2);
      tmem_wait_ld();
    }
    // V' in C-fragment order over the consumed U -- with two DMMA warps, only
    // once both have finished reading U (named barrier of the SMSP's pair)
    if constexpr (SPLIT == 2) named_bar(1 + q, 64);
#pragma unroll
    for (int lb = 0; lb < NB; ++lb) tmem_st4d(uv + 8 * (NB0 + lb), vr[lb][0], vr[lb][1], vi[lb][0], vi[lb][1]);
    tmem_wait_st();
    tmem_fence_before();
    mbar_arrive(&sh.full_v[q][g]);
  }
}

// 3M complex GEMM (Gauss): per node block three real accumulators
//   P1 = sum ur kr,  P2 = sum ui ki,  P3 = sum (ur + ui)(kr + ki)
//   V' = W + (P1 - P2) + i (P3 - P1 - P2)
// i.e. 3 DMMAs per block and k-step instead of 4 (6 b^2 instead of 8 b^2 real
// flops per case-iteration); kr + ki and ur + ui are formed in registers.
// One k-step (compile-time H selects the half of the A fragment D4).
template <int KS, int B0, int NBP, int NKS, int H>
__device__ __forceinline__ void kstep3(double (&p1)[NBP][2], double (&p2)[NBP][2], double (&p3)[NBP][2], const D4& af,
                                       const double2* kb, const double* ksb, int ks) {
  const double ur = af.get(2 * H), ui = af.get(2 * H + 1);
  const double us = ur + ui;
  const double2* k0 = kb + size_t(ks) * 32;
#pragma unroll
  for (int lb = 0; lb < NBP; ++lb) {
    const double2 k = k0[size_t(B0 + lb) * KS * 32];
    // kr + ki: precomputed in shared memory for the first NKS blocks
    const double kss = (B0 + lb < NKS) ? ksb[(size_t(B0 + lb) * KS + ks) * 32] : k.x + k.y;
    dmma884(p1[lb][0], p1[lb][1], ur, k.x);
    dmma884(p2[lb][0], p2[lb][1], ui, k.y);
    dmma884(p3[lb][0], p3[lb][1], us, kss);
  }
}

// Shared-memory layout of the kernel: K^T fragments (kr, ki) [NB][KS][32],
// W re / im [NB*8] each, EW staging [8][64], Shared; the 3M variant adds
// W re + im [NB*8] and, for as many node blocks as fit, kr + ki [NKS][KS][32].
template <int NB, int KS, bool M3>
struct Layout {
  static constexpr size_t k_bytes = size_t(NB) * KS * 32 * 16;
  static constexpr size_t w_off = k_bytes;
  static constexpr size_t stage_off = w_off + size_t(NB) * 8 * 16;
  static constexpr size_t shared_off = stage_off + 8 * 64 * 16;
  static constexpr size_t wsum_off = shared_off + 256;
  static constexpr size_t ks_off = wsum_off + (M3 ? size_t(NB) * 8 * 8 : 0);
  static constexpr size_t cap = 232448;  // 227 KB opt-in maximum per block
  static constexpr size_t plane = size_t(KS) * 32 * 8;
  static constexpr int fit = int((cap - ks_off) / plane);
  static constexpr int NKS = !M3 ? 0 : (fit < NB ? fit : NB);
  static constexpr size_t bytes = ks_off + size_t(NKS) * plane;
};

// One pass over all k-steps for node blocks [B0, B0 + NBP); returns V' of
// those blocks in C-fragment order (v[lb] = re0, re1, im0, im1).  The
// accumulators start at P1 = Re W, P2 = 0, P3 = Re W + Im W, so
// V' = (P1 - P2) + i ((P3 - P1) - P2).
template <int KS, int B0, int NBP, int NKS>
__device__ __forceinline__ void pass3(uint32_t uv, double (&v)[NBP][4], const double2* kb, const double* ksb,
                                      const double* w_re, const double* w_sum, int qq) {
  double p1[NBP][2], p2[NBP][2], p3[NBP][2];
#pragma unroll
  for (int lb = 0; lb < NBP; ++lb) {
    const double2 wr = reinterpret_cast<const double2*>(w_re)[(8 * (B0 + lb) + 2 * qq) / 2];
    const double2 ws = reinterpret_cast<const double2*>(w_sum)[(8 * (B0 + lb) + 2 * qq) / 2];
    p1[lb][0] = wr.x;
    p1[lb][1] = wr.y;
    p2[lb][0] = p2[lb][1] = 0.0;
    p3[lb][0] = ws.x;
    p3[lb][1] = ws.y;
  }
  // k-steps in groups of 4 (two TMEM A-fragment loads, ping-pong) with no
  // run-time conditions in the loop; the KS % 4 tail is unrolled at compile time
  D4 a0, a1;
  tmem_ld4d(uv, a0);
  tmem_wait_ld();
  constexpr int KM = KS / 4 * 4;
#pragma unroll 1
  for (int kp = 0; kp < KM; kp += 4) {
    tmem_ld4d(uv + 4 * (kp + 2), a1);
    kstep3<KS, B0, NBP, NKS, 0>(p1, p2, p3, a0, kb, ksb, kp);
    kstep3<KS, B0, NBP, NKS, 1>(p1, p2, p3, a0, kb, ksb, kp + 1);
    tmem_wait_ld();
    if (kp + 4 < KS) tmem_ld4d(uv + 4 * (kp + 4), a0);  // uniform; false only on the last pass
    kstep3<KS, B0, NBP, NKS, 0>(p1, p2, p3, a1, kb, ksb, kp + 2);
    kstep3<KS, B0, NBP, NKS, 1>(p1, p2, p3, a1, kb, ksb, kp + 3);
    tmem_wait_ld();
  }
  if constexpr (KS - KM >= 1) kstep3<KS, B0, NBP, NKS, 0>(p1, p2, p3, a0, kb, ksb, KM);
  if constexpr (KS - KM >= 2) kstep3<KS, B0, NBP, NKS, 1>(p1, p2, p3, a0, kb, ksb, KM + 1);
  if constexpr (KS - KM >= 3) {
    tmem_ld4d(uv + 4 * (KM + 2), a1);
    tmem_wait_ld();
    kstep3<KS, B0, NBP, NKS, 0>(p1, p2, p3, a1, kb, ksb, KM + 2);
  }
#pragma unroll
  for (int lb = 0; lb < NBP; ++lb) {
    v[lb][0] = p1[lb][0] - p2[lb][0];
    v[lb][1] = p1[lb][1] - p2[lb][1];
    v[lb][2] = (p3[lb][0] - p1[lb][0]) - p2[lb][0];
    v[lb][3] = (p3[lb][1] - p1[lb][1]) - p2[lb][1];
  }
}

template <int NBP>
__device__ __forceinline__ void store3(uint32_t dst, const double (&v)[NBP][4]) {
#pragma unroll
  for (int lb = 0; lb < NBP; ++lb) tmem_st4d(dst + 8 * lb, v[lb][0], v[lb][1], v[lb][2], v[lb][3]);
}

// The 3M GEMM of a group is shared: the MMA warp does node blocks [0, NM),
// the group's EW warp the last NE = NB - NM blocks (it is otherwise idle while
// the MMA warp works), so two DMMA streams feed the SMSP's tensor pipe.
// V' of blocks [0, kM3Pass0) goes to the group's scratch columns; every other
// block's V' overwrites U in the hand-off buffer, so it is stored only once
// both warps are done reading U (mbarriers ew_u and full_v).
// 3M DMMA warp (one per SMSP, both groups), node blocks [0, NM).
template <int NB, int KS, int NKS, int NM>
__device__ __forceinline__ void mma_warp3(const Args& a, Shared& sh, const double2* k_sm, const double* ks_sm,
                                          const double* w_re, const double* w_sum, int q, int lane, uint32_t tm) {
  constexpr int NE = NB - NM;
  constexpr int P0 = NM < kM3Pass0 ? NM : kM3Pass0;  // blocks of the first pass (to scratch)
  static_assert(NE == 0 || NM >= kM3Pass0 || NB <= kM3Pass0, "EW blocks must lie past the scratch blocks");
  uint32_t par[2] = {0u, 0u}, epar[2] = {0u, 0u};
  bool alive[2] = {true, true};
  const int qq = lane & 3;
  const double2* kb = k_sm + lane;
  const double* ksb = ks_sm + lane;
  PhaseClock pc;
  pc.start();
  for (int g = 0; alive[0] || alive[1]; g ^= 1) {
    if (!alive[g]) continue;
    pc.mark(5);
    mbar_wait(&sh.full_u[q][g], par[g]);
    par[g] ^= 1u;
    tmem_fence_after();
    pc.mark(0);
    if (sh.done[q][g]) {
      alive[g] = false;
      continue;
    }
    pc.round();
    const uint32_t uv = tm + g * kGroupCols;
    if constexpr (NB <= kM3Pass0) {  // everything fits the scratch-free single pass
      double v[NB][4];
      pass3<KS, 0, NB, NKS>(uv, v, kb, ksb, w_re, w_sum, qq);
      store3<NB>(uv, v);
    } else {
      {
        double v[P0][4];
        pass3<KS, 0, P0, NKS>(uv, v, kb, ksb, w_re, w_sum, qq);
        store3<P0>(tm + kScratchCol + g * 8 * kM3Pass0, v);
      }
      if constexpr (NM > P0) {
        double v[NM - P0][4];
        pass3<KS, P0, NM - P0, NKS>(uv, v, kb, ksb, w_re, w_sum, qq);
        if constexpr (NE > 0) {  // the EW warp may still be reading U
          mbar_wait(&sh.ew_u[q][g], epar[g]);
          epar[g] ^= 1u;
          tmem_fence_after();
        }
        store3<NM - P0>(uv + 8 * P0, v);
      }
    }
    tmem_wait_st();
    tmem_fence_before();
    mbar_arrive(&sh.full_v[q][g]);
    pc.mark(1);
  }
  pc.flush();
}

template <int NB, int KS, bool M3, int NKS, int NM>
__device__ __forceinline__ void ew_warp(const Args& a, Shared& sh, double2* stage, int q, int g, int lane,
                                        uint32_t tm, const double2* k_sm, const double* ks_sm, const double* w_re,
                                        const double* w_sum) {
  constexpr int NE = NB - NM;
  const int slot = lane >> 2, qq = lane & 3;
  const int b = a.b;
  const int64_t tau = a.tau;
  const uint32_t uv = tm + g * kGroupCols, vc = uv + 104;
  // where the MMA warp left V' of node block lb
  const uint32_t scr = tm + kScratchCol + g * 8 * kM3Pass0;
  auto vp = [&](int lb) -> uint32_t {
    return (M3 && NB > kM3Pass0 && lb < kM3Pass0) ? scr + 8 * lb : uv + 8 * lb;
  };
  int cid = INT_MAX, nxt = INT_MAX, n_it = 0;
  bool fresh = true;  // this lane's slot starts from the flat voltage next round
  uint32_t par = 0u;

  auto prefetch = [&](int c) {
    if (c >= tau) return;
#pragma unroll
    for (int lb = 0; lb < NB; ++lb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int node = 8 * lb + 2 * qq + e;
        if (node < b) {
          const double* p = a.S + 2 * (node * a.s_node + int64_t(c) * a.s_case);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
        }
      }
  };
  // the quad's first lane claims a case for its slot if `want`; the quad shares it
  auto claim_slot = [&](bool want) {
    int c = INT_MAX;
    if (qq == 0 && want) c = claim(a.counter);
    return __shfl_sync(0xffffffffu, c, lane & ~3);
  };

  cid = claim_slot(true);
  nxt = claim_slot(true);
  if (cid >= tau) cid = INT_MAX;
  prefetch(cid);
  prefetch(nxt);
  PhaseClock pc;
  pc.start();

  for (;;) {
    pc.round();
    // ---- guard, keep the iterate (TMEM), U = S*/conj(v) in A-fragment order ----
    // S of the slot's case is re-read every round (the 64 slots x 148 SMs x 1.6 KB
    // working set stays in L2), two node blocks ahead of its use so the L2
    // latency overlaps the previous blocks' arithmetic.
    auto load_s = [&](double2 (&dst)[2], int lb) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int node = 8 * lb + 2 * qq + e;
        dst[e] = (lb < NB && cid < tau && node < b) ? ldg_c128(a.S, node * a.s_node + int64_t(cid) * a.s_case)
                                                    : make_double2(0.0, 0.0);
      }
    };
    double2 sq[3][2];
    load_s(sq[0], 0);
    load_s(sq[1], 1);
#pragma unroll
    for (int lb = 0; lb < NB; ++lb) {
      load_s(sq[(lb + 2) % 3], lb + 2);
      const double2* sv = sq[lb % 3];
      D4 nv;
      tmem_ld4d(vp(lb), nv);  // V' of the last GEMM (ignored by fresh slots)
      tmem_wait_ld();
      double xr[2], xi[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        xr[e] = fresh ? a.v_flat_re : nv.get(e);
        xi[e] = fresh ? a.v_flat_im : nv.get(2 + e);
        double m2 = __fma_rn(xr[e], xr[e], xi[e] * xi[e]);
        double r;
        if constexpr (M3) {
          if (maybe_tiny(xr[e], xi[e]) && m2 < kZeroGuard2) {  // fpi.py:39-41
            xr[e] = kZeroGuard;
            xi[e] = 0.0;
            m2 = kZeroGuard * kZeroGuard;
          }
          r = rcp_nr(m2);
        } else {
          if (m2 < kZeroGuard2) {  // fpi.py:39-41
            xr[e] = kZeroGuard;
            xi[e] = 0.0;
            m2 = kZeroGuard * kZeroGuard;
          }
          r = 1.0 / m2;
        }
        const double sr = sv[e].x, si = -sv[e].y;  // S* (dense.py:154)
        const double ur = __fma_rn(sr, xr[e], -(si * xi[e])) * r;
        const double ui = __fma_rn(sr, xi[e], si * xr[e]) * r;
        stage[slot * 8 + 2 * qq + e] = make_double2(ur, ui);  // C layout -> staging
      }
      tmem_st4d(vc + 8 * lb, xr[0], xr[1], xi[0], xi[1]);
      __syncwarp();
      // A layout: k-steps 2lb (nodes 8lb+qq) and 2lb+1 (nodes 8lb+4+qq)
      const double2 u0 = stage[slot * 8 + qq];
      const double2 u1 = stage[slot * 8 + 4 + qq];
      __syncwarp();
      if (2 * lb < KS) tmem_st4d(uv + 8 * lb, u0.x, u0.y, u1.x, u1.y);
    }
    tmem_wait_st();
    tmem_fence_before();
    mbar_arrive(&sh.full_u[q][g]);
    fresh = false;
    pc.mark(2);

    if constexpr (M3 && NE > 0) {
      // this warp's share of the group's GEMM: node blocks [NM, NB)
      double v[NE > 0 ? NE : 1][4];
      pass3<KS, NM, NE, NKS>(uv, v, k_sm + lane, ks_sm + lane, w_re, w_sum, qq);
      pc.mark(1);  // (timing build) the EW warp's GEMM share
      tmem_fence_before();
      mbar_arrive(&sh.ew_u[q][g]);  // done reading U
      mbar_wait(&sh.full_v[q][g], par);
      par ^= 1u;
      tmem_fence_after();
      store3<NE>(uv + 8 * NM, v);
      tmem_wait_st();
    } else {
      // ---- wait for V' of this group ----
      mbar_wait(&sh.full_v[q][g], par);
      par ^= 1u;
      tmem_fence_after();
    }
    pc.mark(3);
    // ---- per-case step test (dense.py:125-126, 189-193) ----
    bool small = true;
#pragma unroll
    for (int lb = 0; lb < NB; ++lb) {
      D4 nv, ov;
      tmem_ld4d(vp(lb), nv);
      tmem_ld4d(vc + 8 * lb, ov);
      tmem_wait_ld();
      if constexpr (M3) {
        double dr[2], di[2];
        bool ok[2], unsure[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          dr[e] = nv.get(e) - ov.get(e);
          di[e] = nv.get(2 + e) - ov.get(2 + e);
          const int m = max(abs_hi(dr[e]), abs_hi(di[e]));
          const bool pad = 8 * lb + 2 * qq + e >= b;
          ok[e] = pad || m < a.tol_hi_small;
          unsure[e] = !ok[e] && m <= a.tol_hi_big;
        }
        if (__any_sync(0xffffffffu, unsure[0] || unsure[1])) {  // rare: |delta| within [0.7 tol, tol]
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (unsure[e]) ok[e] = __fma_rn(dr[e], dr[e], di[e] * di[e]) < a.tol2;
        }
        small = small && ok[0] && ok[1];
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double dr = nv.get(e) - ov.get(e), di = nv.get(2 + e) - ov.get(2 + e);
          const int node = 8 * lb + 2 * qq + e;
          if (node < b && !(__fma_rn(dr, dr, di * di) < a.tol2)) small = false;  // NaN never passes
        }
      }
    }
    const uint32_t ball = __ballot_sync(0xffffffffu, small);
    const bool my_small = ((ball >> (slot * 4)) & 0xFu) == 0xFu;
    bool done = false;
    if (cid != INT_MAX) {
      ++n_it;
      done = my_small || n_it >= a.max_iter;
    }
    pc.mark(4);
    if (__any_sync(0xffffffffu, done)) {
      // retire: V' of the retiring slots to global memory, per-case count
#pragma unroll
      for (int lb = 0; lb < NB; ++lb) {
        D4 nv;
        tmem_ld4d(vp(lb), nv);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int node = 8 * lb + 2 * qq + e;
          if (done && node < b) {
            double* p = a.V + 2 * (node * a.v_node + int64_t(cid) * a.v_case);
            p[0] = nv.get(e);
            p[1] = nv.get(2 + e);
          }
        }
      }
      if (done && qq == 0) a.iters[cid] = n_it;
      // refill from the case claimed one refill ahead; claim the one after it
      const int fresh_id = claim_slot(done);
      if (done) {
        cid = nxt < tau ? nxt : INT_MAX;
        nxt = fresh_id;
        n_it = 0;
        fresh = true;
        prefetch(nxt);
      }
    }
    pc.mark(5);
    if (__all_sync(0xffffffffu, cid == INT_MAX)) {
      if (lane == 0) sh.done[q][g] = 1;
      __syncwarp();
      tmem_fence_before();
      mbar_arrive(&sh.full_u[q][g]);
      break;
    }
  }
  pc.flush();
}

// SPLIT DMMA warps per SMSP share each GEMM (node blocks split NBA / NB - NBA):
// SPLIT = 1: 12 warps (4 DMMA + 8 EW); SPLIT = 2: 16 warps (8 DMMA + 8 EW), so
// two DMMA streams feed every FP64 tensor pipe.
template <int NB, int KS, int SPLIT, bool M3, int NM>
__global__ void __launch_bounds__(32 * (8 + 4 * SPLIT), 1) dense_ws_kernel(const Args a) {
  constexpr int NBA = SPLIT == 1 ? NB : (NB + 1) / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using L = Layout<NB, KS, M3>;
  const int b = a.b;
  double2* k_sm = reinterpret_cast<double2*>(smem_raw);                 // [NB][KS][32]
  double* w_re = reinterpret_cast<double*>(smem_raw + L::w_off);        // [NB*8]
  double* w_im = w_re + NB * 8;
  double2* stage = reinterpret_cast<double2*>(smem_raw + L::stage_off);  // [8 EW warps][64]
  Shared& sh = *reinterpret_cast<Shared*>(smem_raw + L::shared_off);
  double* w_sum = reinterpret_cast<double*>(smem_raw + L::wsum_off);     // [NB*8] (3M)
  double* ks_sm = reinterpret_cast<double*>(smem_raw + L::ks_off);       // [NKS][KS][32] (3M)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  constexpr int kT = 32 * (8 + 4 * SPLIT);
  if (!a.img) {  // A/B (TPF_WS_GATHER=1): every CTA gathers K^T / W from global itself
    for (int idx = tid; idx < NB * KS * 32; idx += kT) {
      const int l = idx & 31, ks = (idx >> 5) % KS, nb = (idx >> 5) / KS;
      const int row = 8 * nb + (l >> 2), col = 4 * ks + (l & 3);
      const double2 k = (row < b && col < b) ? ldg_c128(a.K, int64_t(row) * b + col) : make_double2(0.0, 0.0);
      k_sm[idx] = k;
      if (M3 && nb < L::NKS) ks_sm[idx] = k.x + k.y;
    }
    for (int i = tid; i < NB * 8; i += kT) {
      const double2 w = (i < b) ? ldg_c128(a.W, i) : make_double2(0.0, 0.0);
      w_re[i] = w.x;
      w_im[i] = w.y;
      if (M3) w_sum[i] = w.x + w.y;
    }
  }
  if (tid == 0) {
    for (int q = 0; q < 4; ++q)
      for (int g = 0; g < 2; ++g) {
        mbar_init(&sh.full_u[q][g], 32);
        mbar_init(&sh.full_v[q][g], 32 * SPLIT);
        mbar_init(&sh.ew_u[q][g], 32);
        sh.done[q][g] = 0;
      }
    mbar_init(&sh.kbar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the async proxy sees the initialised barrier
    if (a.img) {
      // K^T, W (and the 3M sums) arrive as two bulk copies of the launch's image (TMA engine)
      constexpr uint32_t bytes_a = uint32_t(L::stage_off), bytes_b = uint32_t(L::bytes - L::wsum_off);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&sh.kbar)),
                   "r"(bytes_a + bytes_b)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(smem_raw)),
                   "l"(a.img), "r"(bytes_a), "r"(smem_u32(&sh.kbar))
                   : "memory");
      if (bytes_b)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(smem_raw + L::wsum_off)),
            "l"(a.img + L::wsum_off), "r"(bytes_b), "r"(smem_u32(&sh.kbar))
            : "memory");
    }
  }
  __syncthreads();
  if (a.img) mbar_wait(&sh.kbar, 0);
  if (warp == 0) tmem_alloc(&sh.tmem, kTmemCols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const int q = warp & 3;
  const uint32_t tm = sh.tmem + (uint32_t(32 * q) << 16);
  const int wg = warp >> 2;
  if (wg == 0) {
    if constexpr (M3)
      mma_warp3<NB, KS, L::NKS, NM>(a, sh, k_sm, ks_sm, w_re, w_sum, q, lane, tm);
    else
      mma_warp<KS, 0, NBA, SPLIT>(a, sh, k_sm, w_re, w_im, q, lane, tm);
  } else if (SPLIT == 2 && wg == 1) {
    if constexpr (SPLIT == 2) mma_warp<KS, NBA, NB - NBA, SPLIT>(a, sh, k_sm, w_re, w_im, q, lane, tm);
  } else {
    const int e = warp - 4 * SPLIT;  // 0..7
    ew_warp<NB, KS, M3, L::NKS, NM>(a, sh, stage + e * 64, q, e >> 2, lane, tm, k_sm, ks_sm, w_re, w_sum);
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(sh.tmem, kTmemCols);
}

// The launch's shared-memory image of K^T in DMMA B-fragment order (conflict-free
// LDS.128 per fragment), W, and for the 3M GEMM Kr + Ki of the first NKS node
// blocks and W_re + W_im (the same DADDs the GEMM would do): what every CTA's
// prologue used to gather from K and W element by element, built once.
template <int NB, int KS, bool M3>
__global__ void __launch_bounds__(256) ws_image_kernel(const double* __restrict__ K, const double* __restrict__ W,
                                                       int b, unsigned char* img) {
  using L = Layout<NB, KS, M3>;
  double2* k_sm = reinterpret_cast<double2*>(img);
  double* w_re = reinterpret_cast<double*>(img + L::w_off);
  double* w_im = w_re + NB * 8;
  double* w_sum = reinterpret_cast<double*>(img + L::wsum_off);
  double* ks_sm = reinterpret_cast<double*>(img + L::ks_off);
  const int stride = gridDim.x * blockDim.x;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < NB * KS * 32; idx += stride) {
    const int l = idx & 31, ks = (idx >> 5) % KS, nb = (idx >> 5) / KS;
    const int row = 8 * nb + (l >> 2), col = 4 * ks + (l & 3);
    const double2 k = (row < b && col < b) ? ldg_c128(K, int64_t(row) * b + col) : make_double2(0.0, 0.0);
    k_sm[idx] = k;
    if (M3 && nb < L::NKS) ks_sm[idx] = k.x + k.y;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < NB * 8; i += stride) {
    const double2 w = (i < b) ? ldg_c128(W, i) : make_double2(0.0, 0.0);
    w_re[i] = w.x;
    w_im[i] = w.y;
    if (M3) w_sum[i] = w.x + w.y;
  }
}

template <int NB, int KS, int SPLIT, bool M3, int NM = NB>
int launch(const Args& a_in, cudaStream_t st, int sms) {
  static_assert(sizeof(Shared) <= 256, "Shared must fit its 256-byte slot");
  const size_t smem = Layout<NB, KS, M3>::bytes;
  Args a = a_in;
  // the image lives in the workspace after the 256-byte counter slot
  static const bool gather = [] {  // A/B: TPF_WS_GATHER=1 gathers K per CTA instead
    const char* e = getenv("TPF_WS_GATHER");
    return e && e[0] == '1';
  }();
  static const bool img_only = [] {  // A/B: TPF_WS_GATHER=2 builds the image but gathers per CTA
    const char* e = getenv("TPF_WS_GATHER");
    return e && e[0] == '2';
  }();
  unsigned char* img = static_cast<unsigned char*>(static_cast<void*>(a.counter)) + 256;
  a.img = nullptr;
  if (!gather) {
    ws_image_kernel<NB, KS, M3><<<16, 256, 0, st>>>(a.K, a.W, a.b, img);
    cudaError_t e0 = cudaGetLastError();
    if (e0 != cudaSuccess) return set_cuda_error("launch(ws_image_kernel)", e0);
    if (!img_only) a.img = img;
  }
  cudaError_t err = cudaFuncSetAttribute(dense_ws_kernel<NB, KS, SPLIT, M3, NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (err != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(dense_ws)", err);
  int64_t grid = sms;
  const int64_t need = (a.tau + 63) / 64;  // 64 slots per CTA
  if (need < grid) grid = need;
  if (grid < 1) grid = 1;
  dense_ws_kernel<NB, KS, SPLIT, M3, NM><<<unsigned(grid), 32 * (8 + 4 * SPLIT), smem, st>>>(a);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(dense_ws_kernel)", err);
  return TPF_OK;
}

}  // namespace ws

#ifdef TPF_AB_VARIANTS  // A/B-only kernels (tools/build_timing.sh -DTPF_AB_VARIANTS); not in libtpf.so
// ---------------------------------------------------------------------------
// "Solo" variant: 8 independent warps per SM, each owning 8 case slots and all
// node blocks, each doing its own GEMM and elementwise work.  Two DMMA
// streams per SM sub-partition (one warp issuing DMMAs cannot fill the FP64
// tensor pipe: ~20 cycles per DMMA instead of 16 with one LDS per 4 DMMAs);
// while one warp is in its elementwise phase the other keeps the pipe busy.
// Per warp in its TMEM lane quadrant: U in A-fragment order (100 columns) and
// the guarded iterate (104 columns); S is re-read from L2 each round.  No
// inter-warp synchronisation at all after the prologue.
namespace solo {

constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;

template <int NB, int KS>
__global__ void __launch_bounds__(kThreads, 1) dense_solo_kernel(const ws::Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = a.b;
  const int64_t tau = a.tau;
  double2* k_sm = reinterpret_cast<double2*>(smem_raw);                 // [NB][KS][32]
  double* w_re = reinterpret_cast<double*>(k_sm + size_t(NB) * KS * 32);  // [NB*8]
  double* w_im = w_re + NB * 8;
  double2* stage_all = reinterpret_cast<double2*>(w_im + NB * 8);       // [8 warps][64]
  uint32_t* tmem_sm = reinterpret_cast<uint32_t*>(stage_all + kWarps * 64);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot = lane >> 2, qq = lane & 3;

  for (int idx = tid; idx < NB * KS * 32; idx += kThreads) {
    const int l = idx & 31, ks = (idx >> 5) % KS, nb = (idx >> 5) / KS;
    const int row = 8 * nb + (l >> 2), col = 4 * ks + (l & 3);
    k_sm[idx] = (row < b && col < b) ? ldg_c128(a.K, int64_t(row) * b + col) : make_double2(0.0, 0.0);
  }
  for (int i = tid; i < NB * 8; i += kThreads) {
    const double2 w = (i < b) ? ldg_c128(a.W, i) : make_double2(0.0, 0.0);
    w_re[i] = w.x;
    w_im[i] = w.y;
  }
  if (warp == 0) tmem_alloc(tmem_sm, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tm = *tmem_sm + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * 256);
  const uint32_t uv = tm, vc = tm + 104;  // U (A order, 100 cols) | guarded iterate (C order, 104 cols)
  double2* stage = stage_all + warp * 64;
  const double2* kb = k_sm + lane;

  auto claim_slot = [&](bool want) {
    int c = INT_MAX;
    if (qq == 0 && want) c = ws::claim(a.counter);
    return __shfl_sync(0xffffffffu, c, lane & ~3);
  };
  auto prefetch = [&](int c) {
    if (c >= tau) return;
#pragma unroll
    for (int lb = 0; lb < NB; ++lb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int node = 8 * lb + 2 * qq + e;
        if (node < b) {
          const double* p = a.S + 2 * (node * a.s_node + int64_t(c) * a.s_case);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
        }
      }
  };

  int cid = claim_slot(true);
  int nxt = claim_slot(true);
  if (cid >= tau) cid = INT_MAX;
  prefetch(cid);
  prefetch(nxt);
  int n_it = 0;

  double vr[NB][2], vi[NB][2];  // the iterate entering the next U (flat start)
#pragma unroll
  for (int lb = 0; lb < NB; ++lb)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      vr[lb][e] = a.v_flat_re;
      vi[lb][e] = a.v_flat_im;
    }

  for (;;) {
    // ---- guard, keep the iterate (TMEM), U = S*/conj(v) in A-fragment order (TMEM) ----
#pragma unroll
    for (int lb = 0; lb < NB; ++lb) {
      double xr[2], xi[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int node = 8 * lb + 2 * qq + e;
        const double2 sv = (cid < tau && node < b) ? ldg_c128(a.S, node * a.s_node + int64_t(cid) * a.s_case)
                                                   : make_double2(0.0, 0.0);
        xr[e] = vr[lb][e];
        xi[e] = vi[lb][e];
        double m2 = __fma_rn(xr[e], xr[e], xi[e] * xi[e]);
        if (m2 < kZeroGuard2) {  // fpi.py:39-41
          xr[e] = kZeroGuard;
          xi[e] = 0.0;
          m2 = kZeroGuard * kZeroGuard;
        }
        const double r = 1.0 / m2;
        const double sr = sv.x, si = -sv.y;  // S* (dense.py:154)
        stage[slot * 8 + 2 * qq + e] =
            make_double2(__fma_rn(sr, xr[e], -(si * xi[e])) * r, __fma_rn(sr, xi[e], si * xr[e]) * r);
      }
      tmem_st4d(vc + 8 * lb, xr[0], xr[1], xi[0], xi[1]);
      __syncwarp();
      const double2 u0 = stage[slot * 8 + qq];
      const double2 u1 = stage[slot * 8 + 4 + qq];
      __syncwarp();
      if (2 * lb < KS) tmem_st4d(uv + 8 * lb, u0.x, u0.y, u1.x, u1.y);
    }
    tmem_wait_st();

    // ---- GEMM: V' = W + U K^T ----
#pragma unroll
    for (int lb = 0; lb < NB; ++lb) {
      const double2 wr = reinterpret_cast<const double2*>(w_re)[(8 * lb + 2 * qq) / 2];
      const double2 wi = reinterpret_cast<const double2*>(w_im)[(8 * lb + 2 * qq) / 2];
      vr[lb][0] = wr.x;
      vr[lb][1] = wr.y;
      vi[lb][0] = wi.x;
      vi[lb][1] = wi.y;
    }
    {
      D4 a0, a1;
      tmem_ld4d(uv, a0);
      tmem_wait_ld();
#pragma unroll 1
      for (int kp = 0; kp < KS; kp += 4) {
        if (kp + 2 < KS) tmem_ld4d(uv + 4 * (kp + 2), a1);
        ws::kpair<NB, KS>(vr, vi, a0, kb, kp);
        tmem_wait_ld();
        if (kp + 4 < KS) tmem_ld4d(uv + 4 * (kp + 4), a0);
        if (kp + 2 < KS) ws::kpair<NB, KS>(vr, vi, a1, kb, kp + 2);
        tmem_wait_ld();
      }
    }

    // ---- per-case step test (dense.py:125-126, 189-193) ----
    bool small = true;
#pragma unroll
    for (int lb = 0; lb < NB; ++lb) {
      D4 ov;
      tmem_ld4d(vc + 8 * lb, ov);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double dr = vr[lb][e] - ov.get(e), di = vi[lb][e] - ov.get(2 + e);
        const int node = 8 * lb + 2 * qq + e;
        if (node < b && !(__fma_rn(dr, dr, di * di) < a.tol2)) small = false;  // NaN never passes
      }
    }
    const uint32_t ball = __ballot_sync(0xffffffffu, small);
    const bool my_small = ((ball >> (slot * 4)) & 0xFu) == 0xFu;
    bool done = false;
    if (cid != INT_MAX) {
      ++n_it;
      done = my_small || n_it >= a.max_iter;
    }
    if (__any_sync(0xffffffffu, done)) {
      if (done) {
#pragma unroll
        for (int lb = 0; lb < NB; ++lb)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int node = 8 * lb + 2 * qq + e;
            if (node < b) {
              double* p = a.V + 2 * (node * a.v_node + int64_t(cid) * a.v_case);
              p[0] = vr[lb][e];
              p[1] = vi[lb][e];
            }
          }
        if (qq == 0) a.iters[cid] = n_it;
      }
      const int fresh_id = claim_slot(done);
      if (done) {
        cid = nxt < tau ? nxt : INT_MAX;
        nxt = fresh_id;
        n_it = 0;
        prefetch(nxt);
#pragma unroll
        for (int lb = 0; lb < NB; ++lb)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            vr[lb][e] = a.v_flat_re;
            vi[lb][e] = a.v_flat_im;
          }
      }
    }
    if (__all_sync(0xffffffffu, cid == INT_MAX)) break;
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(*tmem_sm, 512);
}

template <int NB, int KS>
int launch(const ws::Args& a, cudaStream_t st, int sms) {
  const size_t smem = size_t(NB) * KS * 32 * 16 + size_t(NB) * 8 * 16 + kWarps * 64 * 16 + 64;
  cudaError_t err = cudaFuncSetAttribute(dense_solo_kernel<NB, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
  if (err != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(dense_solo)", err);
  int64_t grid = sms;
  const int64_t need = (a.tau + 63) / 64;
  if (need < grid) grid = need;
  if (grid < 1) grid = 1;
  dense_solo_kernel<NB, KS><<<unsigned(grid), kThreads, smem, st>>>(a);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(dense_solo_kernel)", err);
  return TPF_OK;
}

}  // namespace solo
#endif  // TPF_AB_VARIANTS
}  // namespace tpf

using namespace tpf;

static int hi_word(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return int(u >> 32) & 0x7fffffff;
}

#ifdef TPF_PHASE_TIMING
extern "C" int tpf_debug_ws_phase_cycles(long long* out) {
  return cudaMemcpyFromSymbol(out, ws::g_ws_cyc, sizeof(ws::g_ws_cyc)) == cudaSuccess ? 0 : 1;
}
#endif

// Variants (chosen once per process): default 3M GEMM with the EW warps taking
// TPF_WS_NE node blocks (C2: 6.25 ms).  In A/B builds only (-DTPF_AB_VARIANTS,
// not libtpf.so): TPF_WS_4M=1 the 4-DMMA GEMM on one DMMA warp per SMSP
// (7.43 ms) and TPF_WS_SPLIT=2 two 4M DMMA warps per SMSP (8.17 ms: the EW
// warps cannot refill U fast enough).
template <int NB, int KS>
static int ws_launch(const ws::Args& a, cudaStream_t st, int sms) {
#ifdef TPF_AB_VARIANTS  // A/B builds only: the 4M and two-DMMA-warp variants
  static const int split = [] {
    const char* e = getenv("TPF_WS_SPLIT");
    return (e && e[0] == '2') ? 2 : 1;
  }();
  static const bool four = [] {
    const char* e = getenv("TPF_WS_4M");
    return e && e[0] == '1';
  }();
  if constexpr (NB >= 2) {
    if (split == 2) return ws::launch<NB, KS, 2, false>(a, st, sms);
  }
  if (four) return ws::launch<NB, KS, 1, false>(a, st, sms);
#endif
  // node blocks of the GEMM done by the elementwise warps: 5 at 13 node blocks
  // (tuned on C2: NE 2..7 measured 6.69 / 6.56 / 6.34 / 6.31 / 6.58 / 6.63 ms),
  // otherwise min(4, blocks - 6) so the EW blocks lie past the 6 scratch
  // blocks; TPF_WS_NE=0 disables the EW share, any other value keeps the
  // generic min(4, blocks - 6)
  static const int ne = [] {
    const char* e = getenv("TPF_WS_NE");
    return e ? atoi(e) : 5;
  }();
  if constexpr (NB == 13) {
    if (ne == 5) return ws::launch<NB, KS, 1, true, NB - 5>(a, st, sms);
  }
  if constexpr (NB > ws::kM3Pass0) {
    // the EW blocks must lie past the scratch blocks: NM >= kM3Pass0
    constexpr int nm = NB - 4 >= ws::kM3Pass0 ? NB - 4 : ws::kM3Pass0;
    if (ne != 0) return ws::launch<NB, KS, 1, true, nm>(a, st, sms);
  }
  return ws::launch<NB, KS, 1, true>(a, st, sms);
}

extern "C" int tpf_dense_ws_fpi_c128(int64_t tau, int32_t b, const double* S, int64_t s_node_stride,
                                     int64_t s_case_stride, const double* K, const double* W, double v_flat_re,
                                     double v_flat_im, double tol, int32_t max_iter, double* V, int64_t v_node_stride,
                                     int64_t v_case_stride, int32_t* iters, void* workspace, size_t workspace_bytes,
                                     void* stream) {
  if (tau < 0 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_dense_ws_fpi_c128: need tau >= 0 and b >= 1");
  if (b > 104) return set_error(TPF_ERR_UNSUPPORTED, "tpf_dense_ws_fpi_c128: b > 104");
  if (tau > INT_MAX - 4096) return set_error(TPF_ERR_INVALID, "tau too large for one launch; shard it");
  if (!(tol > 0.0)) return set_error(TPF_ERR_INVALID, "tolerance must be positive");
  if (max_iter < 1) return set_error(TPF_ERR_INVALID, "max_iterations must be >= 1");
  if (tau == 0) return TPF_OK;
  if (!S || !K || !W || !V || !iters || !workspace || workspace_bytes < tpf_dense_workspace_bytes(b))
    return set_error(TPF_ERR_INVALID, "tpf_dense_ws_fpi_c128: null pointer or small workspace");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t err = cudaMemsetAsync(workspace, 0, sizeof(unsigned long long), st);
  if (err != cudaSuccess) return set_cuda_error("cudaMemsetAsync(counter)", err);
  ws::Args a;
  a.tau = tau;
  a.b = b;
  a.ks_count = (b + 3) / 4;
  a.S = S;
  a.s_node = s_node_stride;
  a.s_case = s_case_stride;
  a.K = K;
  a.W = W;
  a.v_flat_re = v_flat_re;
  a.v_flat_im = v_flat_im;
  a.tol2 = tol * tol;
  a.max_iter = max_iter;
  a.V = V;
  a.v_node = v_node_stride;
  a.v_case = v_case_stride;
  a.iters = iters;
  a.counter = static_cast<unsigned long long*>(workspace);
  // step-test bracket: |d| < hi_small<<32 <= 0.7 tol  =>  |delta|^2 < 0.98 tol^2;
  // |d| > (hi_big + 1)<<32 > tol  =>  |delta|^2 > tol^2 (monotone rounding)
  a.tol_hi_small = hi_word(0.7 * tol);
  a.tol_hi_big = hi_word(tol);
  switch ((b + 7) / 8) {
    case 1: return a.ks_count == 2 ? ws_launch<1, 2>(a, st, sms) : ws_launch<1, 1>(a, st, sms);
    case 2: return a.ks_count == 4 ? ws_launch<2, 4>(a, st, sms) : ws_launch<2, 3>(a, st, sms);
    case 3: return a.ks_count == 6 ? ws_launch<3, 6>(a, st, sms) : ws_launch<3, 5>(a, st, sms);
    case 4: return a.ks_count == 8 ? ws_launch<4, 8>(a, st, sms) : ws_launch<4, 7>(a, st, sms);
    case 5: return a.ks_count == 10 ? ws_launch<5, 10>(a, st, sms) : ws_launch<5, 9>(a, st, sms);
    case 6: return a.ks_count == 12 ? ws_launch<6, 12>(a, st, sms) : ws_launch<6, 11>(a, st, sms);
    case 7: return a.ks_count == 14 ? ws_launch<7, 14>(a, st, sms) : ws_launch<7, 13>(a, st, sms);
    case 8: return a.ks_count == 16 ? ws_launch<8, 16>(a, st, sms) : ws_launch<8, 15>(a, st, sms);
    case 9: return a.ks_count == 18 ? ws_launch<9, 18>(a, st, sms) : ws_launch<9, 17>(a, st, sms);
    case 10: return a.ks_count == 20 ? ws_launch<10, 20>(a, st, sms) : ws_launch<10, 19>(a, st, sms);
    case 11: return a.ks_count == 22 ? ws_launch<11, 22>(a, st, sms) : ws_launch<11, 21>(a, st, sms);
    case 12: return a.ks_count == 24 ? ws_launch<12, 24>(a, st, sms) : ws_launch<12, 23>(a, st, sms);
    case 13: return a.ks_count == 26 ? ws_launch<13, 26>(a, st, sms) : ws_launch<13, 25>(a, st, sms);
    default: break;
  }
  return set_error(TPF_ERR_UNSUPPORTED, "unsupported b");
}

#ifdef TPF_AB_VARIANTS
extern "C" int tpf_dense_solo_fpi_c128(int64_t tau, int32_t b, const double* S, int64_t s_node_stride,
                                       int64_t s_case_stride, const double* K, const double* W, double v_flat_re,
                                       double v_flat_im, double tol, int32_t max_iter, double* V,
                                       int64_t v_node_stride, int64_t v_case_stride, int32_t* iters,
                                       void* workspace, size_t workspace_bytes, void* stream) {
  if (tau < 0 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_dense_solo_fpi_c128: need tau >= 0 and b >= 1");
  if (b > 104) return set_error(TPF_ERR_UNSUPPORTED, "tpf_dense_solo_fpi_c128: b > 104");
  if (tau > INT_MAX - 4096) return set_error(TPF_ERR_INVALID, "tau too large for one launch; shard it");
  if (!(tol > 0.0)) return set_error(TPF_ERR_INVALID, "tolerance must be positive");
  if (max_iter < 1) return set_error(TPF_ERR_INVALID, "max_iterations must be >= 1");
  if (tau == 0) return TPF_OK;
  if (!S || !K || !W || !V || !iters || !workspace || workspace_bytes < 256)
    return set_error(TPF_ERR_INVALID, "tpf_dense_solo_fpi_c128: null pointer or small workspace");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t err = cudaMemsetAsync(workspace, 0, sizeof(unsigned long long), st);
  if (err != cudaSuccess) return set_cuda_error("cudaMemsetAsync(counter)", err);
  ws::Args a;
  a.tau = tau;
  a.b = b;
  a.ks_count = (b + 3) / 4;
  a.S = S;
  a.s_node = s_node_stride;
  a.s_case = s_case_stride;
  a.K = K;
  a.W = W;
  a.v_flat_re = v_flat_re;
  a.v_flat_im = v_flat_im;
  a.tol2 = tol * tol;
  a.max_iter = max_iter;
  a.V = V;
  a.v_node = v_node_stride;
  a.v_case = v_case_stride;
  a.iters = iters;
  a.counter = static_cast<unsigned long long*>(workspace);
  switch ((b + 7) / 8) {
    case 1: return a.ks_count == 2 ? solo::launch<1, 2>(a, st, sms) : solo::launch<1, 1>(a, st, sms);
    case 2: return a.ks_count == 4 ? solo::launch<2, 4>(a, st, sms) : solo::launch<2, 3>(a, st, sms);
    case 3: return a.ks_count == 6 ? solo::launch<3, 6>(a, st, sms) : solo::launch<3, 5>(a, st, sms);
    case 4: return a.ks_count == 8 ? solo::launch<4, 8>(a, st, sms) : solo::launch<4, 7>(a, st, sms);
    case 5: return a.ks_count == 10 ? solo::launch<5, 10>(a, st, sms) : solo::launch<5, 9>(a, st, sms);
    case 6: return a.ks_count == 12 ? solo::launch<6, 12>(a, st, sms) : solo::launch<6, 11>(a, st, sms);
    case 7: return a.ks_count == 14 ? solo::launch<7, 14>(a, st, sms) : solo::launch<7, 13>(a, st, sms);
    case 8: return a.ks_count == 16 ? solo::launch<8, 16>(a, st, sms) : solo::launch<8, 15>(a, st, sms);
    case 9: return a.ks_count == 18 ? solo::launch<9, 18>(a, st, sms) : solo::launch<9, 17>(a, st, sms);
    case 10: return a.ks_count == 20 ? solo::launch<10, 20>(a, st, sms) : solo::launch<10, 19>(a, st, sms);
    case 11: return a.ks_count == 22 ? solo::launch<11, 22>(a, st, sms) : solo::launch<11, 21>(a, st, sms);
    case 12: return a.ks_count == 24 ? solo::launch<12, 24>(a, st, sms) : solo::launch<12, 23>(a, st, sms);
    case 13: return a.ks_count == 26 ? solo::launch<13, 26>(a, st, sms) : solo::launch<13, 25>(a, st, sms);
    default: break;
  }
  return set_error(TPF_ERR_UNSUPPORTED, "unsupported b");
}
#endif  // TPF_AB_VARIANTS
