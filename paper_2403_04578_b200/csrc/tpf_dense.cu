// Dense Tensor Power Flow on sm_100a: persistent FP64-DMMA fixed-point kernel.
//
// Replaces the hot loop of the reference `batch_solve_dense`
// (pkg/src/tpflow/dense.py:166-193, per-iteration op chain `_iterate_chunk`
// dense.py:114-126):   V' = K (S* ./ conj(V)) + W,  K = -inv(Y_dd),
// written case-major as V'(case, :) = U(case, :) K^T + W with U = S*/conj(V).
//
// Layout of the work (b <= 104, so K fits in shared memory):
//   * one CTA per SM, 8 warps, persistent;
//   * K^T lives in shared memory for the whole launch, pre-swizzled into the
//     B-fragment order of mma.m8n8k4 (one 16-byte (re,im) pair per lane per
//     fragment, so every fragment load is a conflict-free LDS.128);
//   * warps work in pairs; a pair owns 8 case "slots" (the M=8 rows of the MMA)
//     and splits the 8*NB output nodes between its two warps (7/6 blocks at
//     b=100, alternated between pairs so every SM sub-partition gets the same
//     FP64 work);
//   * the iterate V, the old iterate and S* of a slot stay in registers across
//     iterations (C-fragment layout); only U = S*/conj(V) goes through shared
//     memory (A-fragment order), once per iteration;
//   * complex GEMM = 4 real DMMAs per (k-step, node block):
//       Re += Ur*Kr - Ui*Ki,  Im += Ur*Ki + Ui*Kr,   accumulators start at W;
//   * epilogue: per-case |V'-V|^2 < tol^2 over all nodes (warp ballot + pair
//     exchange), per-case freeze, and immediate refill of a frozen slot with
//     the next unsolved case from a global atomic counter (continuous
//     batching: no tile waits for its slowest case).
// Each case's arithmetic is independent of the slot, warp, CTA or launch it
// runs in, so results are bitwise invariant to permutation and sharding.
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "tpf_common.cuh"
#include "tpf_internal.h"

#ifdef TPF_PHASE_TIMING
// per warp: [0] elementwise, [1] barrier U, [2] GEMM, [3] epilogue math, [4] barrier flags,
// [5] retire/refill, [6] iterations, [7] total
__device__ long long g_phase[148 * 2 * 8][8];
#define PHASE_MARK(i)                         \
  do {                                        \
    const long long _t = clock64();           \
    ph[i] += _t - ph_t;                       \
    ph_t = _t;                                \
  } while (0)
#else
#define PHASE_MARK(i) \
  do {                \
  } while (0)
#endif

namespace tpf {

constexpr int kPairs = 4;          // warp pairs per CTA
constexpr int kWarps = 2 * kPairs;  // 8 warps
constexpr int kThreads = 32 * kWarps;

struct DenseArgs {
  int64_t tau;
  int b;
  int ks_count;  // k-steps of 4 input nodes: ceil(b/4)
  const double* S;
  int64_t s_node, s_case;  // strides in complex elements
  const double* K;         // b x b complex, row-major
  const double* W;         // b complex
  double v_flat_re, v_flat_im;
  double tol2;
  int max_iter;
  double* V;
  int64_t v_node, v_case;
  int32_t* iters;
  unsigned long long* counter;  // next unclaimed case
};

template <int NB>
struct DenseSmem {
  static constexpr int kMaxKs = 2 * NB;
  // K^T in B-fragment order: [nb][ks][lane] -> (Kr, Ki) of K[8nb + lane/4][4ks + lane%4]
  static constexpr size_t k_bytes(int ks) { return size_t(NB) * ks * 32 * sizeof(double2); }
  // U in A-fragment order per pair: [pair][ks][lane] -> U[slot lane/4][node 4ks + lane%4]
  static constexpr size_t u_bytes(int ks) { return size_t(kPairs) * ks * 32 * sizeof(double2); }
  static constexpr size_t w_bytes() { return size_t(NB) * 8 * sizeof(double2); }
  static constexpr size_t misc_bytes() { return 1024; }
  static size_t total(int ks) { return k_bytes(ks) + u_bytes(ks) + w_bytes() + misc_bytes(); }
};

// Next unclaimed case index, saturated at INT_MAX (= idle slot).
__device__ __forceinline__ int claim_case(unsigned long long* counter) {
  const unsigned long long c = atomicAdd(counter, 1ull);
  return c < (unsigned long long)INT_MAX ? int(c) : INT_MAX;
}

// One k-step of the complex GEMM for NBW node blocks: two passes so that the
// two DMMAs accumulating into the same fragment are 2*NBW instructions apart.
template <int NBH, int NBW>
__device__ __forceinline__ void kstep(double (&vr)[NBH][2], double (&vi)[NBH][2], const double2& u,
                                      const double2 (&kf)[NBW]) {
  const double nui = neg_int(u.y);
#pragma unroll
  for (int lb = 0; lb < NBW; ++lb) {
    dmma884(vr[lb][0], vr[lb][1], u.x, kf[lb].x);
    dmma884(vi[lb][0], vi[lb][1], u.x, kf[lb].y);
  }
#pragma unroll
  for (int lb = 0; lb < NBW; ++lb) {
    dmma884(vr[lb][0], vr[lb][1], nui, kf[lb].y);
    dmma884(vi[lb][0], vi[lb][1], u.y, kf[lb].x);
  }
}

template <int NBW>
__device__ __forceinline__ void load_frags(double2& u, double2 (&kf)[NBW], const double2* kb, const double2* ub,
                                           int ks, int KS) {
  u = ub[ks * 32];
#pragma unroll
  for (int lb = 0; lb < NBW; ++lb) kf[lb] = kb[(size_t(lb) * KS + ks) * 32];
}

// V' += U K^T for this warp's NBW node blocks; fragments ping-pong between two
// register sets so the next k-step's shared-memory loads overlap the DMMAs.
template <int NBH, int NBW>
__device__ __forceinline__ void gemm_warp(double (&vr)[NBH][2], double (&vi)[NBH][2], const double2* kb,
                                          const double2* ub, int KS) {
  double2 u0, u1, k0[NBW], k1[NBW];
  load_frags<NBW>(u0, k0, kb, ub, 0, KS);
#pragma unroll 1
  for (int ks = 0; ks < KS; ks += 2) {
    const bool odd = ks + 1 < KS;
    if (odd) load_frags<NBW>(u1, k1, kb, ub, ks + 1, KS);
    kstep<NBH, NBW>(vr, vi, u0, k0);
    if (ks + 2 < KS) load_frags<NBW>(u0, k0, kb, ub, ks + 2, KS);
    if (odd) kstep<NBH, NBW>(vr, vi, u1, k1);
  }
}

// 3M variant (Gauss, as the default ws kernel): P1 += ur kr, P2 += ui ki,
// P3 += (ur + ui)(kr + ki), each accumulator over the k-steps in the same order
// as the ws kernel, so the two kernels give the same bits.
template <int NBH, int NBW>
__device__ __forceinline__ void kstep3p(double (&p1)[NBH][2], double (&p2)[NBH][2], double (&p3)[NBH][2],
                                        const double2& u, const double2 (&kf)[NBW]) {
  const double us = u.x + u.y;
#pragma unroll
  for (int lb = 0; lb < NBW; ++lb) {
    const double kss = kf[lb].x + kf[lb].y;
    dmma884(p1[lb][0], p1[lb][1], u.x, kf[lb].x);
    dmma884(p2[lb][0], p2[lb][1], u.y, kf[lb].y);
    dmma884(p3[lb][0], p3[lb][1], us, kss);
  }
}

template <int NBH, int NBW>
__device__ __forceinline__ void gemm_warp3(double (&p1)[NBH][2], double (&p2)[NBH][2], double (&p3)[NBH][2],
                                           const double2* kb, const double2* ub, int KS) {
  double2 u0, u1, k0[NBW], k1[NBW];
  load_frags<NBW>(u0, k0, kb, ub, 0, KS);
#pragma unroll 1
  for (int ks = 0; ks < KS; ks += 2) {
    const bool odd = ks + 1 < KS;
    if (odd) load_frags<NBW>(u1, k1, kb, ub, ks + 1, KS);
    kstep3p<NBH, NBW>(p1, p2, p3, u0, k0);
    if (ks + 2 < KS) load_frags<NBW>(u0, k0, kb, ub, ks + 2, KS);
    if (odd) kstep3p<NBH, NBW>(p1, p2, p3, u1, k1);
  }
}

template <int NB, bool M3>
__global__ void __launch_bounds__(kThreads, 1) dense_fpi_kernel(const DenseArgs a) {
  constexpr int NBH = (NB + 1) / 2;  // max node blocks per warp
  constexpr uint32_t kTmemCols = 256;  // 2 warps per lane quadrant x 128 columns
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int KS = a.ks_count;
  double2* k_sm = reinterpret_cast<double2*>(smem_raw);
  double2* u_all = k_sm + size_t(NB) * KS * 32;
  double2* w_sm = u_all + size_t(kPairs) * KS * 32;
  uint32_t* flags = reinterpret_cast<uint32_t*>(w_sm + NB * 8);  // [pair][2]
  int* next_ids = reinterpret_cast<int*>(flags + 2 * kPairs);     // [pair][8 slots][2]
  uint32_t* tmem_base_sm = reinterpret_cast<uint32_t*>(next_ids + kPairs * 16);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int pair = warp >> 1;
  const int half = warp & 1;
  const int q = lane & 3;      // C-fragment column group: nodes 2q, 2q+1 of a block
  const int slot = lane >> 2;  // C/A-fragment row: case slot 0..7
  const int b = a.b;
  const int64_t tau = a.tau;

  if (warp == 0) tmem_alloc(tmem_base_sm, kTmemCols);

  // ---- stage K^T fragments and W into shared memory (once per launch) ----
  for (int idx = tid; idx < NB * KS * 32; idx += kThreads) {
    const int l = idx & 31;
    const int ks = (idx >> 5) % KS;
    const int nb = (idx >> 5) / KS;
    const int row = 8 * nb + (l >> 2);
    const int col = 4 * ks + (l & 3);
    double2 v = make_double2(0.0, 0.0);
    if (row < b && col < b) v = ldg_c128(a.K, int64_t(row) * b + col);
    k_sm[idx] = v;
  }
  for (int i = tid; i < NB * 8; i += kThreads) {
    const double2 w = (i < b) ? ldg_c128(a.W, i) : make_double2(0.0, 0.0);
    reinterpret_cast<double*>(w_sm)[i] = w.x;           // re plane
    reinterpret_cast<double*>(w_sm)[NB * 8 + i] = w.y;  // im plane
  }

  // ---- slot bookkeeping: two prefetched case ids per slot (ring of 2) ----
  if (half == 0 && lane < 8) {
    next_ids[(pair * 8 + lane) * 2 + 0] = claim_case(a.counter);
    next_ids[(pair * 8 + lane) * 2 + 1] = claim_case(a.counter);
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();

  // TMEM holds, per thread, S* (columns [0,8*NBH)) and the old iterate
  // (columns [8*NBH, 16*NBH)) of its C-fragment entries: 4 doubles per block.
  const uint32_t tm = *tmem_base_sm + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * 128);
  const uint32_t tm_s = tm, tm_o = tm + 8 * NBH;

  // this warp's node blocks (alternate the larger half between pairs)
  const int n_big = NBH, n_small = NB - NBH;
  const bool big_first = ((pair >> 1) & 1) == 0;
  const int nbw = (half == 0) == big_first ? n_big : n_small;
  const int nb0 = half == 0 ? 0 : (big_first ? n_big : n_small);

  double2* u_sm = u_all + size_t(pair) * KS * 32;
  const int bar_id = 1 + pair;

  double vr[NBH][2], vi[NBH][2];  // iterate / accumulators (C layout)
  int cid = INT_MAX;  // current case of my slot (INT_MAX = idle)
  int n_it = 0;       // updates applied to the current case
  int refills = 0;    // ring position

  // S* entries of case c for block lb of this thread (zeros for padding / idle)
  auto fetch_s = [&](int c, int lb, double& s0r, double& s0i, double& s1r, double& s1i) {
    s0r = s0i = s1r = s1i = 0.0;
    const int node = 8 * (nb0 + lb) + 2 * q;
    if (c < tau) {
      if (node < b) {
        const double2 s = ldg_c128(a.S, node * a.s_node + int64_t(c) * a.s_case);
        s0r = s.x;
        s0i = -s.y;  // S* (dense.py:154)
      }
      if (node + 1 < b) {
        const double2 s = ldg_c128(a.S, (node + 1) * a.s_node + int64_t(c) * a.s_case);
        s1r = s.x;
        s1i = -s.y;
      }
    }
  };
  auto flat_start = [&](int lb) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      vr[lb][e] = a.v_flat_re;
      vi[lb][e] = a.v_flat_im;
    }
  };

  // Warm L2 with this thread's entries of the case its slot will take next, so
  // the refill load after a freeze hits L2 instead of HBM.
  auto prefetch_case = [&](int c) {
    if (c >= tau) return;
#pragma unroll
    for (int lb = 0; lb < NBH; ++lb) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int node = 8 * (nb0 + lb) + 2 * q + e;
        if (lb < nbw && node < b) {
          const double* p = a.S + 2 * (node * a.s_node + int64_t(c) * a.s_case);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
        }
      }
    }
  };

  // initial fill (refill #0)
  cid = next_ids[(pair * 8 + slot) * 2 + 0];
  refills = 1;
  if (cid >= tau) cid = INT_MAX;
#pragma unroll
  for (int lb = 0; lb < NBH; ++lb) {
    if (lb < nbw) {
      double s0r, s0i, s1r, s1i;
      fetch_s(cid, lb, s0r, s0i, s1r, s1i);
      tmem_st4d(tm_s + 8 * lb, s0r, s1r, s0i, s1i);
    }
    flat_start(lb);
  }
  tmem_wait_st();
  prefetch_case(next_ids[(pair * 8 + slot) * 2 + 1]);
  bool want_prefetch = false;

#ifdef TPF_PHASE_TIMING
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_t = clock64();
  const long long ph_start = ph_t;
#endif
  for (;;) {
    // ---------- elementwise: guard, keep old iterate, U = S*/conj(V) ----------
    {
      D4 sv[NBH];
#pragma unroll
      for (int lb = 0; lb < NBH; ++lb)
        if (lb < nbw) tmem_ld4d(tm_s + 8 * lb, sv[lb]);
      tmem_wait_ld();
#pragma unroll
      for (int lb = 0; lb < NBH; ++lb) {
        if (lb < nbw) {
          double xr2[2], xi2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double xr = vr[lb][e], xi = vi[lb][e];
            double m2 = __fma_rn(xr, xr, xi * xi);
            if (m2 < kZeroGuard2) {  // fpi.py:39-41 / dense.py:170-172
              xr = kZeroGuard;
              xi = 0.0;
              m2 = kZeroGuard * kZeroGuard;
            }
            xr2[e] = xr;
            xi2[e] = xi;
            // S*/conj(v) = S* v / |v|^2
            const double srr = sv[lb].get(e), sii = sv[lb].get(2 + e);
            const double r = M3 ? rcp_nr(m2) : 1.0 / m2;
            const double ur = __fma_rn(srr, xr, -(sii * xi)) * r;
            const double ui = __fma_rn(srr, xi, sii * xr) * r;
            const int node = 8 * (nb0 + lb) + 2 * q + e;
            const int ks = node >> 2;
            if (ks < KS) u_sm[ks * 32 + slot * 4 + (node & 3)] = make_double2(ur, ui);
          }
          tmem_st4d(tm_o + 8 * lb, xr2[0], xr2[1], xi2[0], xi2[1]);
        }
      }
    }
    tmem_wait_st();
    PHASE_MARK(0);
    named_bar(bar_id, 64);  // U complete for both halves
    PHASE_MARK(1);
    if (want_prefetch) {  // the ring entry written after the last refill is visible now
      prefetch_case(next_ids[(pair * 8 + slot) * 2 + (refills & 1)]);
      want_prefetch = false;
    }

    // ---------- GEMM: V' = W + U K^T on FP64 tensor cores ----------
    if constexpr (M3) {
      double p1[NBH][2], p2[NBH][2], p3[NBH][2];
#pragma unroll
      for (int lb = 0; lb < NBH; ++lb) {
        if (lb < nbw) {
          const double2 wr = w_sm[(8 * (nb0 + lb) + 2 * q) / 2];
          const double2 wi = w_sm[(NB * 8 + 8 * (nb0 + lb) + 2 * q) / 2];
          p1[lb][0] = wr.x;
          p1[lb][1] = wr.y;
          p2[lb][0] = p2[lb][1] = 0.0;
          p3[lb][0] = wr.x + wi.x;
          p3[lb][1] = wr.y + wi.y;
        }
      }
      const double2* kb = k_sm + size_t(nb0) * KS * 32 + lane;
      if (nbw == NBH) {
        gemm_warp3<NBH, NBH>(p1, p2, p3, kb, u_sm + lane, KS);
      } else {
        if constexpr (NB - NBH > 0) gemm_warp3<NBH, NB - NBH>(p1, p2, p3, kb, u_sm + lane, KS);
      }
#pragma unroll
      for (int lb = 0; lb < NBH; ++lb) {
        if (lb < nbw) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            vr[lb][e] = p1[lb][e] - p2[lb][e];
            vi[lb][e] = (p3[lb][e] - p1[lb][e]) - p2[lb][e];
          }
        }
      }
    } else {
#pragma unroll
      for (int lb = 0; lb < NBH; ++lb) {
        if (lb < nbw) {
          // (node 2q, 2q+1) pairs of each plane land directly in the DMMA register pairs
          const double2 wr = w_sm[(8 * (nb0 + lb) + 2 * q) / 2];
          const double2 wi = w_sm[(NB * 8 + 8 * (nb0 + lb) + 2 * q) / 2];
          vr[lb][0] = wr.x;
          vr[lb][1] = wr.y;
          vi[lb][0] = wi.x;
          vi[lb][1] = wi.y;
        }
      }
      const double2* kb = k_sm + size_t(nb0) * KS * 32 + lane;
      if (nbw == NBH) {
        gemm_warp<NBH, NBH>(vr, vi, kb, u_sm + lane, KS);
      } else {
        if constexpr (NB - NBH > 0) gemm_warp<NBH, NB - NBH>(vr, vi, kb, u_sm + lane, KS);
      }
    }

    PHASE_MARK(2);
    // ---------- epilogue: per-case step test (dense.py:125-126, 189-193) ----------
    bool small = true;
    {
      D4 ov[NBH];
#pragma unroll
      for (int lb = 0; lb < NBH; ++lb)
        if (lb < nbw) tmem_ld4d(tm_o + 8 * lb, ov[lb]);
      tmem_wait_ld();
#pragma unroll
      for (int lb = 0; lb < NBH; ++lb) {
        if (lb < nbw) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int node = 8 * (nb0 + lb) + 2 * q + e;
            const double dr = vr[lb][e] - ov[lb].get(e);
            const double di = vi[lb][e] - ov[lb].get(2 + e);
            const double d2 = __fma_rn(dr, dr, di * di);
            // NaN/inf never compare small: they hold the case open to the cap
            if (node < b && !(d2 < a.tol2)) small = false;
          }
        }
      }
    }
    const uint32_t ball = __ballot_sync(0xffffffffu, small);
    if (lane == 0) flags[pair * 2 + half] = ball;
    PHASE_MARK(3);
    named_bar(bar_id, 64);  // flags of both halves visible; U reads finished
    PHASE_MARK(4);
    const uint32_t both = flags[pair * 2] & flags[pair * 2 + 1];
    const bool my_small = ((both >> (slot * 4)) & 0xFu) == 0xFu;

    bool done = false;
    if (cid != INT_MAX) {
      ++n_it;
      done = my_small || n_it >= a.max_iter;
    }
    if (done) {
      // retire: V and per-case iteration count
#pragma unroll
      for (int lb = 0; lb < NBH; ++lb) {
        if (lb < nbw) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int node = 8 * (nb0 + lb) + 2 * q + e;
            if (node < b) {  // two 8-byte stores: (re, im) are not a register pair
              double* p = a.V + 2 * (node * a.v_node + int64_t(cid) * a.v_case);
              p[0] = vr[lb][e];
              p[1] = vi[lb][e];
            }
          }
        }
      }
      if (half == 0 && q == 0) a.iters[cid] = n_it;
      // refill from the prefetch ring; warp 0 of the pair tops the ring up
      const int ring = (pair * 8 + slot) * 2;
      const int nc = next_ids[ring + (refills & 1)];
      if (half == 0 && q == 0) next_ids[ring + ((refills + 1) & 1)] = claim_case(a.counter);
      ++refills;
      cid = (nc < tau) ? nc : INT_MAX;
      n_it = 0;
      want_prefetch = cid != INT_MAX;
    }
    // TMEM access is warp-collective (.sync.aligned): the whole warp rewrites
    // S*, retiring lanes with their new case, the others with what they hold.
    if (__any_sync(0xffffffffu, done)) {
      D4 cur[NBH];
#pragma unroll
      for (int lb = 0; lb < NBH; ++lb)
        if (lb < nbw) tmem_ld4d(tm_s + 8 * lb, cur[lb]);
      tmem_wait_ld();
#pragma unroll
      for (int lb = 0; lb < NBH; ++lb) {
        if (lb < nbw) {
          double s0r = cur[lb].get(0), s1r = cur[lb].get(1), s0i = cur[lb].get(2), s1i = cur[lb].get(3);
          if (done) {
            fetch_s(cid, lb, s0r, s0i, s1r, s1i);
            flat_start(lb);
          }
          tmem_st4d(tm_s + 8 * lb, s0r, s1r, s0i, s1i);
        }
      }
    }
    tmem_wait_st();
    PHASE_MARK(5);
#ifdef TPF_PHASE_TIMING
    ph[6] += 1;
#endif
    if (__all_sync(0xffffffffu, cid == INT_MAX)) break;
  }
#ifdef TPF_PHASE_TIMING
  ph[7] = clock64() - ph_start;
  if (lane == 0 && blockIdx.x < 148 * 2)
    for (int i = 0; i < 8; ++i) g_phase[blockIdx.x * 8 + warp][i] = ph[i];
#endif
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(*tmem_base_sm, kTmemCols);
}

template <int NB>
static int launch_dense(const DenseArgs& a, cudaStream_t stream, int sm_count) {
  // 3M GEMM + Newton reciprocal (bitwise equal to the default ws kernel); A/B
  // builds (-DTPF_AB_VARIANTS) also carry the 4-DMMA arithmetic (TPF_WS_4M=1)
#ifdef TPF_AB_VARIANTS
  static const bool four = [] {
    const char* e = getenv("TPF_WS_4M");
    return e && e[0] == '1';
  }();
  auto kern = four ? dense_fpi_kernel<NB, false> : dense_fpi_kernel<NB, true>;
#else
  auto kern = dense_fpi_kernel<NB, true>;
#endif
  const size_t smem = DenseSmem<NB>::total(a.ks_count);
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (err != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(dense)", err);
  int per_sm = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (err != cudaSuccess) return set_cuda_error("occupancy(dense)", err);
  if (per_sm < 1) return set_error(TPF_ERR_UNSUPPORTED, "dense kernel does not fit on an SM");
  if (per_sm > 2) per_sm = 2;  // each CTA holds 256 of the SM's 512 TMEM columns
  // slots in flight = 8 per pair; never launch more CTAs than needed
  const int64_t slots_per_cta = 8 * kPairs;
  int64_t grid = int64_t(per_sm) * sm_count;
  const int64_t need = (a.tau + slots_per_cta - 1) / slots_per_cta;
  if (need < grid) grid = need;
  if (grid < 1) grid = 1;
  kern<<<unsigned(grid), kThreads, smem, stream>>>(a);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(dense_fpi_kernel)", err);
  return TPF_OK;
}

size_t dense_smem_bytes(int b) {
  const int nb = (b + 7) / 8, ks = (b + 3) / 4;
  return size_t(nb) * ks * 32 * 16 + size_t(kPairs) * ks * 32 * 16 + size_t(nb) * 8 * 16 + 1024;
}

}  // namespace tpf

using namespace tpf;

#ifdef TPF_PHASE_TIMING
extern "C" int tpf_debug_phase_cycles(long long* out, int n) {
  return cudaMemcpyFromSymbol(out, g_phase, sizeof(long long) * 8 * (n < 148 * 16 ? n : 148 * 16)) == cudaSuccess
             ? 0 : 2;
}
#endif

extern "C" int tpf_dense_max_nodes(void) { return 104; }

extern "C" size_t tpf_dense_workspace_bytes(int32_t b) {
  (void)b;
  return 256 + 232448;  // counter slot + the ws kernel's shared-memory image (<= 227 KB)
}

extern "C" int tpf_dense_ws_fpi_c128(int64_t tau, int32_t b, const double* S, int64_t s_node_stride,
                                     int64_t s_case_stride, const double* K, const double* W, double v_flat_re,
                                     double v_flat_im, double tol, int32_t max_iter, double* V, int64_t v_node_stride,
                                     int64_t v_case_stride, int32_t* iters, void* workspace, size_t workspace_bytes,
                                     void* stream);

// Kernel selection for tpf_dense_fpi_c128.  Both kernels compute the same
// bits (3M GEMM, Newton reciprocal), so the choice is purely a speed one:
// batches of at most two waves of the ws kernel's slots are latency-bound
// (each case gets its own slot), and the pair kernel's shorter rounds (two
// warps on each slot group's GEMM and elementwise work) win there (C1: 0.069
// -> 0.046 ms; b=100, tau=8,760: 0.26 -> 0.16 ms); longer batches are
// throughput-bound and the ws kernel wins.  TPF_DENSE_KERNEL=pairs|ws forces
// one.
static bool use_pairs_kernel(int64_t tau) {
  static const int forced = [] {
    const char* e = getenv("TPF_DENSE_KERNEL");
    if (e && strcmp(e, "pairs") == 0) return 1;
    if (e && strcmp(e, "ws") == 0) return 0;
    return -1;
  }();
  if (forced >= 0) return forced == 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return tau <= int64_t(2) * sms * 64;
}

extern "C" int tpf_dense_pairs_fpi_c128(int64_t tau, int32_t b, const double* S, int64_t s_node_stride,
                                        int64_t s_case_stride, const double* K, const double* W,
                                        double v_flat_re, double v_flat_im, double tol, int32_t max_iter,
                                        double* V, int64_t v_node_stride, int64_t v_case_stride,
                                        int32_t* iters, void* workspace, size_t workspace_bytes,
                                        void* stream);

extern "C" int tpf_dense_fpi_c128(int64_t tau, int32_t b, const double* S, int64_t s_node_stride,
                                  int64_t s_case_stride, const double* K, const double* W,
                                  double v_flat_re, double v_flat_im, double tol, int32_t max_iter,
                                  double* V, int64_t v_node_stride, int64_t v_case_stride,
                                  int32_t* iters, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  if (use_pairs_kernel(tau))
    return tpf_dense_pairs_fpi_c128(tau, b, S, s_node_stride, s_case_stride, K, W, v_flat_re, v_flat_im, tol,
                                    max_iter, V, v_node_stride, v_case_stride, iters, workspace, workspace_bytes,
                                    stream);
  return tpf_dense_ws_fpi_c128(tau, b, S, s_node_stride, s_case_stride, K, W, v_flat_re, v_flat_im, tol, max_iter,
                               V, v_node_stride, v_case_stride, iters, workspace, workspace_bytes, stream);
}

extern "C" int tpf_dense_pairs_fpi_c128(int64_t tau, int32_t b, const double* S, int64_t s_node_stride,
                                        int64_t s_case_stride, const double* K, const double* W,
                                        double v_flat_re, double v_flat_im, double tol, int32_t max_iter,
                                        double* V, int64_t v_node_stride, int64_t v_case_stride,
                                        int32_t* iters, void* workspace, size_t workspace_bytes,
                                        void* stream) {
  if (tau < 0 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_dense_fpi_c128: need tau >= 0 and b >= 1");
  if (b > 104)
    return set_error(TPF_ERR_UNSUPPORTED,
                     "tpf_dense_fpi_c128: b > 104 does not fit K in shared memory; use tpf_dense_fpi_large_c128");
  if (tau > INT_MAX - 4096) return set_error(TPF_ERR_INVALID, "tpf_dense_fpi_c128: tau too large for one launch; shard it");
  if (!(tol > 0.0)) return set_error(TPF_ERR_INVALID, "tolerance must be positive");
  if (max_iter < 1) return set_error(TPF_ERR_INVALID, "max_iterations must be >= 1");
  if (tau == 0) return TPF_OK;
  if (!S || !K || !W || !V || !iters) return set_error(TPF_ERR_INVALID, "tpf_dense_pairs_fpi_c128: null pointer");
  if (!workspace || workspace_bytes < tpf_dense_workspace_bytes(b))
    return set_error(TPF_ERR_INVALID, "tpf_dense_fpi_c128: workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return set_cuda_error("cudaGetDevice", err);
  err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (err != cudaSuccess) return set_cuda_error("cudaDeviceGetAttribute", err);
  err = cudaMemsetAsync(workspace, 0, sizeof(unsigned long long), st);
  if (err != cudaSuccess) return set_cuda_error("cudaMemsetAsync(counter)", err);

  DenseArgs a;
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
    case 1: return launch_dense<1>(a, st, sms);
    case 2: return launch_dense<2>(a, st, sms);
    case 3: return launch_dense<3>(a, st, sms);
    case 4: return launch_dense<4>(a, st, sms);
    case 5: return launch_dense<5>(a, st, sms);
    case 6: return launch_dense<6>(a, st, sms);
    case 7: return launch_dense<7>(a, st, sms);
    case 8: return launch_dense<8>(a, st, sms);
    case 9: return launch_dense<9>(a, st, sms);
    case 10: return launch_dense<10>(a, st, sms);
    case 11: return launch_dense<11>(a, st, sms);
    case 12: return launch_dense<12>(a, st, sms);
    case 13: return launch_dense<13>(a, st, sms);
    default: break;
  }
  return set_error(TPF_ERR_UNSUPPORTED, "unsupported b");
}
