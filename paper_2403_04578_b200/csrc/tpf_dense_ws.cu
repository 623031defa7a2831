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
//     fragment); the GEMM issues, per k-step, the 26 DMMAs that do not depend
//     on each other before the 26 that accumulate onto them.
#include <climits>
#include <cstdlib>

#include "tpf_common.cuh"
#include "tpf_internal.h"

namespace tpf {
namespace ws {

// 12 warps: warps 0-3: MMA (SMSP w), 4-7: EW group 0, 8-11: EW group 1
// (the SPLIT=2 variant launches 16 warps: see ws_launch)
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kGroupCols = 208;  // 104 (U / V' hand-off) + 104 (guarded iterate)

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
};

__device__ __forceinline__ int claim(unsigned long long* counter) {
  const unsigned long long c = atomicAdd(counter, 1ull);
  return c < (unsigned long long)INT_MAX ? int(c) : INT_MAX;
}

struct Shared {
  uint64_t full_u[4][2];  // EW -> MMA: U of group g ready (or group finished)
  uint64_t full_v[4][2];  // MMA -> EW: V' of group g ready
  int done[4][2];
  uint32_t tmem;
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

template <int NB, int KS>
__device__ __forceinline__ void ew_warp(const Args& a, Shared& sh, double2* stage, int q, int g, int lane,
                                        uint32_t tm) {
  const int slot = lane >> 2, qq = lane & 3;
  const int b = a.b;
  const int64_t tau = a.tau;
  const uint32_t uv = tm + g * kGroupCols, vc = uv + 104;
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

  for (;;) {
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
      tmem_ld4d(uv + 8 * lb, nv);  // V' of the last GEMM (ignored by fresh slots)
      tmem_wait_ld();
      double xr[2], xi[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        xr[e] = fresh ? a.v_flat_re : nv.get(e);
        xi[e] = fresh ? a.v_flat_im : nv.get(2 + e);
        double m2 = __fma_rn(xr[e], xr[e], xi[e] * xi[e]);
        if (m2 < kZeroGuard2) {  // fpi.py:39-41
          xr[e] = kZeroGuard;
          xi[e] = 0.0;
          m2 = kZeroGuard * kZeroGuard;
        }
        const double r = 1.0 / m2;
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

    // ---- wait for V' of this group, per-case step test (dense.py:125-126, 189-193) ----
    mbar_wait(&sh.full_v[q][g], par);
    par ^= 1u;
    tmem_fence_after();
    bool small = true;
#pragma unroll
    for (int lb = 0; lb < NB; ++lb) {
      D4 nv, ov;
      tmem_ld4d(uv + 8 * lb, nv);
      tmem_ld4d(vc + 8 * lb, ov);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double dr = nv.get(e) - ov.get(e), di = nv.get(2 + e) - ov.get(2 + e);
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
      // retire: V' of the retiring slots to global memory, per-case count
#pragma unroll
      for (int lb = 0; lb < NB; ++lb) {
        D4 nv;
        tmem_ld4d(uv + 8 * lb, nv);
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
    if (__all_sync(0xffffffffu, cid == INT_MAX)) {
      if (lane == 0) sh.done[q][g] = 1;
      __syncwarp();
      tmem_fence_before();
      mbar_arrive(&sh.full_u[q][g]);
      break;
    }
  }
}

// SPLIT DMMA warps per SMSP share each GEMM (node blocks split NBA / NB - NBA):
// SPLIT = 1: 12 warps (4 DMMA + 8 EW); SPLIT = 2: 16 warps (8 DMMA + 8 EW), so
// two DMMA streams feed every FP64 tensor pipe.
template <int NB, int KS, int SPLIT>
__global__ void __launch_bounds__(32 * (8 + 4 * SPLIT), 1) dense_ws_kernel(const Args a) {
  constexpr int NBA = SPLIT == 1 ? NB : (NB + 1) / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = a.b;
  double2* k_sm = reinterpret_cast<double2*>(smem_raw);                 // [NB][KS][32]
  double* w_re = reinterpret_cast<double*>(k_sm + size_t(NB) * KS * 32);  // [NB*8]
  double* w_im = w_re + NB * 8;
  double2* stage = reinterpret_cast<double2*>(w_im + NB * 8);           // [8 EW warps][64]
  Shared& sh = *reinterpret_cast<Shared*>(stage + 8 * 64);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  constexpr int kT = 32 * (8 + 4 * SPLIT);
  for (int idx = tid; idx < NB * KS * 32; idx += kT) {
    const int l = idx & 31, ks = (idx >> 5) % KS, nb = (idx >> 5) / KS;
    const int row = 8 * nb + (l >> 2), col = 4 * ks + (l & 3);
    k_sm[idx] = (row < b && col < b) ? ldg_c128(a.K, int64_t(row) * b + col) : make_double2(0.0, 0.0);
  }
  for (int i = tid; i < NB * 8; i += kT) {
    const double2 w = (i < b) ? ldg_c128(a.W, i) : make_double2(0.0, 0.0);
    w_re[i] = w.x;
    w_im[i] = w.y;
  }
  if (tid == 0) {
    for (int q = 0; q < 4; ++q)
      for (int g = 0; g < 2; ++g) {
        mbar_init(&sh.full_u[q][g], 32);
        mbar_init(&sh.full_v[q][g], 32 * SPLIT);
        sh.done[q][g] = 0;
      }
  }
  if (warp == 0) tmem_alloc(&sh.tmem, kTmemCols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const int q = warp & 3;
  const uint32_t tm = sh.tmem + (uint32_t(32 * q) << 16);
  const int wg = warp >> 2;
  if (wg == 0) {
    mma_warp<KS, 0, NBA, SPLIT>(a, sh, k_sm, w_re, w_im, q, lane, tm);
  } else if (SPLIT == 2 && wg == 1) {
    if constexpr (SPLIT == 2) mma_warp<KS, NBA, NB - NBA, SPLIT>(a, sh, k_sm, w_re, w_im, q, lane, tm);
  } else {
    const int e = warp - 4 * SPLIT;  // 0..7
    ew_warp<NB, KS>(a, sh, stage + e * 64, q, e >> 2, lane, tm);
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(sh.tmem, kTmemCols);
}

template <int NB, int KS, int SPLIT>
int launch(const Args& a, cudaStream_t st, int sms) {
  const size_t smem = size_t(NB) * a.ks_count * 32 * 16 + size_t(NB) * 8 * 16 + 8 * 64 * 16 + sizeof(Shared) + 64;
  cudaError_t err = cudaFuncSetAttribute(dense_ws_kernel<NB, KS, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (err != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(dense_ws)", err);
  int64_t grid = sms;
  const int64_t need = (a.tau + 63) / 64;  // 64 slots per CTA
  if (need < grid) grid = need;
  if (grid < 1) grid = 1;
  dense_ws_kernel<NB, KS, SPLIT><<<unsigned(grid), 32 * (8 + 4 * SPLIT), smem, st>>>(a);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(dense_ws_kernel)", err);
  return TPF_OK;
}

}  // namespace ws

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
}  // namespace tpf

using namespace tpf;

// Default: one DMMA warp per SMSP (12 warps).  TPF_WS_SPLIT=2 selects two DMMA
// warps per SMSP sharing each GEMM (16 warps); measured slower on C2 (8.17 vs
// 7.38 ms): the elementwise warps then cannot refill U fast enough.
template <int NB, int KS>
static int ws_launch(const ws::Args& a, cudaStream_t st, int sms) {
  static const int split = [] {
    const char* e = getenv("TPF_WS_SPLIT");
    return (e && e[0] == '2') ? 2 : 1;
  }();
  if constexpr (NB >= 2) {
    if (split == 2) return ws::launch<NB, KS, 2>(a, st, sms);
  }
  return ws::launch<NB, KS, 1>(a, st, sms);
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
  if (!S || !K || !W || !V || !iters || !workspace || workspace_bytes < 256)
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
