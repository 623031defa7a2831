// Dense Tensor Power Flow for feeders too large for a shared-memory-resident K
// (b > 104; config C5 is b = 1,000, K = 16 MB, which lives in the 126 MB L2).
//
// Same update as tpf_dense.cu (dense.py:114-126), organised as an
// iteration-synchronous loop over a compacted ACTIVE SET of cases, because
// near voltage collapse the per-case iteration counts are heavy-tailed
// (C5: batch 58 iterations, per-case mean 10.4): every iteration only the
// still-unconverged cases enter the GEMM.
//
// Per iteration (launches that early-exit when the active set is empty or
// outside their range):
//   prep    U[k, a] = S*_{k,c} / conj(v_{k,c}) for active case c = act[a]
//           (zero-voltage guard), node-major so the writes coalesce over a;
//   gemm    V'[a, n] = W[n] + sum_k U[k, a] K[n, k] on FP64 tensor cores:
//           64x64 complex CTA tiles, 16-node k-slabs double-buffered through
//           shared memory with cp.async (zero-filled at the edges), 8 warps of
//           32x16 complex each, 3 real DMMA.8x8x4 per complex fragment (3M); the
//           epilogue reads the old iterate, writes the new one in place and
//           flags the case if any |dv|^2 >= tol^2 (or non-finite);
//   compact count the update, keep flagged cases below max_iter.
//   step    advance the device-resident iteration and set the loop condition.
// The loop itself runs on the device: a CUDA graph WHILE node around these
// launches (joined to the caller's stream capture, or built and launched per
// call), so no launch is spent on iterations past the hand-off.  Once at most
// kPtMax cases remain, tail_persistent_kernel runs every remaining iteration
// in one cooperative launch (below); tail_kernel is the per-iteration
// fallback when its CTAs cannot all be resident.
// The k-order of every dot product is fixed, so a case's bits do not depend
// on its position in the active set (permutation / shard invariance).
#include <climits>
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "tpf_common.cuh"
#include "tpf_internal.h"

namespace tpf {
namespace {

constexpr int TM = 64;   // cases per CTA tile
constexpr int TN = 64;   // output nodes per CTA tile
constexpr int TK = 16;   // input nodes per k-slab (4 k-steps)
constexpr int KSTEPS = TK / 4;
constexpr int MF = TM / 8, NF = TN / 8;
constexpr int LTHREADS = 256;
constexpr int kPtMax = 256;  // persistent hand-off: active cases at most this (tail_persistent_kernel)
constexpr int kMidM = 1184;  // 32-case GEMM tiles at most this many active cases (more CTAs per iteration)

struct LargeArgs {
  int64_t tau;
  int b;
  const double2* S;
  int64_t s_node, s_case;
  const double2* K;  // b x b row-major
  const double2* W;
  double2 v_flat;
  double tol2;
  int max_iter;
  double2* V;
  int64_t v_node, v_case;
  int32_t* iters;
  // workspace
  int32_t* act[2];
  int32_t* count;  // [2]: active counts of the two lists
  int32_t* bad;    // per active position
  double2* U;      // b x tau, node-major, ld = tau
  // persistent tail (tail_persistent_kernel)
  double2* U2;       // [2][kPtMax][b]: slot-major U, double-buffered across iterations
  int32_t* stamp;    // [kPtMax]: iteration + 1 at which the slot's case last moved >= tol
  int handoff;       // gemm_kernel runs while more than this many cases are active
  int32_t* iter;     // the iteration in flight (device-resident: the loop may run on the device)
  int loop_min;      // the iteration loop continues while more than this many cases are active
  uint32_t* gbar;    // grid-barrier arrivals
};

__global__ void init_kernel(LargeArgs a, cudaGraphConditionalHandle loop) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j == 0) {
    a.count[0] = int(a.tau);
    a.count[1] = 0;
    *a.iter = 0;
    *a.gbar = 0u;
    if (loop) cudaGraphSetConditional(loop, a.tau > a.loop_min ? 1u : 0u);
  }
  for (int64_t i = j; i < kPtMax; i += int64_t(gridDim.x) * blockDim.x) a.stamp[i] = 0;
  if (j >= a.tau) return;
  a.act[0][j] = int(j);
  a.iters[j] = 0;
  for (int i = 0; i < a.b; ++i) a.V[i * a.v_node + j * a.v_case] = a.v_flat;
}

__global__ void prep_kernel(LargeArgs a) {
  const int cur = *a.iter & 1;
  const int n_act = a.count[cur];
  const int* act = a.act[cur];
  // the output list of this iteration's compaction was the input of the previous one
  if (blockIdx.x == 0 && threadIdx.x == 0) a.count[cur ^ 1] = 0;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < int64_t(n_act) * a.b;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int k = int(idx / n_act);
    const int p = int(idx - int64_t(k) * n_act);
    const int c = act[p];
    double2 v = a.V[k * a.v_node + int64_t(c) * a.v_case];
    double m2 = __fma_rn(v.x, v.x, v.y * v.y);
    if (m2 < kZeroGuard2) {
      v = make_double2(kZeroGuard, 0.0);
      m2 = kZeroGuard * kZeroGuard;
    }
    const double2 s = __ldg(a.S + k * a.s_node + int64_t(c) * a.s_case);
    const double r = 1.0 / m2;
    const double ur = __fma_rn(s.x, v.x, s.y * v.y) * r;  // conj(s) v / |v|^2
    const double ui = __fma_rn(s.x, v.y, -(s.y * v.x)) * r;
    a.U[int64_t(k) * a.tau + p] = make_double2(ur, ui);
    if (k == 0) a.bad[p] = 0;
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = pred ? 16 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}

// CTA tile TMV cases x TN nodes, 8 warps as WM x (8/WM), for the bulk of the
// solve (TMV = 64).  When at most kTailM cases are still active (near voltage
// collapse a few cases need many more iterations) tail_kernel runs instead;
// each launch exits at once when the active count is outside its range.
// Both issue the same DMMAs in the same order for every output element, so a
// case's bits do not depend on which one ran an iteration.
constexpr int kTailM = 64;

// NST-stage cp.async pipeline over the k-slabs: the bulk kernel double-buffers;
// the tail (few cases, so few CTAs each streaming a 64-node slice of K from L2)
// keeps NST - 1 slabs in flight to cover the L2 latency.  The stage count does
// not change the k-order.
template <int TMV, int WM, int NST>
__global__ void __launch_bounds__(LTHREADS) gemm_kernel(LargeArgs a) {
  const int cur = *a.iter & 1;
  constexpr int WN = 8 / WM;
  constexpr int MFR = TMV / WM / 8, NFR = TN / WN / 8;  // fragments per warp tile
  constexpr int MFT = TMV / 8;                         // m-fragments per CTA tile
  const int n_act = a.count[cur];
  if (TMV == 32 ? (n_act <= a.handoff || n_act > kMidM) : n_act <= max(a.handoff, kMidM)) return;
  const int m0 = blockIdx.x * TMV;
  if (m0 >= n_act) return;
  const int n0 = blockIdx.y * TN;
  const int b = a.b;
  // fragment-ordered slabs: A[ks][mf][lane], B[ks][nf][lane]
  extern __shared__ __align__(16) double2 dyn_smem[];
  double2 (*As)[KSTEPS * MFT * 32] = reinterpret_cast<double2 (*)[KSTEPS * MFT * 32]>(dyn_smem);
  double2 (*Bs)[KSTEPS * NF * 32] = reinterpret_cast<double2 (*)[KSTEPS * NF * 32]>(dyn_smem + NST * KSTEPS * MFT * 32);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN;
  const int wn = warp % WN;

  auto load_slab = [&](int stage, int k0) {
    // A: TMV x TK elements, element e: m = e % TMV (fast, coalesced over cases), kk = e / TMV
    for (int e = tid; e < TMV * TK; e += LTHREADS) {
      const int m = e % TMV, kk = e / TMV;
      const int gm = m0 + m, gk = k0 + kk;
      const bool ok = gm < n_act && gk < b;
      const double2* src = ok ? a.U + int64_t(gk) * a.tau + gm : a.U;
      const int ks = kk >> 2, mf = m >> 3;
      cp_async16(&As[stage][(ks * MFT + mf) * 32 + (m & 7) * 4 + (kk & 3)], src, ok);
    }
    // B: K[n][k], element e: kk = e % TK (fast, contiguous in a K row), n = e / TK
    for (int e = tid; e < TN * TK; e += LTHREADS) {
      const int kk = e % TK, n = e / TK;
      const int gn = n0 + n, gk = k0 + kk;
      const bool ok = gn < b && gk < b;
      const double2* src = ok ? a.K + int64_t(gn) * b + gk : a.K;
      const int ks = kk >> 2, nf = n >> 3;
      cp_async16(&Bs[stage][(ks * NF + nf) * 32 + (n & 7) * 4 + (kk & 3)], src, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  // 3M complex products (Gauss, as in the b <= 104 kernel): per fragment pair
  // P1 = sum ar br, P2 = sum ai bi, P3 = sum (ar + ai)(br + bi); re = P1 - P2,
  // im = (P3 - P1) - P2 -- 3 DMMAs instead of 4, at MFR + NFR DADDs per k-step
  double p1[MFR][NFR][2], p2[MFR][NFR][2], p3[MFR][NFR][2];
#pragma unroll
  for (int i = 0; i < MFR; ++i)
#pragma unroll
    for (int j = 0; j < NFR; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) p1[i][j][e] = p2[i][j][e] = p3[i][j][e] = 0.0;

  const int nslabs = (b + TK - 1) / TK;
  // one commit group per slab (empty past the end), so slab s is complete when
  // at most NST - 2 newer groups are pending
#pragma unroll
  for (int st = 0; st < NST - 1; ++st) {
    if (st < nslabs)
      load_slab(st, st * TK);
    else
      asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int s = 0; s < nslabs; ++s) {
    const int stage = s % NST;
    asm volatile("cp.async.wait_group %0;" ::"n"(NST - 2) : "memory");
    __syncthreads();  // slab s visible to all; every thread is done with slab s - 1
    if (s + NST - 1 < nslabs)
      load_slab((s + NST - 1) % NST, (s + NST - 1) * TK);
    else
      asm volatile("cp.async.commit_group;" ::: "memory");
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
      double2 af[MFR], bf[NFR];
      double as[MFR], bs[NFR];
#pragma unroll
      for (int i = 0; i < MFR; ++i) {
        af[i] = As[stage][(ks * MFT + wm * MFR + i) * 32 + lane];
        as[i] = af[i].x + af[i].y;
      }
#pragma unroll
      for (int j = 0; j < NFR; ++j) {
        bf[j] = Bs[stage][(ks * NF + wn * NFR + j) * 32 + lane];
        bs[j] = bf[j].x + bf[j].y;
      }
#pragma unroll
      for (int i = 0; i < MFR; ++i) {
#pragma unroll
        for (int j = 0; j < NFR; ++j) {
          dmma884(p1[i][j][0], p1[i][j][1], af[i].x, bf[j].x);
          dmma884(p2[i][j][0], p2[i][j][1], af[i].y, bf[j].y);
          dmma884(p3[i][j][0], p3[i][j][1], as[i], bs[j]);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  double cr[MFR][NFR][2], ci[MFR][NFR][2];
#pragma unroll
  for (int i = 0; i < MFR; ++i)
#pragma unroll
    for (int j = 0; j < NFR; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        cr[i][j][e] = p1[i][j][e] - p2[i][j][e];
        ci[i][j][e] = (p3[i][j][e] - p1[i][j][e]) - p2[i][j][e];
      }

  // epilogue: V' = acc + W, step test against the (guarded) old iterate, in-place update
  const int* act = a.act[cur];
#pragma unroll
  for (int i = 0; i < MFR; ++i) {
    const int m = m0 + wm * (MFR * 8) + i * 8 + (lane >> 2);
    bool row_bad = false;
    const bool mvalid = m < n_act;
    const int c = mvalid ? act[m] : 0;
#pragma unroll
    for (int j = 0; j < NFR; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = n0 + wn * (NFR * 8) + j * 8 + 2 * (lane & 3) + e;
        if (mvalid && n < b) {
          double2* vp = a.V + n * a.v_node + int64_t(c) * a.v_case;
          double2 old = *vp;
          if (__fma_rn(old.x, old.x, old.y * old.y) < kZeroGuard2) old = make_double2(kZeroGuard, 0.0);
          const double2 w = __ldg(a.W + n);
          const double2 nv = make_double2(cr[i][j][e] + w.x, ci[i][j][e] + w.y);
          const double dr = nv.x - old.x, di = nv.y - old.y;
          if (!(__fma_rn(dr, dr, di * di) < a.tol2)) row_bad = true;
          *vp = nv;
        }
      }
    }
    row_bad |= __shfl_xor_sync(0xffffffffu, row_bad, 1);
    row_bad |= __shfl_xor_sync(0xffffffffu, row_bad, 2);
    if (row_bad && mvalid && (lane & 3) == 0) atomicOr(a.bad + m, 1);
  }
}

// The heavy tail (at most kTailM cases still active): one warp per 8 x 8
// output fragment (8 cases x 8 nodes), no CTA barriers.  Each lane streams the
// single A element (case lane / 4, k = 4 ks + lane % 4) and B element (node
// lane / 4, same k) it feeds to the DMMA through a private ring of kTailDepth
// cp.async stages, so the only serial chain per fragment is the DMMA
// accumulation itself.  The k-steps, the zero padding of k to a multiple of TK,
// the 3M products and the epilogue are those of gemm_kernel: a case's bits do
// not depend on which kernel ran an iteration.
constexpr int kTailDepth = 16;

constexpr int kTailWarps = 4;  // one fragment per SM sub-partition: the DMMA pipe is per SMSP

__global__ void __launch_bounds__(32 * kTailWarps) tail_kernel(LargeArgs a) {
  const int cur = *a.iter & 1;
  const int n_act = a.count[cur];
  if (n_act > kTailM) return;
  const int m0 = blockIdx.y * 8;
  if (m0 >= n_act) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = a.b;
  const int n0 = (blockIdx.x * kTailWarps + warp) * 8;
  if (n0 >= b) return;
  extern __shared__ __align__(16) double2 dyn_smem[];  // [warps][kTailDepth][A, B][32 lanes]
  double2 (*rg)[2][32] = reinterpret_cast<double2 (*)[2][32]>(dyn_smem + size_t(warp) * kTailDepth * 64);
  const int nks = (b + TK - 1) / TK * KSTEPS;  // k-steps of 4, padded like the slabs
  const int mr = m0 + (lane >> 2), nr = n0 + (lane >> 2), kk = lane & 3;
  const bool mok = mr < n_act, nok = nr < b;
  const double2* ua = a.U + mr;
  const double2* kb = a.K + int64_t(nok ? nr : 0) * b;
  auto issue = [&](const int ks) {
    const int k = 4 * ks + kk;
    const bool kok = k < b;
    const int st = ks % kTailDepth;
    cp_async16(&rg[st][0][lane], (mok && kok) ? ua + int64_t(k) * a.tau : a.U, mok && kok);
    cp_async16(&rg[st][1][lane], (nok && kok) ? kb + k : a.K, nok && kok);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll 1
  for (int ks = 0; ks < kTailDepth - 1; ++ks) {
    if (ks < nks)
      issue(ks);
    else
      asm volatile("cp.async.commit_group;" ::: "memory");
  }
  double p1[2] = {0.0, 0.0}, p2[2] = {0.0, 0.0}, p3[2] = {0.0, 0.0};
  // kTailUnroll k-steps per pass (nks is a multiple of KSTEPS = 4): their
  // operands read together, then the DMMA chains; slabs of the next pass
  // refill the stages the previous pass read
  constexpr int kTailUnroll = KSTEPS;
#pragma unroll 1
  for (int ks0 = 0; ks0 < nks; ks0 += kTailUnroll) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kTailDepth - 1 - kTailUnroll) : "memory");
    double2 af[kTailUnroll], bf[kTailUnroll];
#pragma unroll
    for (int u = 0; u < kTailUnroll; ++u) {  // this lane's own copies
      const int st = (ks0 + u) % kTailDepth;
      af[u] = rg[st][0][lane];
      bf[u] = rg[st][1][lane];
    }
#pragma unroll
    for (int u = 0; u < kTailUnroll; ++u) {
      if (ks0 + kTailDepth - 1 + u < nks)
        issue(ks0 + kTailDepth - 1 + u);
      else
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
#pragma unroll
    for (int u = 0; u < kTailUnroll; ++u) {
      const double as = af[u].x + af[u].y, bs = bf[u].x + bf[u].y;
      dmma884(p1[0], p1[1], af[u].x, bf[u].x);
      dmma884(p2[0], p2[1], af[u].y, bf[u].y);
      dmma884(p3[0], p3[1], as, bs);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  // epilogue of gemm_kernel for one fragment
  const int* act = a.act[cur];
  const int m = mr;
  bool row_bad = false;
  const int c = mok ? act[m] : 0;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int n = n0 + 2 * (lane & 3) + e;
    if (mok && n < b) {
      const double cr = p1[e] - p2[e];
      const double ci = (p3[e] - p1[e]) - p2[e];
      double2* vp = a.V + n * a.v_node + int64_t(c) * a.v_case;
      double2 old = *vp;
      if (__fma_rn(old.x, old.x, old.y * old.y) < kZeroGuard2) old = make_double2(kZeroGuard, 0.0);
      const double2 w = __ldg(a.W + n);
      const double2 nv = make_double2(cr + w.x, ci + w.y);
      const double dr = nv.x - old.x, di = nv.y - old.y;
      if (!(__fma_rn(dr, dr, di * di) < a.tol2)) row_bad = true;
      *vp = nv;
    }
  }
  row_bad |= __shfl_xor_sync(0xffffffffu, row_bad, 1);
  row_bad |= __shfl_xor_sync(0xffffffffu, row_bad, 2);
  if (row_bad && mok && (lane & 3) == 0) atomicOr(a.bad + m, 1);
}

// ---- Small active sets as ONE persistent launch -----------------------------
// Once at most kPtMax cases are active (C5: from iteration 14 of 58, 171
// cases falling to 1 over the last 44), an iteration is too little work for
// 64x64 GEMM tiles (few CTAs, each latency-bound) and the remaining
// iterations are mostly launch and latency overhead.  One cooperative launch
// of ceil(b / 8) CTAs runs them all.  CTA x owns output nodes [8x, 8x + 8) for
// every iteration and keeps those 8 rows of K resident in shared memory (one
// bulk copy per row at entry).  The active cases go in groups of 8 (each CTA
// starts at a different group); per group a producer warp streams the
// group's U rows in kPtSK-node slabs through a kPtStages-deep ring
// (cp.async.bulk + mbarriers) and three consumer warps each run ONE of the 3M
// product chains (P1, P2, P3) over the whole k range, so the chain latency
// (26 cycles per dependent DMMA; P3's operand sums make it ~40) rather than
// one warp's issue rate sets the pace.  The first consumer warp finishes the
// fragment exactly as gemm_kernel's epilogue does (same DMMAs, same k-order,
// same zero padding of k to a multiple of TK: a case's bits do not depend on
// which kernel ran an iteration), forms the next iteration's U for its nodes
// (slot-major, double-buffered; a generic -> async proxy fence before the
// other CTAs' bulk reads) and stamps cases that moved >= tol.  A grid barrier
// then lets every CTA rebuild the same ordered active list.  kPtTeams > 1
// runs several groups per CTA at once; measured slower at b = 1,000 (four
// teams: shared-memory operand traffic of unblocked 8x8 fragments, ~60k
// cycles per round of four groups against ~19k per group for one team).
constexpr int kPtSK = 64;                  // k per ring slab (16 k-steps)
constexpr int kPtStages = 8;               // ring depth per team
constexpr int kPtTeams = 1;
constexpr int kPtRow = kPtSK * 16 + 64;    // bytes per slab row; +64 B puts the two rows a quarter-warp reads in different banks
constexpr int kPtStage = 8 * kPtRow;       // the U rows of one group of 8 cases
constexpr int kPtThreads = 32 * 4 * kPtTeams;  // per team: 3 consumer warps + 1 producer warp
static_assert(kPtSK % 4 == 0 && (TK * 4) % kPtSK == 0, "slabs tile the k-slabs of TK");
static_assert(kPtStages <= 32, "parities");
// resident K row stride: nks * 64 bytes rounded to 128, + 64 (bank offset as above)
__host__ __device__ constexpr int pt_krow(int nks) { return (nks * 64 + 127) / 128 * 128 + 64; }

struct PtShared {
  uint64_t full[kPtTeams][kPtStages], empty[kPtTeams][kPtStages], kbar;
  double hand[kPtTeams][2][32][2];
  int warp_sum[kPtThreads / 32];
  int list[kPtMax];
  int n;
};
__host__ __device__ constexpr size_t pt_smem_bytes(int nks) {
  return size_t(8) * pt_krow(nks) + size_t(kPtTeams) * kPtStages * kPtStage + sizeof(PtShared);
}

__device__ __forceinline__ void pt_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void pt_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// all CTAs of the (cooperative) grid; `target` = barriers so far x gridDim.x
__device__ __forceinline__ void pt_grid_sync(uint32_t* gbar, uint32_t target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(gbar, 1u);
    uint32_t v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gbar) : "memory");
      if (v >= target) break;
      __nanosleep(32);
    }
  }
  __syncthreads();
}

// U = conj(s) v / |v|^2 with the zero-voltage guard, bit-identical to prep_kernel
__device__ __forceinline__ double2 pt_u(double2 v, double2 s) {
  double m2 = __fma_rn(v.x, v.x, v.y * v.y);
  if (m2 < kZeroGuard2) {
    v = make_double2(kZeroGuard, 0.0);
    m2 = kZeroGuard * kZeroGuard;
  }
  const double r = 1.0 / m2;
  return make_double2(__fma_rn(s.x, v.x, s.y * v.y) * r, __fma_rn(s.x, v.y, -(s.y * v.x)) * r);
}

template <int W>
__device__ __forceinline__ double pt_operand(double2 v) {
  return W == 0 ? v.x : W == 1 ? v.y : v.x + v.y;
}

// Product chain W of one fragment over all nks k-steps: per slab the operand
// loads issue ahead of its dependent DMMAs; the last slab zeroes operands past
// b (gemm_kernel's zero padding up to a multiple of TK).
template <int W>
__device__ __forceinline__ void pt_chain(const unsigned char* ring, const unsigned char* kres, int krow,
                                         uint64_t* full, uint64_t* empty, uint32_t q, int nslab, int nks, int b,
                                         int lane, double& p0, double& p1) {
  constexpr int KS = kPtSK / 4;
  const int rowa = (lane >> 2) * kPtRow + (lane & 3) * 16;
  const unsigned char* kb0 = kres + (lane >> 2) * krow + (lane & 3) * 16;
  for (int sl = 0; sl < nslab; ++sl, ++q) {
    const int st = q % kPtStages;
    mbar_wait(&full[st], (q / kPtStages) & 1);
    const unsigned char* sa = ring + size_t(st) * kPtStage + rowa;
    const unsigned char* sb = kb0 + sl * kPtSK * 16;
    const int kse = min(KS, nks - sl * KS);
    if (kse == KS && (sl + 1) * kPtSK <= b) {
      double x[KS], y[KS];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        x[ks] = pt_operand<W>(*reinterpret_cast<const double2*>(sa + ks * 64));
        y[ks] = pt_operand<W>(*reinterpret_cast<const double2*>(sb + ks * 64));
      }
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) dmma884(p0, p1, x[ks], y[ks]);
    } else {
#pragma unroll 1
      for (int ks = 0; ks < kse; ++ks) {
        const bool kok = sl * kPtSK + 4 * ks + (lane & 3) < b;
        double2 av = *reinterpret_cast<const double2*>(sa + ks * 64);
        double2 bv = *reinterpret_cast<const double2*>(sb + ks * 64);
        if (!kok) av = bv = make_double2(0.0, 0.0);
        dmma884(p0, p1, pt_operand<W>(av), pt_operand<W>(bv));
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
}

__global__ void __launch_bounds__(kPtThreads, 1) tail_persistent_kernel(LargeArgs a) {
  const int it0 = *a.iter, cur = it0 & 1;
  const int n_entry = a.count[cur];
  if (n_entry == 0 || n_entry > kPtMax) return;
  const int b = a.b;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int team = warp < 3 * kPtTeams ? warp / 3 : warp - 3 * kPtTeams, role = warp < 3 * kPtTeams ? warp % 3 : 3;
  const int n0 = blockIdx.x * 8;
  const int nks = (b + TK - 1) / TK * KSTEPS;  // k-steps of 4, padded like gemm_kernel's slabs
  const int nslab = (nks * 4 + kPtSK - 1) / kPtSK;
  const int nrows = min(8, b - n0);
  const int krow = pt_krow(nks);
  extern __shared__ __align__(128) unsigned char pt_smem[];
  unsigned char* kres = pt_smem;                                    // [8][krow]: this CTA's K rows
  unsigned char* rings = pt_smem + 8 * krow;                        // [team][stage][8][kPtRow]: U slabs
  PtShared& sh = *reinterpret_cast<PtShared*>(rings + size_t(kPtTeams) * kPtStages * kPtStage);
  unsigned char* ring = rings + size_t(team) * kPtStages * kPtStage;
  const int* act = a.act[cur];  // slot -> case, fixed for the whole launch
  const size_t uplane = size_t(kPtMax) * b;

  if (tid == 0) {
    for (int t = 0; t < kPtTeams; ++t)
      for (int i = 0; i < kPtStages; ++i) {
        mbar_init(&sh.full[t][i], 1);
        mbar_init(&sh.empty[t][i], 3);
      }
    mbar_init(&sh.kbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    sh.n = n_entry;
    pt_expect_tx(&sh.kbar, uint32_t(nrows) * b * 16u);
    for (int r = 0; r < nrows; ++r) pt_bulk(kres + r * krow, a.K + int64_t(n0 + r) * b, uint32_t(b) * 16u, &sh.kbar);
  }
  for (int q = tid; q < n_entry; q += kPtThreads) sh.list[q] = q;
  // zero K past b and the rows past the feeder's last node (gemm_kernel's zero fill)
  for (int e = tid; e < 8 * (krow / 16); e += kPtThreads) {
    const int r = e / (krow / 16), k = e - r * (krow / 16);
    if (r >= nrows || k >= b) *reinterpret_cast<double2*>(kres + r * krow + k * 16) = make_double2(0.0, 0.0);
  }
  // U of the entry iteration for this CTA's nodes (prep_kernel's values, slot-major)
  for (int e = tid; e < nrows * n_entry; e += kPtThreads) {
    const int r = e / n_entry, q = e - r * n_entry, n = n0 + r, c = act[q];
    a.U2[size_t(q) * b + n] =
        pt_u(a.V[n * a.v_node + int64_t(c) * a.v_case], __ldg(a.S + n * a.s_node + int64_t(c) * a.s_case));
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
  uint32_t nbar = 1;
  pt_grid_sync(a.gbar, nbar * gridDim.x);

  uint32_t q_ring = 0;  // this team's ring slabs issued (producer) / consumed (consumers)
  bool k_ready = false;
  for (int it = it0;; ++it) {
    const int n = sh.n;
    const int par = (it - it0) & 1;
    const double2* usrc = a.U2 + par * uplane;
    const int ngroups = (n + 7) / 8;
    if (role == 3) {
      // producer of this team: its groups' U rows, slab by slab.  cp.async
      // (generic proxy) because other CTAs wrote U with plain stores.
      if (lane == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // other CTAs' U stores -> bulk reads
        for (int gi = team; gi < ngroups; gi += kPtTeams) {
          // CTAs walk the groups from different starting points, so that the
          // 125 CTAs do not all read the same U rows at the same time
          const int g = (gi + blockIdx.x) % ngroups;
          const int g0 = g * 8, gcnt = min(8, n - g0);
          for (int sl = 0; sl < nslab; ++sl, ++q_ring) {
            const int st = q_ring % kPtStages;
            mbar_wait(&sh.empty[team][st], ((q_ring / kPtStages) & 1) ^ 1);
            const int k0 = sl * kPtSK;
            const uint32_t bytes = uint32_t(min(kPtSK, b - k0)) * 16u;
            unsigned char* stage = ring + size_t(st) * kPtStage;
            pt_expect_tx(&sh.full[team][st], bytes * uint32_t(gcnt));
            for (int m = 0; m < gcnt; ++m)
              pt_bulk(stage + m * kPtRow, usrc + size_t(sh.list[g0 + m]) * b + k0, bytes, &sh.full[team][st]);
          }
        }
      }
      __syncwarp();
    } else {
      if (!k_ready) {
        mbar_wait(&sh.kbar, 0);
        k_ready = true;
      }
      for (int gi = team; gi < ngroups; gi += kPtTeams) {
        // CTAs walk the groups from different starting points, so that the
        // 125 CTAs do not all read the same U rows at the same time
        const int g = (gi + blockIdx.x) % ngroups;
        const int g0 = g * 8, gcnt = min(8, n - g0);
        // the epilogue's operands, loaded ahead of the chain
        const int m = lane >> 2;
        const bool mok = m < gcnt;
        const int slot = mok ? sh.list[g0 + m] : 0;
        const int c = act[slot];
        double2 vold[2], wv[2], sv[2];
        if (role == 0) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int nn = 2 * (lane & 3) + e, nd = n0 + nn;
            if (mok && nn < nrows) {
              vold[e] = a.V[nd * a.v_node + int64_t(c) * a.v_case];
              wv[e] = __ldg(a.W + nd);
              sv[e] = __ldg(a.S + nd * a.s_node + int64_t(c) * a.s_case);
            }
          }
        }
        double p0 = 0.0, p1 = 0.0;
        if (role == 0)
          pt_chain<0>(ring, kres, krow, sh.full[team], sh.empty[team], q_ring, nslab, nks, b, lane, p0, p1);
        else if (role == 1)
          pt_chain<1>(ring, kres, krow, sh.full[team], sh.empty[team], q_ring, nslab, nks, b, lane, p0, p1);
        else
          pt_chain<2>(ring, kres, krow, sh.full[team], sh.empty[team], q_ring, nslab, nks, b, lane, p0, p1);
        q_ring += nslab;
        if (role > 0) {
          sh.hand[team][role - 1][lane][0] = p0;
          sh.hand[team][role - 1][lane][1] = p1;
        }
        named_bar(1 + team, 96);
        if (role == 0) {
          // gemm_kernel's epilogue for this fragment, plus the next U and the stamp
          bool row_bad = false;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int nn = 2 * (lane & 3) + e, nd = n0 + nn;
            if (mok && nn < nrows) {
              const double q2 = sh.hand[team][0][lane][e], q3 = sh.hand[team][1][lane][e];
              const double q1 = e == 0 ? p0 : p1;
              const double cr = q1 - q2;
              const double ci = (q3 - q1) - q2;
              double2 old = vold[e];
              if (__fma_rn(old.x, old.x, old.y * old.y) < kZeroGuard2) old = make_double2(kZeroGuard, 0.0);
              const double2 nv = make_double2(cr + wv[e].x, ci + wv[e].y);
              const double dr = nv.x - old.x, di = nv.y - old.y;
              if (!(__fma_rn(dr, dr, di * di) < a.tol2)) row_bad = true;
              a.V[nd * a.v_node + int64_t(c) * a.v_case] = nv;
              a.U2[(par ^ 1) * uplane + size_t(slot) * b + nd] = pt_u(nv, sv[e]);
            }
          }
          row_bad |= __shfl_xor_sync(0xffffffffu, row_bad, 1);
          row_bad |= __shfl_xor_sync(0xffffffffu, row_bad, 2);
          if (row_bad && mok && (lane & 3) == 0) a.stamp[slot] = it + 1;
          asm volatile("fence.proxy.async.global;" ::: "memory");  // U stores -> other CTAs' bulk reads
        }
        named_bar(1 + team, 96);  // hand[] free for the team's next group
      }
    }
    ++nbar;
    pt_grid_sync(a.gbar, nbar * gridDim.x);
    // every CTA rebuilds the same ordered list from the stamps (CTA 0 counts the update)
    int nn = 0;
    for (int base = 0; base < n; base += kPtThreads) {
      const int q = base + tid;
      int slot = 0;
      bool keep = false;
      if (q < n) {
        slot = sh.list[q];
        if (blockIdx.x == 0) a.iters[act[slot]] = it + 1;
        keep = __ldcg(a.stamp + slot) == it + 1 && it + 1 < a.max_iter;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) sh.warp_sum[warp] = __popc(bal);
      __syncthreads();  // warp counts ready; every read of this round's slots done
      int before = nn;
      for (int w = 0; w < warp; ++w) before += sh.warp_sum[w];
      int total = nn;
      for (int w = 0; w < kPtThreads / 32; ++w) total += sh.warp_sum[w];
      if (keep) sh.list[before + __popc(bal & ((1u << lane) - 1u))] = slot;
      nn = total;
      __syncthreads();  // warp_sum reusable
    }
    if (nn == 0) break;
    if (tid == 0) sh.n = nn;
    __syncthreads();
  }
  // nothing is in flight (every issued slab was consumed); retire the host loop
  if (blockIdx.x == 0 && tid == 0) {
    a.count[0] = 0;
    a.count[1] = 0;
  }
}

__global__ void compact_kernel(LargeArgs a) {
  const int cur = *a.iter & 1;
  const int n_act = a.count[cur];
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_act) return;
  const int c = a.act[cur][p];
  const int it = a.iters[c] + 1;
  a.iters[c] = it;
  if (a.bad[p] && it < a.max_iter) {
    const int q = atomicAdd(a.count + (cur ^ 1), 1);
    a.act[cur ^ 1][q] = c;
  }
}

// Advance the device-resident iteration; with a device-side loop, decide
// whether its body (prep, gemm, [tail,] compact, step) runs again.
__global__ void step_kernel(LargeArgs a, cudaGraphConditionalHandle loop) {
  const int it = *a.iter;
  *a.iter = it + 1;
  if (loop) cudaGraphSetConditional(loop, (a.count[(it & 1) ^ 1] > a.loop_min && it + 1 < a.max_iter) ? 1u : 0u);
}

}  // namespace
}  // namespace tpf

using namespace tpf;

namespace {
// Executable graphs of eager calls, released once their launch has completed
// (checked at this thread's next call; the rest at thread exit).
struct LaunchedGraph {
  cudaGraphExec_t exec;
  cudaEvent_t done;
};
struct GraphReaper {
  std::vector<LaunchedGraph> items;
  void reap(bool all) {
    size_t keep = 0;
    for (auto& x : items) {
      cudaError_t q = all ? cudaEventSynchronize(x.done) : cudaEventQuery(x.done);
      if (q == cudaErrorNotReady) {
        cudaGetLastError();  // not an error: still running
        items[keep++] = x;
        continue;
      }
      cudaGraphExecDestroy(x.exec);
      cudaEventDestroy(x.done);
    }
    items.resize(keep);
  }
  ~GraphReaper() { reap(true); }
};
thread_local GraphReaper g_reaper;
}  // namespace

extern "C" size_t tpf_dense_large_workspace_bytes(int64_t tau, int32_t b) {
  const size_t t = size_t(tau > 0 ? tau : 1);
  return 256 + 3 * t * 4 + 64 + t * size_t(b) * 16 + 2 * size_t(kPtMax) * b * 16 + size_t(kPtMax) * 4 + 2048;
}

extern "C" int tpf_dense_fpi_large_c128(int64_t tau, int32_t b, const double* S, int64_t s_node_stride,
                                        int64_t s_case_stride, const double* K, const double* W, double v_flat_re,
                                        double v_flat_im, double tol, int32_t max_iter, double* V,
                                        int64_t v_node_stride, int64_t v_case_stride, int32_t* iters,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  if (tau < 0 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_dense_fpi_large_c128: need tau >= 0 and b >= 1");
  if (tau > INT_MAX / 2) return set_error(TPF_ERR_INVALID, "tpf_dense_fpi_large_c128: tau too large; shard it");
  if (!(tol > 0.0)) return set_error(TPF_ERR_INVALID, "tolerance must be positive");
  if (max_iter < 1) return set_error(TPF_ERR_INVALID, "max_iterations must be >= 1");
  if (tau == 0) return TPF_OK;
  if (!S || !K || !W || !V || !iters || !workspace)
    return set_error(TPF_ERR_INVALID, "tpf_dense_fpi_large_c128: null pointer");
  if (workspace_bytes < tpf_dense_large_workspace_bytes(tau, b))
    return set_error(TPF_ERR_INVALID, "tpf_dense_fpi_large_c128: workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LargeArgs a;
  a.tau = tau;
  a.b = b;
  a.S = reinterpret_cast<const double2*>(S);
  a.s_node = s_node_stride;
  a.s_case = s_case_stride;
  a.K = reinterpret_cast<const double2*>(K);
  a.W = reinterpret_cast<const double2*>(W);
  a.v_flat = make_double2(v_flat_re, v_flat_im);
  a.tol2 = tol * tol;
  a.max_iter = max_iter;
  a.V = reinterpret_cast<double2*>(V);
  a.v_node = v_node_stride;
  a.v_case = v_case_stride;
  a.iters = iters;
  char* w = static_cast<char*>(workspace);
  auto take = [&](size_t n) {
    char* p = w;
    w += (n + 255) / 256 * 256;
    return p;
  };
  a.count = reinterpret_cast<int32_t*>(take(64));
  a.act[0] = reinterpret_cast<int32_t*>(take(size_t(tau) * 4));
  a.act[1] = reinterpret_cast<int32_t*>(take(size_t(tau) * 4));
  a.bad = reinterpret_cast<int32_t*>(take(size_t(tau) * 4));
  a.U = reinterpret_cast<double2*>(take(size_t(tau) * b * 16));
  a.handoff = kTailM;
  a.U2 = reinterpret_cast<double2*>(take(2 * size_t(kPtMax) * b * 16));
  a.stamp = reinterpret_cast<int32_t*>(take(kPtMax * 4));
  a.gbar = reinterpret_cast<uint32_t*>(a.count + 8);
  a.iter = a.count + 2;
  if (size_t(w - static_cast<char*>(workspace)) > workspace_bytes)
    return set_error(TPF_ERR_INVALID, "tpf_dense_fpi_large_c128: workspace too small");

  const unsigned tb = unsigned((tau + 255) / 256);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const dim3 ggrid(unsigned((tau + TM - 1) / TM), unsigned((b + TN - 1) / TN));
  const unsigned pgrid = unsigned(sms) * 8;
  constexpr int kBulkStages = 2;
  const int gsmem = int(kBulkStages * KSTEPS * (MF + NF) * 32 * sizeof(double2));
  cudaError_t aerr = cudaFuncSetAttribute(gemm_kernel<TM, 2, kBulkStages>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, gsmem);
  if (aerr != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(gemm_kernel)", aerr);
  // partial active sets (kMidM or fewer cases): 32-case tiles, twice the CTAs
  const int msmem = int(kBulkStages * KSTEPS * (32 / 8 + NF) * 32 * sizeof(double2));
  aerr = cudaFuncSetAttribute(gemm_kernel<32, 2, kBulkStages>, cudaFuncAttributeMaxDynamicSharedMemorySize, msmem);
  if (aerr != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(gemm_kernel<32>)", aerr);
  const dim3 mgrid(unsigned((std::min<int64_t>(tau, kMidM) + 31) / 32), unsigned((b + TN - 1) / TN));
  // node groups fastest: the active fragments (cases m0 < n_act) of one
  // iteration spread over the SMs
  const dim3 tgrid(unsigned((b + 8 * kTailWarps - 1) / (8 * kTailWarps)), unsigned(kTailM / 8));
  const int tsmem = int(kTailWarps * kTailDepth * 64 * sizeof(double2));
  aerr = cudaFuncSetAttribute(tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem);
  if (aerr != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(tail_kernel)", aerr);
  // the persistent kernel needs its ceil(b / 8) CTAs co-resident (one per SM:
  // b <= 1,184 on a B200) and its shared memory; otherwise gemm_kernel runs
  // down to kTailM active cases and tail_kernel each iteration below that
  const int pt_ctas = (b + 7) / 8;
  const size_t ptsmem = pt_smem_bytes((b + TK - 1) / TK * KSTEPS);
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  bool persistent = std::getenv("TPF_LARGE_TAIL_LAUNCHES") == nullptr && ptsmem <= size_t(smem_optin);
  if (persistent) {
    aerr = cudaFuncSetAttribute(tail_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ptsmem));
    if (aerr != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(tail_persistent_kernel)", aerr);
    int per_sm = 0, coop = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tail_persistent_kernel, kPtThreads, ptsmem);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    persistent = coop && per_sm >= 1 && pt_ctas <= per_sm * sms;
  }
  a.handoff = persistent ? kPtMax : kTailM;
  a.loop_min = persistent ? kPtMax : 0;

  // The iteration loop runs on the device: a CUDA graph WHILE node around
  // prep -> gemm -> [tail ->] compact -> step, whose condition step_kernel
  // sets (more than loop_min cases active, iterations left), then the
  // persistent kernel once.  Inside a stream capture the nodes join the
  // captured graph; otherwise a graph is built, launched and released.
  // TPF_LARGE_HOST_LOOP=1 (or a graph API failure before anything was
  // enqueued) launches the max_iter iterations from the host instead, each
  // kernel exiting early once its range is empty.
  const bool want_graph = std::getenv("TPF_LARGE_HOST_LOOP") == nullptr;
  if (want_graph) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* cdeps = nullptr;
    size_t ncdeps = 0;
    cudaError_t e = cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &cdeps, &ncdeps);
    if (e != cudaSuccess) return set_cuda_error("cudaStreamGetCaptureInfo", e);
    const bool captured = cs == cudaStreamCaptureStatusActive;
    std::vector<cudaGraphNode_t> deps(cdeps, cdeps + (captured ? ncdeps : 0));
    if (!captured) {
      e = cudaGraphCreate(&g, 0);
      if (e != cudaSuccess) return set_cuda_error("cudaGraphCreate", e);
    }
    cudaGraphConditionalHandle loop = 0;
    auto fail = [&](const char* what, cudaError_t err) {
      if (!captured && g) cudaGraphDestroy(g);
      return set_cuda_error(what, err);
    };
    e = cudaGraphConditionalHandleCreate(&loop, g, 0, 0);
    if (e != cudaSuccess) return fail("cudaGraphConditionalHandleCreate", e);
    auto add_kernel = [&](cudaGraph_t graph, std::vector<cudaGraphNode_t>& after, const void* fn, dim3 grid,
                          dim3 block, size_t smem, void** args, bool coop, cudaGraphNode_t* out) {
      cudaKernelNodeParams kp = {};
      kp.func = const_cast<void*>(fn);
      kp.gridDim = grid;
      kp.blockDim = block;
      kp.sharedMemBytes = unsigned(smem);
      kp.kernelParams = args;
      cudaError_t r = cudaGraphAddKernelNode(out, graph, after.data(), after.size(), &kp);
      if (r == cudaSuccess && coop) {
        cudaLaunchAttributeValue v = {};
        v.cooperative = 1;
        r = cudaGraphKernelNodeSetAttribute(*out, cudaLaunchAttributeCooperative, &v);
      }
      if (r == cudaSuccess) after.assign(1, *out);
      return r;
    };
    cudaGraphNode_t node = nullptr;
    void* init_args[] = {&a, &loop};
    e = add_kernel(g, deps, reinterpret_cast<const void*>(init_kernel), dim3(tb), dim3(256), 0, init_args, false, &node);
    if (e != cudaSuccess) return fail("graph: init_kernel", e);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = loop;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    e = cudaGraphAddNode(&node, g, deps.data(), deps.size(), &cp);
    if (e != cudaSuccess) return fail("graph: while node", e);
    deps.assign(1, node);
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    std::vector<cudaGraphNode_t> bdeps;
    cudaGraphNode_t bn = nullptr;
    void* a_args[] = {&a};
    void* step_args[] = {&a, &loop};
    e = add_kernel(body, bdeps, reinterpret_cast<const void*>(prep_kernel), dim3(pgrid), dim3(256), 0, a_args, false, &bn);
    if (e == cudaSuccess)
      e = add_kernel(body, bdeps, reinterpret_cast<const void*>(gemm_kernel<TM, 2, kBulkStages>), ggrid,
                     dim3(LTHREADS), size_t(gsmem), a_args, false, &bn);
    if (e == cudaSuccess)
      e = add_kernel(body, bdeps, reinterpret_cast<const void*>(gemm_kernel<32, 2, kBulkStages>), mgrid,
                     dim3(LTHREADS), size_t(msmem), a_args, false, &bn);
    if (e == cudaSuccess && !persistent)
      e = add_kernel(body, bdeps, reinterpret_cast<const void*>(tail_kernel), tgrid, dim3(32 * kTailWarps),
                     size_t(tsmem), a_args, false, &bn);
    if (e == cudaSuccess)
      e = add_kernel(body, bdeps, reinterpret_cast<const void*>(compact_kernel), dim3(tb), dim3(256), 0, a_args, false, &bn);
    if (e == cudaSuccess)
      e = add_kernel(body, bdeps, reinterpret_cast<const void*>(step_kernel), dim3(1), dim3(1), 0, step_args, false, &bn);
    if (e != cudaSuccess) return fail("graph: loop body", e);
    if (persistent) {
      e = add_kernel(g, deps, reinterpret_cast<const void*>(tail_persistent_kernel), dim3(pt_ctas), dim3(kPtThreads),
                     ptsmem, a_args, true, &node);
      if (e != cudaSuccess) return fail("graph: tail_persistent_kernel", e);
    }
    if (captured) {
      e = cudaStreamUpdateCaptureDependencies(st, deps.data(), deps.size(), cudaStreamSetCaptureDependencies);
      if (e != cudaSuccess) return set_cuda_error("cudaStreamUpdateCaptureDependencies", e);
      return TPF_OK;
    }
    g_reaper.reap(false);
    cudaGraphExec_t ge = nullptr;
    e = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);  // the executable graph does not depend on it
    if (e != cudaSuccess) return set_cuda_error("cudaGraphInstantiate", e);
    e = cudaGraphLaunch(ge, st);
    cudaEvent_t done = nullptr;
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(done, st);
    if (e != cudaSuccess) {
      if (done) cudaEventDestroy(done);
      cudaStreamSynchronize(st);
      cudaGraphExecDestroy(ge);
      return set_cuda_error("cudaGraphLaunch", e);
    }
    g_reaper.items.push_back({ge, done});  // released after the launch completes
    return TPF_OK;
  }

  cudaGraphConditionalHandle none = 0;
  init_kernel<<<tb, 256, 0, st>>>(a, none);
  for (int it = 0; it < max_iter; ++it) {
    prep_kernel<<<pgrid, 256, 0, st>>>(a);
    gemm_kernel<TM, 2, kBulkStages><<<ggrid, LTHREADS, gsmem, st>>>(a);
    gemm_kernel<32, 2, kBulkStages><<<mgrid, LTHREADS, msmem, st>>>(a);
    if (persistent) {
      void* args[] = {&a};
      aerr = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(tail_persistent_kernel), dim3(pt_ctas),
                                         dim3(kPtThreads), args, ptsmem, st);
      if (aerr != cudaSuccess) return set_cuda_error("cudaLaunchCooperativeKernel(tail_persistent_kernel)", aerr);
    } else {
      tail_kernel<<<tgrid, 32 * kTailWarps, tsmem, st>>>(a);
    }
    compact_kernel<<<tb, 256, 0, st>>>(a);
    step_kernel<<<1, 1, 0, st>>>(a, none);
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(dense large)", err);
  return TPF_OK;
}
