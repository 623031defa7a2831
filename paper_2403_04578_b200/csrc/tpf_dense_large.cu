// Dense Tensor Power Flow for feeders too large for a shared-memory-resident K
// (b > 104; config C5 is b = 1,000, K = 16 MB, which lives in the 126 MB L2).
//
// Same update as tpf_dense.cu (dense.py:114-126), organised as an
// iteration-synchronous loop over a compacted ACTIVE SET of cases, because
// near voltage collapse the per-case iteration counts are heavy-tailed
// (C5: batch 58 iterations, per-case mean 10.4): every iteration only the
// still-unconverged cases enter the GEMM.
//
// Per iteration (three launches, all early-exit when the active set is empty):
//   prep    U[k, a] = S*_{k,c} / conj(v_{k,c}) for active case c = act[a]
//           (zero-voltage guard), node-major so the writes coalesce over a;
//   gemm    V'[a, n] = W[n] + sum_k U[k, a] K[n, k] on FP64 tensor cores:
//           64x64 complex CTA tiles, 16-node k-slabs double-buffered through
//           shared memory with cp.async (zero-filled at the edges), 8 warps of
//           32x16 complex each, 3 real DMMA.8x8x4 per complex fragment (3M); the
//           epilogue reads the old iterate, writes the new one in place and
//           flags the case if any |dv|^2 >= tol^2 (or non-finite);
//   compact count the update, keep flagged cases below max_iter.
// The k-order of every dot product is fixed, so a case's bits do not depend
// on its position in the active set (permutation / shard invariance).
#include <climits>

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
};

__global__ void init_kernel(LargeArgs a) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j == 0) {
    a.count[0] = int(a.tau);
    a.count[1] = 0;
  }
  if (j >= a.tau) return;
  a.act[0][j] = int(j);
  a.iters[j] = 0;
  for (int i = 0; i < a.b; ++i) a.V[i * a.v_node + j * a.v_case] = a.v_flat;
}

__global__ void prep_kernel(LargeArgs a, int cur) {
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
__global__ void __launch_bounds__(LTHREADS) gemm_kernel(LargeArgs a, int cur) {
  constexpr int WN = 8 / WM;
  constexpr int MFR = TMV / WM / 8, NFR = TN / WN / 8;  // fragments per warp tile
  constexpr int MFT = TMV / 8;                         // m-fragments per CTA tile
  const int n_act = a.count[cur];
  if (TMV == 8 ? n_act > kTailM : n_act <= kTailM) return;
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

__global__ void __launch_bounds__(32 * kTailWarps) tail_kernel(LargeArgs a, int cur) {
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

__global__ void compact_kernel(LargeArgs a, int cur) {
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

}  // namespace
}  // namespace tpf

using namespace tpf;

extern "C" size_t tpf_dense_large_workspace_bytes(int64_t tau, int32_t b) {
  const size_t t = size_t(tau > 0 ? tau : 1);
  return 256 + 3 * t * 4 + 64 + t * size_t(b) * 16 + 1024;
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
  if (size_t(w - static_cast<char*>(workspace)) > workspace_bytes)
    return set_error(TPF_ERR_INVALID, "tpf_dense_fpi_large_c128: workspace too small");

  const unsigned tb = unsigned((tau + 255) / 256);
  init_kernel<<<tb, 256, 0, st>>>(a);
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
  // node groups fastest: the active fragments (cases m0 < n_act) of one
  // iteration spread over the SMs
  const dim3 tgrid(unsigned((b + 8 * kTailWarps - 1) / (8 * kTailWarps)), unsigned(kTailM / 8));
  const int tsmem = int(kTailWarps * kTailDepth * 64 * sizeof(double2));
  aerr = cudaFuncSetAttribute(tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem);
  if (aerr != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(tail_kernel)", aerr);
  for (int it = 0; it < max_iter; ++it) {
    const int cur = it & 1;
    prep_kernel<<<pgrid, 256, 0, st>>>(a, cur);
    gemm_kernel<TM, 2, kBulkStages><<<ggrid, LTHREADS, gsmem, st>>>(a, cur);
    tail_kernel<<<tgrid, 32 * kTailWarps, tsmem, st>>>(a, cur);
    compact_kernel<<<tb, 256, 0, st>>>(a, cur);
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(dense large)", err);
  return TPF_OK;
}
