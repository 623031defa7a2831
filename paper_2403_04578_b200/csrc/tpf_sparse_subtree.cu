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
// the up-sweep value z in registers (compile-time slot index).  Shared
// memory: the sweep exchange vector X (by position), the per-position
// structure, the child lists and Proot.  Per case the loads arrive by TMA
// (2-D tensor copy of one column of the node-major S, or a 1-D bulk copy of a
// case-major column) into X in original node order, the next case's column is
// prefetched into L2 by TMA while this one iterates, and V leaves the same way
// (TMA store from X).  The residual post-check (fpi.py:221-240) is fused: the
// final V is in X in original node order, Y_dd's rows come as ELL per position.
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
constexpr int kSubThreads = 32 * kSubWarps;
constexpr int kParentNone = -32768;
constexpr int kMaxRW = 16;

struct SubArgs {
  int64_t tau;
  int b, NS, RMAX, RW, P, xcap, nkids;
  int mode;      // 0: node-major S / V (2-D TMA), 1: case-major (1-D bulk)
  int nbox, boxrows;
  const double2* S;
  int64_t s_case;  // mode 1: case stride (complex elements)
  double2* V;
  int64_t v_case;
  const int2* pinfo;      // [P]
  const uint16_t* kids;   // [nkids]
  const double2* coef;    // [3][P]: g, 1/U[m,m], src
  const int32_t* ell_col; // [RW][P]
  const double2* ell_val; // [RW][P]
  int32_t* iters;
  double* resid;          // or null
  unsigned long long* counter;
  double2 v_flat;
  double tol2;
  int max_iter;
  int jD[kSubWarps];
  unsigned sync[kSubWarps];
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

template <int NSL>
__global__ void __launch_bounds__(kSubThreads, 1)
    sparse_subtree_kernel(const __grid_constant__ SubArgs a, const __grid_constant__ CUtensorMap tmS,
                          const __grid_constant__ CUtensorMap tmV) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double2* X = reinterpret_cast<double2*>(smem_raw);                 // [xcap]
  int2* PI = reinterpret_cast<int2*>(X + a.xcap);                    // [P]
  double2* PR = reinterpret_cast<double2*>(PI + a.P);                // [2][W * RMAX * 32]
  uint16_t* KD = reinterpret_cast<uint16_t*>(PR + 2 * kSubWarps * a.RMAX * 32);  // [nkids]
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ int s_case, s_next;
  __shared__ double s_red[kSubWarps];
  __shared__ uint32_t s_tmem;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int P = a.P, NS = a.NS;
  for (int i = tid; i < P; i += kSubThreads) PI[i] = __ldg(a.pinfo + i);
  for (int i = tid; i < a.nkids; i += kSubThreads) KD[i] = __ldg(a.kids + i);
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  // TMEM: lane quadrant warp % 4, column group warp / 4 (3 groups of 8 * NSL <= 168 columns)
  const uint32_t tm = s_tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * 8 * NSL);
  const uint32_t tm_v = tm, tm_s = tm + 4 * NSL;
  const int base = warp * NSL * 32 + lane;  // position of slot j: base + 32 j
  const int topbase = (warp * NSL + NS) * 32;
  const int jD = a.jD[warp];
  const unsigned syncm = a.sync[warp];
  const int RR = kSubWarps * a.RMAX * 32;
  unsigned vmask = 0;  // slots holding a node for this thread
#pragma unroll
  for (int j = 0; j < NSL; ++j)
    if ((uint32_t(PI[base + 32 * j].y) >> 16) != 0xFFFFu) vmask |= 1u << j;
  const double2* cg = a.coef;
  const double2* cu = a.coef + P;
  const double2* cs_src = a.coef + 2 * P;
  const uint32_t in_bytes =
      a.mode == 0 ? uint32_t(a.nbox) * uint32_t(a.boxrows) * 16u : uint32_t(a.b) * 16u;

  auto claim = [&]() {
    const unsigned long long c = atomicAdd(a.counter, 1ull);
    return c < (unsigned long long)a.tau ? int(c) : -1;
  };
  auto child_val = [&](unsigned code, int par) -> double2 {
    if (code >= 0xC000u) return PR[par * RR + int(code - 0xC000u)];
    if (code >= 0x8000u) return X[topbase + int(code - 0x8000u)];
    return X[code];
  };
  if (tid == 0) {
    s_case = claim();
    s_next = s_case >= 0 ? claim() : -1;
  }
  __syncthreads();
  uint32_t phase = 0;
  double2 zr[NSL];

  for (;;) {
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
#pragma unroll
    for (int j = 0; j < NSL; ++j) {
      double2 s = make_double2(0.0, 0.0);
      if (vmask >> j & 1u) s = X[uint32_t(PI[base + 32 * j].y) >> 16];
      tmem_st2(tm_s + 4 * j, s);
      tmem_st2(tm_v + 4 * j, a.v_flat);  // flat start (dense.py:155)
    }
    tmem_wait_st();
    __syncthreads();  // X is free for the sweeps

    int it = 0;
    bool small = false;
    for (;;) {
      const int par = it & 1;
      // ---- up-sweep: slots 0..NS-1 (subtrees), barrier, NS..NSL-1 (top) ----
#pragma unroll
      for (int j = 0; j < NSL; ++j) {
        if (j == NS) {
          // the previous iteration's step test, AND over the CTA (false at it = 0)
          if (__syncthreads_and(small)) goto converged;
        }
        {
          D2 vv, ss;
          tmem_ld2(tm_v + 4 * j, vv);
          tmem_ld2(tm_s + 4 * j, ss);
          tmem_wait_ld();
          if (vmask >> j & 1u) {
            const int p = base + 32 * j;
            const int2 pi = PI[p];
            const int pc = int(int16_t(pi.x & 0xFFFF));
            double2 v = vv.get();
            const double2 sl = ss.get();
            double m2 = __fma_rn(v.x, v.x, v.y * v.y);
            if (m2 < kZeroGuard2) {  // fpi.py:39-41
              v = make_double2(kZeroGuard, 0.0);
              m2 = kZeroGuard * kZeroGuard;
            }
            const double r = rcp_nr(m2);
            const double2 src = pc == kParentNone ? __ldg(cs_src + p) : make_double2(0.0, 0.0);
            // r_m = -(s*/conj(v) + src),  s*/conj(v) = conj(s) v / |v|^2
            double2 z = make_double2(-(__fma_rn(sl.x, v.x, sl.y * v.y) * r + src.x),
                                     -(__fma_rn(sl.x, v.y, -(sl.y * v.x)) * r + src.y));
            const int kf = int(uint32_t(pi.x) >> 16), kc = pi.y & 0xFF;
            for (int k = 0; k < kc; ++k) {
              const double2 pcv = child_val(KD[kf + k], par);
              z.x -= pcv.x;
              z.y -= pcv.y;
            }
            zr[j] = z;
            const double2 P_m = cmul_s(__ldg(cg + p), z);
            X[p] = P_m;
            if (j < NS && j >= jD && pc < 0 && pc != kParentNone)
              PR[par * RR + (warp * a.RMAX + j - jD) * 32 + lane] = P_m;
          }
        }
        if (syncm >> j & 1u) __syncwarp();
      }
      // ---- down-sweep: top slots (root level first), then subtrees, leaves last ----
      small = true;
#pragma unroll
      for (int j = NSL - 1; j >= 0; --j) {
        if (j < NSL - 1 && (syncm >> j & 1u)) __syncwarp();
        if (j == NS - 1) __syncwarp();
        D2 vv;
        tmem_ld2(tm_v + 4 * j, vv);
        tmem_wait_ld();
        double2 v = vv.get();
        double2 w = v;
        if (vmask >> j & 1u) {
          const int p = base + 32 * j;
          const int pc = int(int16_t(PI[p].x & 0xFFFF));
          w = cmul_s(zr[j], __ldg(cu + p));
          if (pc != kParentNone) {
            const double2 wp = pc < 0 ? X[topbase + (-1 - pc)] : X[pc];
            w = cfma_sub_s(w, __ldg(cg + p), wp);
          }
          X[p] = w;
          if (__fma_rn(v.x, v.x, v.y * v.y) < kZeroGuard2) v = make_double2(kZeroGuard, 0.0);
          const double dr = w.x - v.x, di = w.y - v.y;
          if (!(__fma_rn(dr, dr, di * di) < a.tol2)) small = false;  // NaN never passes
        }
        tmem_st2(tm_v + 4 * j, w);
      }
      tmem_wait_st();
      ++it;
      if (it == a.max_iter) break;
    }
  converged:
    __syncthreads();  // every warp is done with X (the cap path leaves without a barrier)
    // ---- retire: V into X in original node order (top nodes: warp 0's copy) ----
#pragma unroll
    for (int j = 0; j < NSL; ++j) {
      D2 vv;
      tmem_ld2(tm_v + 4 * j, vv);
      tmem_wait_ld();
      if ((vmask >> j & 1u) && (j < NS || warp == 0)) X[uint32_t(PI[base + 32 * j].y) >> 16] = vv.get();
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      if (a.mode == 0) {
        for (int k = 0; k < a.nbox; ++k) tma_store_2d(&tmV, 2 * cs, k * a.boxrows, X + k * a.boxrows);
      } else {
        bulk_store(a.V + int64_t(cs) * a.v_case, X, uint32_t(a.b) * 16u);
      }
      bulk_commit();
      a.iters[cs] = it;
    }
    if (a.resid) {
      // residual_per_case (fpi.py:221-240): max_i |s_i + v_i conj(src_i + (Y_dd v)_i)|,
      // the operations of residual_kernel in the same order (Y_dd rows in CSR order)
      double worst = 0.0;
#pragma unroll
      for (int j = 0; j < NSL; ++j) {
        D2 sd;
        tmem_ld2(tm_s + 4 * j, sd);
        tmem_wait_ld();
        const int p = base + 32 * j;
        const int2 pi = PI[p];
        const int rl = (pi.y >> 8) & 0xFF;
        if ((vmask >> j & 1u) && rl > 0) {
          const double2 si = __ldg(cs_src + p);
          double ar = si.x, ai = si.y;
          for (int r0 = 0; r0 < rl; r0 += 4) {  // ELL entries 4 at a time (loads issued together)
            int c[4];
            double2 y[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              if (r0 + r < rl) {
                c[r] = __ldg(a.ell_col + (r0 + r) * P + p);
                y[r] = __ldg(a.ell_val + (r0 + r) * P + p);
              }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              if (r0 + r < rl) {
                const double2 v = X[c[r]];
                ar = __fma_rn(y[r].x, v.x, __fma_rn(-y[r].y, v.y, ar));
                ai = __fma_rn(y[r].x, v.y, __fma_rn(y[r].y, v.x, ai));
              }
            }
          }
          const double2 v = X[uint32_t(pi.y) >> 16];
          const double2 sl = sd.get();
          const double mr = sl.x + (v.x * ar + v.y * ai);
          const double mi = sl.y + (v.y * ar - v.x * ai);
          worst = nanmax(worst, hypot(mr, mi));
        }
      }
      for (int o = 16; o > 0; o >>= 1) worst = nanmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
      if (lane == 0) s_red[warp] = worst;
    }
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
  }
  if (tid == 0) bulk_wait0();
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(s_tmem, 512);
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

template <int NSL>
int sub_launch(const SubArgs& a, const CUtensorMap& ms, const CUtensorMap& mv, size_t smem, int grid,
               cudaStream_t st) {
  auto kern = sparse_subtree_kernel<NSL>;
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

extern "C" int tpf_sparse_subtree_fpi_c128(int64_t tau, int32_t b, const int32_t* meta, int32_t nsl, int32_t ns,
                                           int32_t rmax, int32_t rw, int32_t nkids, const int32_t* pinfo,
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
  if (!meta || !pinfo || !kids || !coef || !ell_col || !ell_val || !S || !V || !iters || !workspace ||
      workspace_bytes < 256)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_subtree_fpi_c128: null pointer or small workspace");
  if (ns < 1 || ns >= nsl || rmax < 1 || rw < 1 || rw > kMaxRW || nkids < 1)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_subtree_fpi_c128: bad schedule");
  int mode;
  if (s_case_stride == 1 && v_case_stride == 1 && s_node_stride >= tau && v_node_stride >= tau)
    mode = 0;  // node-major (the reference layout)
  else if (s_node_stride == 1 && v_node_stride == 1 && s_case_stride >= b && v_case_stride >= b)
    mode = 1;  // case-major (F-order)
  else
    return set_error(TPF_ERR_UNSUPPORTED, "tpf_sparse_subtree_fpi_c128: S / V must be node- or case-major");
  if ((reinterpret_cast<uintptr_t>(S) | reinterpret_cast<uintptr_t>(V)) & 15)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_subtree_fpi_c128: S and V must be 16-byte aligned");
  SubArgs a;
  memset(&a, 0, sizeof a);
  a.tau = tau;
  a.b = b;
  a.NS = ns;
  a.RMAX = rmax;
  a.RW = rw;
  a.P = kSubWarps * nsl * 32;
  a.boxrows = b < 256 ? b : 256;
  a.nbox = (b + a.boxrows - 1) / a.boxrows;
  a.xcap = a.P > a.nbox * a.boxrows ? a.P : a.nbox * a.boxrows;
  a.nkids = nkids;
  a.mode = mode;
  a.S = reinterpret_cast<const double2*>(S);
  a.s_case = s_case_stride;
  a.V = reinterpret_cast<double2*>(V);
  a.v_case = v_case_stride;
  a.pinfo = reinterpret_cast<const int2*>(pinfo);
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
  for (int w = 0; w < kSubWarps; ++w) {
    a.jD[w] = meta[w];
    a.sync[w] = unsigned(meta[kSubWarps + w]);
  }
  const size_t smem = size_t(a.xcap) * 16 + size_t(a.P) * 8 + size_t(2) * kSubWarps * rmax * 32 * 16 +
                      (size_t(nkids) * 2 + 15) / 16 * 16;
  if (smem > 227 * 1024) return set_error(TPF_ERR_UNSUPPORTED, "tpf_sparse_subtree_fpi_c128: schedule too large");
  CUtensorMap ms, mv;
  memset(&ms, 0, sizeof ms);
  memset(&mv, 0, sizeof mv);
  if (mode == 0) {
    int rc = column_map(&ms, S, tau, b, s_node_stride, a.boxrows);
    if (rc != TPF_OK) return rc;
    rc = column_map(&mv, V, tau, b, v_node_stride, a.boxrows);
    if (rc != TPF_OK) return rc;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t err = cudaMemsetAsync(workspace, 0, sizeof(unsigned long long), st);
  if (err != cudaSuccess) return set_cuda_error("cudaMemsetAsync(counter)", err);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = int(tau < sms ? tau : sms);
  switch (nsl) {
    case 6: return sub_launch<6>(a, ms, mv, smem, grid, st);
    case 9: return sub_launch<9>(a, ms, mv, smem, grid, st);
    case 12: return sub_launch<12>(a, ms, mv, smem, grid, st);
    case 15: return sub_launch<15>(a, ms, mv, smem, grid, st);
    case 18: return sub_launch<18>(a, ms, mv, smem, grid, st);
    case 21: return sub_launch<21>(a, ms, mv, smem, grid, st);
    default: break;
  }
  return set_error(TPF_ERR_UNSUPPORTED, "tpf_sparse_subtree_fpi_c128: unsupported slot count");
}
