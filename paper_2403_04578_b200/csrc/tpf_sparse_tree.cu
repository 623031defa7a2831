// Sparse Tensor Power Flow for radial feeders: one case per CTA, all of the
// case's state on chip, level-synchronous tree sweeps.
//
// For a tree-structured Y_dd in leaf-first order the LU has no fill
// (SURVEY.md A.6): row k of L holds only k's children, row k of U only its
// parent.  Grouping nodes by depth, one fixed-point iteration
//     Y_dd v' = -(s* ./ conj(v) + src)          (sparse.py:3-14, 186-197)
// is an up-sweep (deepest level first)
//     z_k = r_k - sum_{c child of k} L_kc z_c,   r_k = -(s_k*/conj(v_k) + src_k)
// and a down-sweep (root level first)
//     w_k = (z_k - U_kp w_p) / U_kk,             v'_k = w_k.
// Both sweeps use the SAME depth levels, so one thread owns node k in both
// and keeps the node's iterate v_k and load s_k in its own Tensor Memory lane
// (4 columns each per "slot"; a slot is one node of one level for every thread
// of the CTA, so TMEM addresses stay warp-uniform).  The sweep vector z/w of
// the whole case lives in shared memory (16 B per node).  Global memory is
// touched once per case: S in, V out (the compulsory traffic).
//
// CTA = 512 threads (16 warps, 4 per TMEM lane quadrant, 128 columns each =
// 16 slots), one CTA per SM (all 512 TMEM columns), persistent over cases.
#include <climits>

#include "tpf_common.cuh"
#include "tpf_internal.h"

namespace tpf {
namespace {

constexpr int kTreeThreads = 512;
constexpr int kMaxSlots = 16;
constexpr int kMaxLevels = 64;

struct TreeArgs {
  int64_t tau;
  int b, levels;
  const double2* S;
  int64_t s_node, s_case;
  double2* V;
  int64_t v_node, v_case;
  int32_t* iters;
  unsigned long long* counter;
  const int32_t* lvl;     // [levels+1] level offsets in level order (root level first), then [levels+1] slot starts
  const int4* info;       // per level-ordered node m: {original node, parent m or -1, first child m, child count}
  const double2* coef;    // per m: {e = Y[parent, m], g = U[m,parent]/U[m,m], uinv = 1/U[m,m], src}
  double2 v_flat;
  double tol2;
  int max_iter;
};

__device__ __forceinline__ double2 cfma_sub(double2 acc, double2 a, double2 x) {  // acc - a*x
  return make_double2(__fma_rn(-a.x, x.x, __fma_rn(a.y, x.y, acc.x)), __fma_rn(-a.x, x.y, __fma_rn(-a.y, x.x, acc.y)));
}
__device__ __forceinline__ double2 cmul2(double2 a, double2 x) {
  return make_double2(__fma_rn(a.x, x.x, -(a.y * x.y)), __fma_rn(a.x, x.y, a.y * x.x));
}

constexpr int kLS = 6;  // max TMEM slots of one level (the host schedule guarantees it)
constexpr int kMaxRoots = 512;

// Sweeps with g_m = U[m,parent] / U[m,m] (so L[p,m] z_m = g_m z_m for symmetric Y):
//   up:   z_m = r_m - sum_c g_c z_c
//   down: w_m = z_m / U[m,m] - g_m w_parent
__global__ void __launch_bounds__(kTreeThreads, 1) sparse_tree_kernel(const TreeArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* T = reinterpret_cast<double2*>(smem_raw);       // [b] sweep vector (zhat, then w)
  double2* P = T + a.b;                                    // [b] e_m * zhat_m, pulled by the parent
  int2* kids = reinterpret_cast<int2*>(P + a.b);           // [b] {first child, count}
  int* par = reinterpret_cast<int*>(kids + a.b);           // [b] parent (-1 at roots)
  __shared__ int s_off[kMaxLevels + 1], s_j0[kMaxLevels + 1];
  __shared__ double2 s_src[kMaxRoots];  // source injection of the root level (zero elsewhere)
  __shared__ int s_slot_lvl[kMaxSlots];
  __shared__ int s_case;
  __shared__ uint32_t s_tmem;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int L = a.levels;
  for (int i = tid; i <= L; i += kTreeThreads) {
    s_off[i] = a.lvl[i];
    s_j0[i] = a.lvl[L + 1 + i];
  }
  for (int m = tid; m < a.b; m += kTreeThreads) {
    const int4 inf = __ldg(&a.info[m]);
    kids[m] = make_int2(inf.z, inf.w);
    par[m] = inf.y;
  }
  __syncthreads();
  for (int m = tid; m < s_off[1] && m < kMaxRoots; m += kTreeThreads) s_src[m] = __ldg(&a.coef[4 * m + 3]);
  if (tid < kMaxSlots) {
    int lv = 0;
    for (int d = 0; d < L; ++d)
      if (s_j0[d] <= tid && tid < s_j0[d + 1]) lv = d;
    s_slot_lvl[tid] = lv;
  }
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tm = s_tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * 128);
  const uint32_t tm_v = tm, tm_s = tm + 4 * kMaxSlots;
  const int nslots = s_j0[L];
  // node of TMEM slot j of this thread (-1 if none): slot j belongs to level s_slot_lvl[j]
  auto slot_node = [&](int j) {
    if (j >= nslots) return -1;
    const int d = s_slot_lvl[j];
    const int m = s_off[d] + (j - s_j0[d]) * kTreeThreads + tid;
    return m < s_off[d + 1] ? m : -1;
  };

  for (;;) {
    if (tid == 0) {
      const unsigned long long c = atomicAdd(a.counter, 1ull);
      s_case = c < (unsigned long long)a.tau ? int(c) : -1;
    }
    __syncthreads();
    const int cs = s_case;
    if (cs < 0) break;

    // ---- load the case: S into TMEM, flat start V (dense.py:155) ----
    // all of this thread's slots at once: the S loads are independent HBM/L2
    // round trips, so they are issued together before any TMEM store
#pragma unroll
    for (int j0 = 0; j0 < kMaxSlots; j0 += 4) {
      double2 sv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = slot_node(j0 + j);
        sv[j] = make_double2(0.0, 0.0);
        if (m >= 0) sv[j] = __ldg(a.S + __ldg(&a.info[m].x) * a.s_node + int64_t(cs) * a.s_case);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j0 + j < nslots) {  // warp-uniform
          tmem_st2(tm_s + 4 * (j0 + j), sv[j]);
          tmem_st2(tm_v + 4 * (j0 + j), a.v_flat);
        }
      }
    }
    tmem_wait_st();

    // Per level, every thread holds the data of its (at most kLS) slots of that
    // level in registers: the TMEM iterate/load and the node coefficients.  A
    // level's loads are issued right after the previous level's arithmetic,
    // BEFORE the barrier, so their latency overlaps the barrier wait.
    //   up:   z_m = r_m - sum_c P_c,  P_m = g_m z_m            (g = U[m,p] / U[m,m])
    //   down: w_m = z_m / U_mm - g_m w_p
    D2 vv[1], ss[1];
    double2 cg[kLS], cu[kLS];
    // global coefficient loads of a level, issued before the barrier that precedes it
    auto issue_up = [&](int d) {
      const int jb = s_j0[d], je = s_j0[d + 1], off = s_off[d], end = s_off[d + 1];
#pragma unroll
      for (int u = 0; u < kLS; ++u) {
        const int m = off + u * kTreeThreads + tid;
        cg[u] = (jb + u < je && m < end) ? __ldg(&a.coef[4 * m + 1]) : make_double2(0.0, 0.0);
      }
    };
    auto issue_down = [&](int d) {
      const int jb = s_j0[d], je = s_j0[d + 1], off = s_off[d], end = s_off[d + 1];
#pragma unroll
      for (int u = 0; u < kLS; ++u) {
        const int m = off + u * kTreeThreads + tid;
        const bool ok = jb + u < je && m < end;
        cu[u] = ok ? __ldg(&a.coef[4 * m + 2]) : make_double2(0.0, 0.0);
        cg[u] = (ok && d > 0) ? __ldg(&a.coef[4 * m + 1]) : make_double2(0.0, 0.0);
      }
    };

    int it = 0;
    issue_up(L - 1);
    while (it < a.max_iter) {
      // ---- up-sweep: deepest level first ----
      for (int d = L - 1; d >= 0; --d) {
        const int off = s_off[d], end = s_off[d + 1], jb = s_j0[d], je = s_j0[d + 1];
#pragma unroll
        for (int u = 0; u < kLS; ++u) {
          const int m = off + u * kTreeThreads + tid;
          if (jb + u < je) {  // warp-uniform
            tmem_ld2(tm_v + 4 * (jb + u), vv[0]);
            tmem_ld2(tm_s + 4 * (jb + u), ss[0]);
            tmem_wait_ld();
          }
          if (jb + u < je && m < end) {
            double2 v = vv[0].get();
            const double2 sl = ss[0].get();
            double m2 = __fma_rn(v.x, v.x, v.y * v.y);
            if (m2 < kZeroGuard2) {  // fpi.py:39-41
              v = make_double2(kZeroGuard, 0.0);
              m2 = kZeroGuard * kZeroGuard;
            }
            const double r = 1.0 / m2;
            const double2 src = d == 0 ? s_src[m] : make_double2(0.0, 0.0);
            // r_m = -(s*/conj(v) + src),  s*/conj(v) = conj(s) v / |v|^2
            double2 z = make_double2(-(__fma_rn(sl.x, v.x, sl.y * v.y) * r + src.x),
                                     -(__fma_rn(sl.x, v.y, -(sl.y * v.x)) * r + src.y));
            const int2 k = kids[m];
            for (int c = k.x; c < k.x + k.y; ++c) {
              const double2 pc = P[c];
              z.x -= pc.x;
              z.y -= pc.y;
            }
            T[m] = z;
            P[m] = cmul2(cg[u], z);
          }
        }
        if (d > 0)
          issue_up(d - 1);
        else
          issue_down(0);
        __syncthreads();
      }
      // ---- down-sweep: root level first, step test, iterate update ----
      bool small = true;
      int all_small = 0;
      for (int d = 0; d < L; ++d) {
        const int off = s_off[d], end = s_off[d + 1], jb = s_j0[d], je = s_j0[d + 1];
#pragma unroll
        for (int u = 0; u < kLS; ++u) {
          if (jb + u < je) {
            const int m = off + u * kTreeThreads + tid;
            tmem_ld2(tm_v + 4 * (jb + u), vv[0]);
            tmem_wait_ld();
            double2 v = vv[0].get();
            double2 w = v;
            if (m < end) {
              w = cmul2(T[m], cu[u]);
              const int p = par[m];
              if (p >= 0) w = cfma_sub(w, cg[u], T[p]);
              T[m] = w;
              if (__fma_rn(v.x, v.x, v.y * v.y) < kZeroGuard2) v = make_double2(kZeroGuard, 0.0);
              const double dr = w.x - v.x, di = w.y - v.y;
              if (!(__fma_rn(dr, dr, di * di) < a.tol2)) small = false;  // NaN never passes
            }
            tmem_st2(tm_v + 4 * (jb + u), w);
          }
        }
        tmem_wait_st();
        if (d + 1 < L) {
          issue_down(d + 1);
          __syncthreads();
        } else {
          all_small = __syncthreads_and(small);
        }
      }
      ++it;
      if (all_small) break;
      issue_up(L - 1);
    }

    // ---- retire: V out, per-case count ----
#pragma unroll
    for (int j0 = 0; j0 < kMaxSlots; j0 += 4) {
      D2 vo[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j0 + j < nslots) tmem_ld2(tm_v + 4 * (j0 + j), vo[j]);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = slot_node(j0 + j);
        if (m >= 0) a.V[__ldg(&a.info[m].x) * a.v_node + int64_t(cs) * a.v_case] = vo[j].get();
      }
    }
    if (tid == 0) a.iters[cs] = it;
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(s_tmem, 512);
}

}  // namespace
}  // namespace tpf

using namespace tpf;

extern "C" int tpf_sparse_tree_max_slots(void) { return kMaxSlots; }

extern "C" int tpf_sparse_tree_fpi_c128(int64_t tau, int32_t b, int32_t levels, const int32_t* level_info,
                                        const int32_t* node_info, const double* node_coef, const double* S,
                                        int64_t s_node_stride, int64_t s_case_stride, double v_flat_re,
                                        double v_flat_im, double tol, int32_t max_iter, double* V,
                                        int64_t v_node_stride, int64_t v_case_stride, int32_t* iters,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  if (tau < 0 || b < 1 || levels < 1 || levels > kMaxLevels)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_fpi_c128: bad shape");
  if (!(tol > 0.0)) return set_error(TPF_ERR_INVALID, "tolerance must be positive");
  if (max_iter < 1) return set_error(TPF_ERR_INVALID, "max_iterations must be >= 1");
  if (tau == 0) return TPF_OK;
  if (!level_info || !node_info || !node_coef || !S || !V || !iters || !workspace || workspace_bytes < 256)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_fpi_c128: null pointer or small workspace");
  const size_t smem = size_t(b) * (2 * sizeof(double2) + sizeof(int2) + sizeof(int));
  if (smem > 220 * 1024) return set_error(TPF_ERR_UNSUPPORTED, "tpf_sparse_tree_fpi_c128: b too large for one SM");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t err = cudaFuncSetAttribute(sparse_tree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (err != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(tree)", err);
  err = cudaMemsetAsync(workspace, 0, sizeof(unsigned long long), st);
  if (err != cudaSuccess) return set_cuda_error("cudaMemsetAsync(counter)", err);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  TreeArgs a;
  a.tau = tau;
  a.b = b;
  a.levels = levels;
  a.S = reinterpret_cast<const double2*>(S);
  a.s_node = s_node_stride;
  a.s_case = s_case_stride;
  a.V = reinterpret_cast<double2*>(V);
  a.v_node = v_node_stride;
  a.v_case = v_case_stride;
  a.iters = iters;
  a.counter = static_cast<unsigned long long*>(workspace);
  a.lvl = level_info;
  a.info = reinterpret_cast<const int4*>(node_info);
  a.coef = reinterpret_cast<const double2*>(node_coef);
  a.v_flat = make_double2(v_flat_re, v_flat_im);
  a.tol2 = tol * tol;
  a.max_iter = max_iter;
  int64_t grid = sms;
  if (tau < grid) grid = tau;
  sparse_tree_kernel<<<unsigned(grid), kTreeThreads, smem, st>>>(a);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(sparse_tree_kernel)", err);
  return TPF_OK;
}
