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
  const double2* coef;    // per m: {e = Y[parent, m], unused, uinv = 1/U[m,m], src}
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

constexpr int kSB = 3;  // slots per batch: their loads are issued together (ILP across slots)

// Scaled sweeps (zhat = z / U_mm, so L[p,c] z_c = Y[p,c] zhat_c):
//   up:   zhat_m = (r_m - sum_c e_c zhat_c) * uinv_m,   e_c = Y[parent(c), c]
//   down: w_m    = zhat_m - uinv_m * e_m * w_parent     (U[m,p] = Y[m,p] = e_m for symmetric Y)
__global__ void __launch_bounds__(kTreeThreads, 1) sparse_tree_kernel(const TreeArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* T = reinterpret_cast<double2*>(smem_raw);       // [b] sweep vector (zhat, then w)
  double2* P = T + a.b;                                    // [b] e_m * zhat_m, pulled by the parent
  int2* kids = reinterpret_cast<int2*>(P + a.b);           // [b] {first child, count}
  int* par = reinterpret_cast<int*>(kids + a.b);           // [b] parent (-1 at roots)
  __shared__ int s_off[kMaxLevels + 1], s_j0[kMaxLevels + 1];
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
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tm = s_tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * 128);
  const uint32_t tm_v = tm, tm_s = tm + 4 * kMaxSlots;

  for (;;) {
    if (tid == 0) {
      const unsigned long long c = atomicAdd(a.counter, 1ull);
      s_case = c < (unsigned long long)a.tau ? int(c) : -1;
    }
    __syncthreads();
    const int cs = s_case;
    if (cs < 0) break;

    // ---- load the case: S into TMEM, flat start V (dense.py:155) ----
    for (int d = 0; d < L; ++d) {
      for (int j = s_j0[d]; j < s_j0[d + 1]; ++j) {
        const int pos = (j - s_j0[d]) * kTreeThreads + tid;
        double2 s = make_double2(0.0, 0.0);
        if (s_off[d] + pos < s_off[d + 1]) {
          const int node = __ldg(&a.info[s_off[d] + pos].x);
          s = __ldg(a.S + node * a.s_node + int64_t(cs) * a.s_case);
        }
        tmem_st2(tm_s + 4 * j, s);
        tmem_st2(tm_v + 4 * j, a.v_flat);
      }
    }
    tmem_wait_st();

    int it = 0;
    while (it < a.max_iter) {
      // ---- up-sweep: deepest level first ----
      for (int d = L - 1; d >= 0; --d) {
        const int off = s_off[d], end = s_off[d + 1], jb = s_j0[d], je = s_j0[d + 1];
        for (int j = jb; j < je; j += kSB) {
          D2 vv[kSB], ss[kSB];
          double2 ui[kSB], src[kSB], e[kSB];
#pragma unroll
          for (int u = 0; u < kSB; ++u) {
            if (j + u < je) {  // warp-uniform
              tmem_ld2(tm_v + 4 * (j + u), vv[u]);
              tmem_ld2(tm_s + 4 * (j + u), ss[u]);
            }
            const int m = off + (j + u - jb) * kTreeThreads + tid;
            const bool ok = j + u < je && m < end;
            ui[u] = ok ? __ldg(&a.coef[4 * m + 2]) : make_double2(0.0, 0.0);
            e[u] = (ok && d > 0) ? __ldg(&a.coef[4 * m]) : make_double2(0.0, 0.0);
            src[u] = (ok && d == 0) ? __ldg(&a.coef[4 * m + 3]) : make_double2(0.0, 0.0);
          }
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < kSB; ++u) {
            const int m = off + (j + u - jb) * kTreeThreads + tid;
            if (j + u < je && m < end) {
              double2 v = vv[u].get();
              const double2 s = ss[u].get();
              double m2 = __fma_rn(v.x, v.x, v.y * v.y);
              if (m2 < kZeroGuard2) {  // fpi.py:39-41
                v = make_double2(kZeroGuard, 0.0);
                m2 = kZeroGuard * kZeroGuard;
              }
              const double r = 1.0 / m2;
              // r_m = -(s*/conj(v) + src),  s*/conj(v) = conj(s) v / |v|^2
              double2 z = make_double2(-(__fma_rn(s.x, v.x, s.y * v.y) * r + src[u].x),
                                       -(__fma_rn(s.x, v.y, -(s.y * v.x)) * r + src[u].y));
              const int2 k = kids[m];
              for (int c = k.x; c < k.x + k.y; ++c) {
                const double2 pc = P[c];
                z.x -= pc.x;
                z.y -= pc.y;
              }
              const double2 zh = cmul2(z, ui[u]);
              T[m] = zh;
              P[m] = cmul2(e[u], zh);
            }
          }
        }
        __syncthreads();
      }
      // ---- down-sweep: root level first, step test, iterate update ----
      bool small = true;
      int all_small = 0;
      for (int d = 0; d < L; ++d) {
        const int off = s_off[d], end = s_off[d + 1], jb = s_j0[d], je = s_j0[d + 1];
        for (int j = jb; j < je; j += kSB) {
          D2 vv[kSB];
          double2 e[kSB], ui[kSB];
#pragma unroll
          for (int u = 0; u < kSB; ++u) {
            if (j + u < je) tmem_ld2(tm_v + 4 * (j + u), vv[u]);
            const int m = off + (j + u - jb) * kTreeThreads + tid;
            const bool ok = j + u < je && m < end && d > 0;
            e[u] = ok ? __ldg(&a.coef[4 * m]) : make_double2(0.0, 0.0);
            ui[u] = ok ? __ldg(&a.coef[4 * m + 2]) : make_double2(0.0, 0.0);
          }
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < kSB; ++u) {
            if (j + u < je) {
              const int m = off + (j + u - jb) * kTreeThreads + tid;
              double2 v = vv[u].get();
              double2 w = v;
              if (m < end) {
                w = T[m];
                const int p = par[m];
                if (p >= 0) w = cfma_sub(w, cmul2(ui[u], e[u]), T[p]);
                T[m] = w;
                if (__fma_rn(v.x, v.x, v.y * v.y) < kZeroGuard2) v = make_double2(kZeroGuard, 0.0);
                const double dr = w.x - v.x, di = w.y - v.y;
                if (!(__fma_rn(dr, dr, di * di) < a.tol2)) small = false;  // NaN never passes
              }
              tmem_st2(tm_v + 4 * (j + u), w);
            }
          }
        }
        tmem_wait_st();
        if (d + 1 < L)
          __syncthreads();
        else
          all_small = __syncthreads_and(small);
      }
      ++it;
      if (all_small) break;
    }

    // ---- retire: V out, per-case count ----
    for (int d = 0; d < L; ++d) {
      for (int j = s_j0[d]; j < s_j0[d + 1]; ++j) {
        D2 vv;
        tmem_ld2(tm_v + 4 * j, vv);
        tmem_wait_ld();
        const int m = s_off[d] + (j - s_j0[d]) * kTreeThreads + tid;
        if (m < s_off[d + 1]) {
          const int node = __ldg(&a.info[m].x);
          a.V[node * a.v_node + int64_t(cs) * a.v_case] = vv.get();
        }
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
