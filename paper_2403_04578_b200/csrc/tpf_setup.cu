// Dense setup on the device for radial feeders: K = -inv(Y_dd) and W = K src
// (reference: dense.py:150-152, K = -np.linalg.inv(Y_dd); W = K @ src).
//
// The reference inverts Y_dd with LAPACK on the host, O(b^3).  On a radial
// feeder Y_dd has a zero-fill tree LU (the one the sparse path factors,
// sparse.py:186), so column j of K is one tree solve Y_dd x = -e_j: an
// up-sweep (children before parents) and a down-sweep, O(b) per column and
// O(b^2) for K.  One thread per column; the b columns run side by side and
// every thread walks the nodes in the same order, so the tree coefficients
// are warp-uniform loads and the per-column values K[orig(m)][j] (row orig(m)
// of K doubles as the solve's working vector) are coalesced across the warp.
// Operations per node are those of the sparse kernels' sweeps (tree_solve_host
// in paper_2403_04578_b200/sparse.py), so K is the solve of the very LU the
// sparse path uses; it agrees with LAPACK's inverse to rounding, not bitwise.
#include "tpf_common.cuh"
#include "tpf_internal.h"

namespace tpf {
namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 x) {
  return make_double2(__fma_rn(a.x, x.x, -(a.y * x.y)), __fma_rn(a.x, x.y, a.y * x.x));
}

// node_info: int32 [b][4] {original node, parent, first child, child count}
// (level order, parents before children); coef planes (level order): [1] g =
// U[m,parent] / U[m,m], [2] 1 / U[m,m].
__global__ void __launch_bounds__(128) tree_inverse_kernel(int b, int levels, const int32_t* __restrict__ level_off,
                                                           const int4* __restrict__ info,
                                                           const double2* __restrict__ coef, double2* __restrict__ K) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= b) return;
  const double2* g = coef + b;
  const double2* uinv = coef + 2 * b;
  // up-sweep, deepest level first: z_m = rhs_m - sum_c g_c z_c, rhs = -e_j
  for (int d = levels - 1; d >= 0; --d) {
    const int m0 = __ldg(level_off + d), m1 = __ldg(level_off + d + 1);
    for (int m = m0; m < m1; ++m) {
      const int4 in = __ldg(info + m);
      double2 z = make_double2(in.x == j ? -1.0 : 0.0, 0.0);
      for (int c = in.z; c < in.z + in.w; ++c) {
        const double2 gc = __ldg(g + c);
        const double2 zc = K[size_t(__ldg(info + c).x) * b + j];
        const double2 p = cmul(gc, zc);
        z.x -= p.x;
        z.y -= p.y;
      }
      K[size_t(in.x) * b + j] = z;
    }
  }
  // down-sweep, root level first: w_m = z_m / U_mm - g_m w_parent
  for (int d = 0; d < levels; ++d) {
    const int m0 = __ldg(level_off + d), m1 = __ldg(level_off + d + 1);
    for (int m = m0; m < m1; ++m) {
      const int4 in = __ldg(info + m);
      double2 w = cmul(K[size_t(in.x) * b + j], __ldg(uinv + m));
      if (in.y >= 0) {
        const double2 p = cmul(__ldg(g + m), K[size_t(__ldg(info + in.y).x) * b + j]);
        w.x -= p.x;
        w.y -= p.y;
      }
      K[size_t(in.x) * b + j] = w;
    }
  }
}

// W = K src (dense.py:152): one warp per row, fixed reduction order
__global__ void __launch_bounds__(256) kw_kernel(int b, const double2* __restrict__ K, const double2* __restrict__ src,
                                                 double2* __restrict__ W) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= b) return;
  double re = 0.0, im = 0.0;
  for (int j = lane; j < b; j += 32) {
    const double2 k = K[size_t(row) * b + j], s = __ldg(src + j);
    re = __fma_rn(k.x, s.x, __fma_rn(-k.y, s.y, re));
    im = __fma_rn(k.x, s.y, __fma_rn(k.y, s.x, im));
  }
  for (int o = 16; o > 0; o >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, o);
    im += __shfl_xor_sync(0xffffffffu, im, o);
  }
  if (lane == 0) W[row] = make_double2(re, im);
}

}  // namespace
}  // namespace tpf

using namespace tpf;

extern "C" int tpf_dense_setup_tree_c128(int32_t b, int32_t levels, const int32_t* level_off,
                                         const int32_t* node_info, const double* node_coef, const double* src,
                                         double* K, double* W, void* stream) {
  if (b < 1 || levels < 1) return set_error(TPF_ERR_INVALID, "tpf_dense_setup_tree_c128: need b >= 1, levels >= 1");
  if (!level_off || !node_info || !node_coef || !src || !K || !W)
    return set_error(TPF_ERR_INVALID, "tpf_dense_setup_tree_c128: null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  tree_inverse_kernel<<<unsigned((b + 127) / 128), 128, 0, st>>>(
      b, levels, level_off, reinterpret_cast<const int4*>(node_info), reinterpret_cast<const double2*>(node_coef),
      reinterpret_cast<double2*>(K));
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(tree_inverse_kernel)", err);
  kw_kernel<<<unsigned((b + 7) / 8), 256, 0, st>>>(b, reinterpret_cast<const double2*>(K),
                                                    reinterpret_cast<const double2*>(src), reinterpret_cast<double2*>(W));
  err = cudaGetLastError();
  return err == cudaSuccess ? TPF_OK : set_cuda_error("launch(kw_kernel)", err);
}
