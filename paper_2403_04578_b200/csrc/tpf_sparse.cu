// Sparse Tensor Power Flow on sm_100a: batched multi-RHS LU trisolves.
//
// Replaces the hot loop of the reference `batch_solve_sparse`
// (pkg/src/tpflow/sparse.py:186-197), which re-solves one tau-block-diagonal
// SuperLU factorization per iteration (sparse.py:192).  Per case j the
// reference block row i reads  -Y_dd[i,:] v' / s_ij* = 1/conj(v_ij) + src_i / s_ij*
// (zero-load rows unscaled, sparse.py:144-151), which is the same equation as
//     Y_dd v'_j = -( s_j* ./ conj(v_j) + src )
// for every row, zero loads included.  So ONE LU of Y_dd (factorized on the
// host, Pr Y_dd Pc = L U) serves all tau cases: each iteration is a forward
// sweep with L and a backward sweep with U on a b x tau right-hand side.
//
// Layout: node-major b x tau (tau contiguous, the reference's LoadMatrix
// layout), one thread per case, so every access to node i of 32 consecutive
// cases is one coalesced 512-byte transaction; the factor entries are read
// uniformly across the warp (broadcast).  Each case iterates independently
// until its own step test passes (per-case freeze).
#include <climits>

#include "tpf_common.cuh"
#include "tpf_internal.h"

namespace tpf {

struct SparseArgs {
  int64_t tau;
  int b;
  const double* S;
  int64_t s_node, s_case;
  const int32_t* l_ptr;  // strictly-lower part of unit-diagonal L, CSR
  const int32_t* l_col;
  const double* l_val;
  const int32_t* u_ptr;  // strictly-upper part of U, CSR
  const int32_t* u_col;
  const double* u_val;
  const double* u_diag_inv;  // 1 / U[k,k]
  const int32_t* row_src;    // forward-sweep row k takes the RHS of node row_src[k] (perm_r inverse)
  const int32_t* col_dst;    // solution of node i sits at permuted index col_dst[i] (perm_c)
  const double* src;         // Y_ds v_s
  double v_flat_re, v_flat_im, tol2;
  int max_iter;
  double* V;
  int64_t v_node, v_case;
  int32_t* iters;
  double* T;  // b x tau scratch, node-major (permuted index), case stride 1
  int64_t t_ld;
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -(a.y * b.y)), __fma_rn(a.x, b.y, a.y * b.x));
}

__global__ void __launch_bounds__(128) sparse_fpi_kernel(const SparseArgs a) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= a.tau) return;
  const int b = a.b;
  double2* T = reinterpret_cast<double2*>(a.T);
  double2* V = reinterpret_cast<double2*>(a.V);
  const double2* S = reinterpret_cast<const double2*>(a.S);
  const double2* src = reinterpret_cast<const double2*>(a.src);
  const double2* lv = reinterpret_cast<const double2*>(a.l_val);
  const double2* uv = reinterpret_cast<const double2*>(a.u_val);
  const double2* ud = reinterpret_cast<const double2*>(a.u_diag_inv);

  // flat start (dense.py:155 / sparse.py:185)
  for (int i = 0; i < b; ++i) V[i * a.v_node + j * a.v_case] = make_double2(a.v_flat_re, a.v_flat_im);

  int n = 0;
  while (n < a.max_iter) {
    // forward sweep: z_k = rhs(row_src[k]) - sum_m L[k,m] z_m,
    // rhs_i = -(s_i* / conj(v_i) + src_i) with the zero-voltage guard on v_i
    for (int k = 0; k < b; ++k) {
      const int i = __ldg(a.row_src + k);
      double2 v = V[i * a.v_node + j * a.v_case];
      double m2 = __fma_rn(v.x, v.x, v.y * v.y);
      if (m2 < kZeroGuard2) {
        v = make_double2(kZeroGuard, 0.0);
        m2 = kZeroGuard * kZeroGuard;
      }
      const double2 s = __ldg(S + i * a.s_node + j * a.s_case);
      const double r = 1.0 / m2;
      // s*/conj(v) = conj(s) v / |v|^2
      const double ur = __fma_rn(s.x, v.x, s.y * v.y) * r;
      const double ui = __fma_rn(s.x, v.y, -(s.y * v.x)) * r;
      const double2 c = __ldg(src + i);
      double zr = -(ur + c.x), zi = -(ui + c.y);
      for (int p = __ldg(a.l_ptr + k); p < __ldg(a.l_ptr + k + 1); ++p) {
        const double2 l = __ldg(lv + p);
        const double2 z = T[__ldg(a.l_col + p) * a.t_ld + j];
        zr = __fma_rn(-l.x, z.x, __fma_rn(l.y, z.y, zr));
        zi = __fma_rn(-l.x, z.y, __fma_rn(-l.y, z.x, zi));
      }
      T[k * a.t_ld + j] = make_double2(zr, zi);
    }
    // backward sweep: w_k = (z_k - sum_m U[k,m] w_m) / U[k,k]
    for (int k = b - 1; k >= 0; --k) {
      double2 z = T[k * a.t_ld + j];
      for (int p = __ldg(a.u_ptr + k); p < __ldg(a.u_ptr + k + 1); ++p) {
        const double2 u = __ldg(uv + p);
        const double2 w = T[__ldg(a.u_col + p) * a.t_ld + j];
        z.x = __fma_rn(-u.x, w.x, __fma_rn(u.y, w.y, z.x));
        z.y = __fma_rn(-u.x, w.y, __fma_rn(-u.y, w.x, z.y));
      }
      T[k * a.t_ld + j] = cmul(z, __ldg(ud + k));
    }
    // scatter to node order, step test (the guarded iterate is the old value)
    bool small = true;
    for (int i = 0; i < b; ++i) {
      const double2 x = T[__ldg(a.col_dst + i) * a.t_ld + j];
      double2 v = V[i * a.v_node + j * a.v_case];
      if (__fma_rn(v.x, v.x, v.y * v.y) < kZeroGuard2) v = make_double2(kZeroGuard, 0.0);
      const double dr = x.x - v.x, di = x.y - v.y;
      if (!(__fma_rn(dr, dr, di * di) < a.tol2)) small = false;
      V[i * a.v_node + j * a.v_case] = x;
    }
    ++n;
    if (small) break;
  }
  a.iters[j] = n;
}

}  // namespace tpf

using namespace tpf;

extern "C" size_t tpf_sparse_workspace_bytes(int64_t tau, int32_t b) {
  return size_t(tau) * size_t(b) * 16 + 256;
}

extern "C" int tpf_sparse_fpi_c128(int64_t tau, int32_t b, const double* S, int64_t s_node_stride,
                                   int64_t s_case_stride, const int32_t* l_ptr, const int32_t* l_col,
                                   const double* l_val, const int32_t* u_ptr, const int32_t* u_col,
                                   const double* u_val, const double* u_diag_inv, const int32_t* perm,
                                   const double* src, double v_flat_re, double v_flat_im, double tol,
                                   int32_t max_iter, double* V, int64_t v_node_stride, int64_t v_case_stride,
                                   int32_t* iters, void* workspace, size_t workspace_bytes, void* stream) {
  if (tau < 0 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_sparse_fpi_c128: need tau >= 0, b >= 1");
  if (!(tol > 0.0)) return set_error(TPF_ERR_INVALID, "tolerance must be positive");
  if (max_iter < 1) return set_error(TPF_ERR_INVALID, "max_iterations must be >= 1");
  if (tau == 0) return TPF_OK;
  if (!S || !l_ptr || !u_ptr || !u_diag_inv || !perm || !src || !V || !iters || !workspace)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_fpi_c128: null pointer");
  if (workspace_bytes < tpf_sparse_workspace_bytes(tau, b))
    return set_error(TPF_ERR_INVALID, "tpf_sparse_fpi_c128: workspace too small");
  SparseArgs a;
  a.tau = tau;
  a.b = b;
  a.S = S;
  a.s_node = s_node_stride;
  a.s_case = s_case_stride;
  a.l_ptr = l_ptr;
  a.l_col = l_col;
  a.l_val = l_val;
  a.u_ptr = u_ptr;
  a.u_col = u_col;
  a.u_val = u_val;
  a.u_diag_inv = u_diag_inv;
  a.row_src = perm;      // perm[0..b): forward row k reads node perm[k]
  a.col_dst = perm + b;  // perm[b..2b): node i's solution at permuted index perm[b+i]
  a.src = src;
  a.v_flat_re = v_flat_re;
  a.v_flat_im = v_flat_im;
  a.tol2 = tol * tol;
  a.max_iter = max_iter;
  a.V = V;
  a.v_node = v_node_stride;
  a.v_case = v_case_stride;
  a.iters = iters;
  a.T = static_cast<double*>(workspace);
  a.t_ld = tau;
  const int threads = 128;
  const int64_t blocks = (tau + threads - 1) / threads;
  sparse_fpi_kernel<<<unsigned(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(a);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(sparse_fpi_kernel)", err);
  return TPF_OK;
}
