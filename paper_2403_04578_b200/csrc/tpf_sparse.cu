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

#include <cstring>

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

// ---------------------------------------------------------------------------
// ZIP loads on radial feeders of any depth / size (the fallback of the tree
// kernel's ZIP mode): one thread per case, nodes in leaf-first order.  Per
// case the tree LU of B = Y_dd + diag(alpha_z s*) (no fill: U[k,k] = B[k,k] -
// sum_c e_c^2 / U[c,c], g_k = e_k / U[k,k]) and fpi_solve's iteration
// (fpi.py:107-206): B v' = -(alpha_p s*/conj(v) + src + alpha_i s*), one
// application when alpha_p s = 0, stop on a non-finite iterate; the ZIP
// residual (fpi.py:209-240) summed over the tree edges.  Scratch: four
// node-major b x tau complex arrays (pivots/sweep, g, 1/U, Y v).
namespace tpf {
namespace {

struct ZipChainArgs {
  int64_t tau;
  int b;
  const double2* S;
  int64_t s_node, s_case;   // original node order
  const int32_t* orig;      // leaf-first position k -> original node
  const int32_t* parent;    // position of k's parent, -1 at roots
  const double2* e;         // Y[k, parent(k)] (symmetric)
  const double2* ydiag;     // Y[k, k]
  const double* alpha;      // [3][b] alpha_z, alpha_i, alpha_p (leaf-first order)
  const double2* src;       // source injection (leaf-first order)
  double2 v_flat;
  const double2* v0;        // initial iterate (original node order) or null: flat start
  double tol2;
  int max_iter;
  double2* V;
  int64_t v_node, v_case;   // original node order
  int32_t* iters;
  double* resid;
  uint8_t* met;
  int32_t* status;
  double2 *Z, *G, *UI, *A;  // scratch, [b][tau]
};

__device__ __forceinline__ double2 cmulz(double2 a, double2 x) {
  return make_double2(__fma_rn(a.x, x.x, -(a.y * x.y)), __fma_rn(a.x, x.y, a.y * x.x));
}

__global__ void __launch_bounds__(128) sparse_zip_chain_kernel(const ZipChainArgs a) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= a.tau) return;
  const int b = a.b;
  const int64_t t = a.tau;
  auto Sk = [&](int k) { return a.S[int64_t(__ldg(a.orig + k)) * a.s_node + j * a.s_case]; };
  auto Vk = [&](int k) -> double2& { return a.V[int64_t(__ldg(a.orig + k)) * a.v_node + j * a.v_case]; };
  // per-case factorization, leaf-first (children before parents)
  bool any = false, bad = false;
  for (int k = 0; k < b; ++k) {
    const double2 s = Sk(k);
    const double az = __ldg(a.alpha + k), ap = __ldg(a.alpha + 2 * b + k);
    const double2 yd = __ldg(a.ydiag + k);
    a.Z[k * t + j] = make_double2(__fma_rn(az, s.x, yd.x), __fma_rn(-az, s.y, yd.y));
    if (ap != 0.0 && (s.x != 0.0 || s.y != 0.0)) any = true;
  }
  for (int k = 0; k < b; ++k) {
    const double2 piv = a.Z[k * t + j];
    const double n2 = __fma_rn(piv.x, piv.x, piv.y * piv.y);
    if (!(n2 > 0.0) || !isfinite(n2)) bad = true;
    const double rr = 1.0 / n2;
    const double2 ui = make_double2(piv.x * rr, -piv.y * rr);
    const double2 e = __ldg(a.e + k);
    const double2 g = cmulz(e, ui);
    a.UI[k * t + j] = ui;
    a.G[k * t + j] = g;
    const int p = __ldg(a.parent + k);
    if (p >= 0) {
      const double2 eg = cmulz(e, g);
      double2 pp = a.Z[p * t + j];
      pp.x -= eg.x;
      pp.y -= eg.y;
      a.Z[p * t + j] = pp;
    }
  }
  if (bad) atomicExch(a.status, 1);
  for (int k = 0; k < b; ++k) Vk(k) = a.v0 ? __ldg(a.v0 + __ldg(a.orig + k)) : a.v_flat;  // fpi.py:141-145
  int n = 0;
  bool met = false;
  while (n < a.max_iter) {
    // right-hand sides, then the up-sweep (leaf-first): Z[p] -= g_k z_k
    for (int k = 0; k < b; ++k) {
      double2 v = Vk(k);
      double m2 = __fma_rn(v.x, v.x, v.y * v.y);
      if (m2 < kZeroGuard2) {
        v = make_double2(kZeroGuard, 0.0);
        m2 = kZeroGuard * kZeroGuard;
      }
      const double r = 1.0 / m2;
      const double2 s = Sk(k);
      const double ai = __ldg(a.alpha + b + k), ap = __ldg(a.alpha + 2 * b + k);
      const double2 c = __ldg(a.src + k);
      const double ur = __fma_rn(s.x, v.x, s.y * v.y) * r, uim = __fma_rn(s.x, v.y, -(s.y * v.x)) * r;
      a.Z[k * t + j] = any ? make_double2(-(ap * ur + c.x + ai * s.x), -(ap * uim + c.y - ai * s.y))
                           : make_double2(-(c.x + ai * s.x), -(c.y - ai * s.y));
    }
    for (int k = 0; k < b; ++k) {
      const int p = __ldg(a.parent + k);
      if (p >= 0) {
        const double2 gz = cmulz(a.G[k * t + j], a.Z[k * t + j]);
        double2 zp = a.Z[p * t + j];
        zp.x -= gz.x;
        zp.y -= gz.y;
        a.Z[p * t + j] = zp;
      }
    }
    // down-sweep (parents first): w_k = z_k / U[k,k] - g_k w_parent; step test, update
    bool small = true, fin = true;
    for (int k = b - 1; k >= 0; --k) {
      double2 w = cmulz(a.Z[k * t + j], a.UI[k * t + j]);
      const int p = __ldg(a.parent + k);
      if (p >= 0) {
        const double2 gw = cmulz(a.G[k * t + j], a.Z[p * t + j]);
        w.x -= gw.x;
        w.y -= gw.y;
      }
      a.Z[k * t + j] = w;
      double2& vk = Vk(k);
      double2 v = vk;
      if (__fma_rn(v.x, v.x, v.y * v.y) < kZeroGuard2) v = make_double2(kZeroGuard, 0.0);
      const double dr = w.x - v.x, di = w.y - v.y;
      if (!(__fma_rn(dr, dr, di * di) < a.tol2)) small = false;
      if (!(isfinite(w.x) && isfinite(w.y))) fin = false;
      vk = w;
    }
    ++n;
    if (!any) {
      met = true;
      break;
    }
    if (!fin) break;
    if (small) {
      met = true;
      break;
    }
  }
  // ZIP residual: max_k |az s |v|^2 + ai s v + ap s + v conj(src + (Y v)_k)|
  for (int k = 0; k < b; ++k) {
    const double2 v = Vk(k);
    a.A[k * t + j] = cmulz(__ldg(a.ydiag + k), v);
  }
  for (int k = 0; k < b; ++k) {
    const int p = __ldg(a.parent + k);
    if (p >= 0) {
      const double2 e = __ldg(a.e + k);
      const double2 ep = cmulz(e, Vk(p)), ek = cmulz(e, Vk(k));
      double2 x = a.A[k * t + j];
      x.x += ep.x;
      x.y += ep.y;
      a.A[k * t + j] = x;
      double2 y = a.A[p * t + j];
      y.x += ek.x;
      y.y += ek.y;
      a.A[p * t + j] = y;
    }
  }
  double worst = 0.0;
  for (int k = 0; k < b; ++k) {
    const double2 v = Vk(k), s = Sk(k), c = __ldg(a.src + k), yv = a.A[k * t + j];
    const double az = __ldg(a.alpha + k), zi = __ldg(a.alpha + b + k), zp = __ldg(a.alpha + 2 * b + k);
    const double v2 = v.x * v.x + v.y * v.y;
    const double2 sv = cmulz(s, v);
    const double lr = az * s.x * v2 + zi * sv.x + zp * s.x, li = az * s.y * v2 + zi * sv.y + zp * s.y;
    const double ar = c.x + yv.x, aim = c.y + yv.y;  // a = src + Y v
    const double mr = lr + (v.x * ar + v.y * aim), mi = li + (v.y * ar - v.x * aim);
    worst = nanmax(worst, hypot(mr, mi));
  }
  a.iters[j] = n;
  a.resid[j] = worst;
  a.met[j] = met ? 1 : 0;
}

}  // namespace
}  // namespace tpf

extern "C" size_t tpf_sparse_zip_chain_workspace_bytes(int64_t tau, int32_t b) {
  return size_t(4) * size_t(tau) * size_t(b) * 16 + 256;
}

extern "C" int tpf_sparse_zip_chain_c128(int64_t tau, int32_t b, const int32_t* orig, const int32_t* parent,
                                         const double* e, const double* ydiag, const double* alpha,
                                         const double* src, const double* S, int64_t s_node_stride,
                                         int64_t s_case_stride, double v_flat_re, double v_flat_im, const double* v0,
                                         double tol, int32_t max_iter, double* V, int64_t v_node_stride, int64_t v_case_stride,
                                         int32_t* iters, double* resid, uint8_t* step_met, int32_t* status,
                                         void* workspace, size_t workspace_bytes, void* stream) {
  if (tau < 0 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_sparse_zip_chain_c128: need tau >= 0, b >= 1");
  if (!(tol > 0.0)) return set_error(TPF_ERR_INVALID, "tolerance must be positive");
  if (max_iter < 1) return set_error(TPF_ERR_INVALID, "max_iterations must be >= 1");
  if (tau == 0) return TPF_OK;
  if (!orig || !parent || !e || !ydiag || !alpha || !src || !S || !V || !iters || !resid || !step_met || !status ||
      !workspace)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_zip_chain_c128: null pointer");
  if (workspace_bytes < tpf_sparse_zip_chain_workspace_bytes(tau, b))
    return set_error(TPF_ERR_INVALID, "tpf_sparse_zip_chain_c128: workspace too small");
  ZipChainArgs a;
  a.tau = tau;
  a.b = b;
  a.S = reinterpret_cast<const double2*>(S);
  a.s_node = s_node_stride;
  a.s_case = s_case_stride;
  a.orig = orig;
  a.parent = parent;
  a.e = reinterpret_cast<const double2*>(e);
  a.ydiag = reinterpret_cast<const double2*>(ydiag);
  a.alpha = alpha;
  a.src = reinterpret_cast<const double2*>(src);
  a.v_flat = make_double2(v_flat_re, v_flat_im);
  a.v0 = reinterpret_cast<const double2*>(v0);
  a.tol2 = tol * tol;
  a.max_iter = max_iter;
  a.V = reinterpret_cast<double2*>(V);
  a.v_node = v_node_stride;
  a.v_case = v_case_stride;
  a.iters = iters;
  a.resid = resid;
  a.met = step_met;
  a.status = status;
  double2* w = static_cast<double2*>(workspace);
  const size_t plane = size_t(tau) * size_t(b);
  a.Z = w;
  a.G = w + plane;
  a.UI = w + 2 * plane;
  a.A = w + 3 * plane;
  const int threads = 128;
  const int64_t blocks = (tau + threads - 1) / threads;
  sparse_zip_chain_kernel<<<unsigned(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(a);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(sparse_zip_chain_kernel)", err);
  return TPF_OK;
}

// ZIP loads on meshed networks (the reference's per-case SuperLU route,
// dense.py:214-230 -> fpi.py:107-206): one thread per case, per-case LU of
// B = Y_dd + diag(alpha_z s*) on a fixed fill pattern (minimum-degree order of
// the symmetrised pattern, no pivoting; host schedule sparse.zip_lu_schedule)
// and fpi_solve's iteration as in the chain kernel above; the ZIP residual
// from Y_dd in CSR.  Scratch: the factor slots [nslot][tau] and one
// right-hand side [b][tau], case-minor so every slot access is coalesced.
namespace tpf {
namespace {

struct ZipLuArgs {
  int64_t tau;
  int b, nslot;
  const double2* S;
  int64_t s_node, s_case;  // original node order
  const int32_t* orig;     // elimination position k -> original node
  const int32_t* kinfo;    // [b][2]: later neighbours m_k, offset into idx
  const int32_t* idx;      // per step: positions[m], L slots[m], U slots[m], targets[m*m]
  const double2* base;     // [nslot] Y_dd at the factor slots
  const double* alpha;     // [3][b] elimination order
  const double2* src;      // elimination order
  const int32_t* rp;       // CSR of Y_dd (original order), residual
  const int32_t* ci;
  const double2* yv;
  double2 v_flat;
  const double2* v0;       // initial iterate (original node order) or null: flat start
  double tol2;
  int max_iter;
  double2* V;
  int64_t v_node, v_case;  // original node order
  int32_t* iters;
  double* resid;
  uint8_t* met;
  int32_t* status;
  double2 *F, *Z;
};

__global__ void __launch_bounds__(128) sparse_zip_lu_kernel(const ZipLuArgs a) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= a.tau) return;
  const int b = a.b;
  const int64_t t = a.tau;
  double2* F = a.F + j;
  double2* Z = a.Z + j;
  auto Sk = [&](int k) { return a.S[int64_t(__ldg(a.orig + k)) * a.s_node + j * a.s_case]; };
  auto Vn = [&](int node) -> double2& { return a.V[int64_t(node) * a.v_node + j * a.v_case]; };
  for (int s = 0; s < a.nslot; ++s) F[s * t] = __ldg(a.base + s);
  bool any = false, bad = false;
  for (int k = 0; k < b; ++k) {
    const double2 s = Sk(k);
    const double az = __ldg(a.alpha + k), ap = __ldg(a.alpha + 2 * b + k);
    const double2 yd = F[k * t];
    F[k * t] = make_double2(__fma_rn(az, s.x, yd.x), __fma_rn(-az, s.y, yd.y));
    if (ap != 0.0 && (s.x != 0.0 || s.y != 0.0)) any = true;
  }
  // right-looking elimination over the fixed pattern; slot k keeps 1 / U[k,k]
  for (int k = 0; k < b; ++k) {
    const double2 piv = F[k * t];
    const double n2 = __fma_rn(piv.x, piv.x, piv.y * piv.y);
    if (!(n2 > 0.0) || !isfinite(n2)) bad = true;
    const double rr = 1.0 / n2;
    const double2 ui = make_double2(piv.x * rr, -piv.y * rr);
    F[k * t] = ui;
    const int m = __ldg(a.kinfo + 2 * k), off = __ldg(a.kinfo + 2 * k + 1);
    const int32_t* ls = a.idx + off + m;
    const int32_t* us = ls + m;
    const int32_t* tg = us + m;
    for (int r = 0; r < m; ++r) {
      const int lr = __ldg(ls + r);
      const double2 l = cmulz(F[lr * t], ui);
      F[lr * t] = l;
      for (int c = 0; c < m; ++c) {
        const int tt = __ldg(tg + r * m + c);
        const double2 lu = cmulz(l, F[__ldg(us + c) * t]);
        double2 x = F[tt * t];
        x.x -= lu.x;
        x.y -= lu.y;
        F[tt * t] = x;
      }
    }
  }
  if (bad) atomicExch(a.status, 1);
  for (int k = 0; k < b; ++k) {  // fpi.py:141-145
    const int i = __ldg(a.orig + k);
    Vn(i) = a.v0 ? __ldg(a.v0 + i) : a.v_flat;
  }
  int n = 0;
  bool met = false;
  while (n < a.max_iter) {
    for (int k = 0; k < b; ++k) {
      double2 v = Vn(__ldg(a.orig + k));
      double m2 = __fma_rn(v.x, v.x, v.y * v.y);
      if (m2 < kZeroGuard2) {
        v = make_double2(kZeroGuard, 0.0);
        m2 = kZeroGuard * kZeroGuard;
      }
      const double r = 1.0 / m2;
      const double2 s = Sk(k);
      const double ai = __ldg(a.alpha + b + k), ap = __ldg(a.alpha + 2 * b + k);
      const double2 c = __ldg(a.src + k);
      const double ur = __fma_rn(s.x, v.x, s.y * v.y) * r, uim = __fma_rn(s.x, v.y, -(s.y * v.x)) * r;
      Z[k * t] = any ? make_double2(-(ap * ur + c.x + ai * s.x), -(ap * uim + c.y - ai * s.y))
                     : make_double2(-(c.x + ai * s.x), -(c.y - ai * s.y));
    }
    // forward (unit L), then backward (U) with the step test and the update
    for (int k = 0; k < b; ++k) {
      const int m = __ldg(a.kinfo + 2 * k), off = __ldg(a.kinfo + 2 * k + 1);
      const double2 zk = Z[k * t];
      for (int r = 0; r < m; ++r) {
        const int p = __ldg(a.idx + off + r);
        const double2 lz = cmulz(F[__ldg(a.idx + off + m + r) * t], zk);
        double2 x = Z[p * t];
        x.x -= lz.x;
        x.y -= lz.y;
        Z[p * t] = x;
      }
    }
    bool small = true, fin = true;
    for (int k = b - 1; k >= 0; --k) {
      const int m = __ldg(a.kinfo + 2 * k), off = __ldg(a.kinfo + 2 * k + 1);
      double2 acc = Z[k * t];
      for (int c = 0; c < m; ++c) {
        const double2 uz = cmulz(F[__ldg(a.idx + off + 2 * m + c) * t], Z[__ldg(a.idx + off + c) * t]);
        acc.x -= uz.x;
        acc.y -= uz.y;
      }
      const double2 w = cmulz(acc, F[k * t]);
      Z[k * t] = w;
      double2& vk = Vn(__ldg(a.orig + k));
      double2 v = vk;
      if (__fma_rn(v.x, v.x, v.y * v.y) < kZeroGuard2) v = make_double2(kZeroGuard, 0.0);
      const double dr = w.x - v.x, di = w.y - v.y;
      if (!(__fma_rn(dr, dr, di * di) < a.tol2)) small = false;
      if (!(isfinite(w.x) && isfinite(w.y))) fin = false;
      vk = w;
    }
    ++n;
    if (!any) {
      met = true;
      break;
    }
    if (!fin) break;
    if (small) {
      met = true;
      break;
    }
  }
  // ZIP residual: max_k |az s |v|^2 + ai s v + ap s + v conj(src + (Y v)_k)|
  double worst = 0.0;
  for (int k = 0; k < b; ++k) {
    const int node = __ldg(a.orig + k);
    double2 yv = make_double2(0.0, 0.0);
    for (int e = __ldg(a.rp + node); e < __ldg(a.rp + node + 1); ++e) {
      const double2 x = cmulz(__ldg(a.yv + e), Vn(__ldg(a.ci + e)));
      yv.x += x.x;
      yv.y += x.y;
    }
    const double2 v = Vn(node), s = Sk(k), c = __ldg(a.src + k);
    const double az = __ldg(a.alpha + k), zi = __ldg(a.alpha + b + k), zp = __ldg(a.alpha + 2 * b + k);
    const double v2 = v.x * v.x + v.y * v.y;
    const double2 sv = cmulz(s, v);
    const double lr = az * s.x * v2 + zi * sv.x + zp * s.x, li = az * s.y * v2 + zi * sv.y + zp * s.y;
    const double ar = c.x + yv.x, aim = c.y + yv.y;
    const double mr = lr + (v.x * ar + v.y * aim), mi = li + (v.y * ar - v.x * aim);
    worst = nanmax(worst, hypot(mr, mi));
  }
  a.iters[j] = n;
  a.resid[j] = worst;
  a.met[j] = met ? 1 : 0;
}

}  // namespace
}  // namespace tpf

extern "C" size_t tpf_sparse_zip_lu_workspace_bytes(int64_t tau, int32_t b, int32_t nslot) {
  return (size_t(nslot) + size_t(b)) * size_t(tau) * 16 + 256;
}

extern "C" int tpf_sparse_zip_lu_c128(int64_t tau, int32_t b, int32_t nslot, const int32_t* orig,
                                      const int32_t* kinfo, const int32_t* idx, const double* base,
                                      const double* alpha, const double* src, const int32_t* y_row_ptr,
                                      const int32_t* y_col, const double* y_val, const double* S,
                                      int64_t s_node_stride, int64_t s_case_stride, double v_flat_re,
                                      double v_flat_im, const double* v0, double tol, int32_t max_iter, double* V,
                                      int64_t v_node_stride, int64_t v_case_stride, int32_t* iters, double* resid,
                                      uint8_t* step_met, int32_t* status, void* workspace, size_t workspace_bytes,
                                      void* stream) {
  if (tau < 0 || b < 1 || nslot < b)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_zip_lu_c128: need tau >= 0, b >= 1, nslot >= b");
  if (!(tol > 0.0)) return set_error(TPF_ERR_INVALID, "tolerance must be positive");
  if (max_iter < 1) return set_error(TPF_ERR_INVALID, "max_iterations must be >= 1");
  if (tau == 0) return TPF_OK;
  if (!orig || !kinfo || !idx || !base || !alpha || !src || !y_row_ptr || !y_col || !y_val || !S || !V || !iters ||
      !resid || !step_met || !status || !workspace)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_zip_lu_c128: null pointer");
  if (workspace_bytes < tpf_sparse_zip_lu_workspace_bytes(tau, b, nslot))
    return set_error(TPF_ERR_INVALID, "tpf_sparse_zip_lu_c128: workspace too small");
  ZipLuArgs a;
  a.tau = tau;
  a.b = b;
  a.nslot = nslot;
  a.S = reinterpret_cast<const double2*>(S);
  a.s_node = s_node_stride;
  a.s_case = s_case_stride;
  a.orig = orig;
  a.kinfo = kinfo;
  a.idx = idx;
  a.base = reinterpret_cast<const double2*>(base);
  a.alpha = alpha;
  a.src = reinterpret_cast<const double2*>(src);
  a.rp = y_row_ptr;
  a.ci = y_col;
  a.yv = reinterpret_cast<const double2*>(y_val);
  a.v_flat = make_double2(v_flat_re, v_flat_im);
  a.v0 = reinterpret_cast<const double2*>(v0);
  a.tol2 = tol * tol;
  a.max_iter = max_iter;
  a.V = reinterpret_cast<double2*>(V);
  a.v_node = v_node_stride;
  a.v_case = v_case_stride;
  a.iters = iters;
  a.resid = resid;
  a.met = step_met;
  a.status = status;
  a.F = static_cast<double2*>(workspace);
  a.Z = a.F + size_t(nslot) * size_t(tau);
  const int threads = 128;
  const int64_t blocks = (tau + threads - 1) / threads;
  sparse_zip_lu_kernel<<<unsigned(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(a);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(sparse_zip_lu_kernel)", err);
  return TPF_OK;
}

// ZIP loads on small meshed networks with the pivoting of the reference's
// per-case SuperLU (fpi.py:119, splu's partial pivoting): one thread per case,
// B = Y_dd + diag(alpha_z s*) dense (b <= kZipDenseMaxB), LU with partial
// pivoting by rows (largest |.|^2 in the column, first on ties), then
// fpi_solve's iteration and ZIP residual exactly as sparse_zip_lu_kernel, in
// original node order.  Scratch, case-minor: the factors [b * b][tau], one
// right-hand side [b][tau] and the pivot rows [b][tau].
namespace tpf {
namespace {

constexpr int kZipDenseMaxB = 64;

__global__ void __launch_bounds__(128) sparse_zip_dense_kernel(const ZipLuArgs a, int32_t* __restrict__ piv) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= a.tau) return;
  const int b = a.b;
  const int64_t t = a.tau;
  double2* F = a.F + j;
  double2* Z = a.Z + j;
  int32_t* P = piv + j;
  auto A = [&](int r, int c) -> double2& { return F[(int64_t(r) * b + c) * t]; };
  auto Sk = [&](int k) { return a.S[int64_t(k) * a.s_node + j * a.s_case]; };
  auto Vn = [&](int node) -> double2& { return a.V[int64_t(node) * a.v_node + j * a.v_case]; };
  for (int s = 0; s < b * b; ++s) F[s * t] = __ldg(a.base + s);
  bool any = false, bad = false;
  for (int k = 0; k < b; ++k) {
    const double2 s = Sk(k);
    const double az = __ldg(a.alpha + k), ap = __ldg(a.alpha + 2 * b + k);
    const double2 yd = A(k, k);
    A(k, k) = make_double2(__fma_rn(az, s.x, yd.x), __fma_rn(-az, s.y, yd.y));
    if (ap != 0.0 && (s.x != 0.0 || s.y != 0.0)) any = true;
  }
  // right-looking LU with row pivoting; the diagonal keeps 1 / U[k,k]
  for (int k = 0; k < b; ++k) {
    int p = k;
    double best = -1.0;
    for (int r = k; r < b; ++r) {
      const double2 x = A(r, k);
      const double n2 = __fma_rn(x.x, x.x, x.y * x.y);
      if (n2 > best) {
        best = n2;
        p = r;
      }
    }
    P[k * t] = p;
    if (p != k)
      for (int c = 0; c < b; ++c) {
        const double2 x = A(k, c);
        A(k, c) = A(p, c);
        A(p, c) = x;
      }
    const double2 pv = A(k, k);
    const double n2 = __fma_rn(pv.x, pv.x, pv.y * pv.y);
    if (!(n2 > 0.0) || !isfinite(n2)) bad = true;
    const double rr = 1.0 / n2;
    const double2 ui = make_double2(pv.x * rr, -pv.y * rr);
    A(k, k) = ui;
    for (int r = k + 1; r < b; ++r) {
      const double2 l = cmulz(A(r, k), ui);
      A(r, k) = l;
      for (int c = k + 1; c < b; ++c) {
        const double2 lu = cmulz(l, A(k, c));
        double2 x = A(r, c);
        x.x -= lu.x;
        x.y -= lu.y;
        A(r, c) = x;
      }
    }
  }
  if (bad) atomicExch(a.status, 1);
  for (int k = 0; k < b; ++k) Vn(k) = a.v0 ? __ldg(a.v0 + k) : a.v_flat;  // fpi.py:141-145
  int n = 0;
  bool met = false;
  while (n < a.max_iter) {
    for (int k = 0; k < b; ++k) {
      double2 v = Vn(k);
      double m2 = __fma_rn(v.x, v.x, v.y * v.y);
      if (m2 < kZeroGuard2) {
        v = make_double2(kZeroGuard, 0.0);
        m2 = kZeroGuard * kZeroGuard;
      }
      const double r = 1.0 / m2;
      const double2 s = Sk(k);
      const double ai = __ldg(a.alpha + b + k), ap = __ldg(a.alpha + 2 * b + k);
      const double2 c = __ldg(a.src + k);
      const double ur = __fma_rn(s.x, v.x, s.y * v.y) * r, uim = __fma_rn(s.x, v.y, -(s.y * v.x)) * r;
      Z[k * t] = any ? make_double2(-(ap * ur + c.x + ai * s.x), -(ap * uim + c.y - ai * s.y))
                     : make_double2(-(c.x + ai * s.x), -(c.y - ai * s.y));
    }
    for (int k = 0; k < b; ++k) {  // the row swaps, in order
      const int p = P[k * t];
      if (p != k) {
        const double2 x = Z[k * t];
        Z[k * t] = Z[int64_t(p) * t];
        Z[int64_t(p) * t] = x;
      }
    }
    for (int k = 0; k < b; ++k) {  // forward (unit L)
      const double2 zk = Z[k * t];
      for (int r = k + 1; r < b; ++r) {
        const double2 lz = cmulz(A(r, k), zk);
        double2 x = Z[r * t];
        x.x -= lz.x;
        x.y -= lz.y;
        Z[r * t] = x;
      }
    }
    bool small = true, fin = true;
    for (int k = b - 1; k >= 0; --k) {  // backward (U), the step test and the update
      double2 acc = Z[k * t];
      for (int c = k + 1; c < b; ++c) {
        const double2 uz = cmulz(A(k, c), Z[c * t]);
        acc.x -= uz.x;
        acc.y -= uz.y;
      }
      const double2 w = cmulz(acc, A(k, k));
      Z[k * t] = w;
      double2& vk = Vn(k);
      double2 v = vk;
      if (__fma_rn(v.x, v.x, v.y * v.y) < kZeroGuard2) v = make_double2(kZeroGuard, 0.0);
      const double dr = w.x - v.x, di = w.y - v.y;
      if (!(__fma_rn(dr, dr, di * di) < a.tol2)) small = false;
      if (!(isfinite(w.x) && isfinite(w.y))) fin = false;
      vk = w;
    }
    ++n;
    if (!any) {
      met = true;
      break;
    }
    if (!fin) break;
    if (small) {
      met = true;
      break;
    }
  }
  // ZIP residual: max_k |az s |v|^2 + ai s v + ap s + v conj(src + (Y v)_k)|
  double worst = 0.0;
  for (int k = 0; k < b; ++k) {
    double2 yv = make_double2(0.0, 0.0);
    for (int e = __ldg(a.rp + k); e < __ldg(a.rp + k + 1); ++e) {
      const double2 x = cmulz(__ldg(a.yv + e), Vn(__ldg(a.ci + e)));
      yv.x += x.x;
      yv.y += x.y;
    }
    const double2 v = Vn(k), s = Sk(k), c = __ldg(a.src + k);
    const double az = __ldg(a.alpha + k), zi = __ldg(a.alpha + b + k), zp = __ldg(a.alpha + 2 * b + k);
    const double v2 = v.x * v.x + v.y * v.y;
    const double2 sv = cmulz(s, v);
    const double lr = az * s.x * v2 + zi * sv.x + zp * s.x, li = az * s.y * v2 + zi * sv.y + zp * s.y;
    const double ar = c.x + yv.x, aim = c.y + yv.y;
    const double mr = lr + (v.x * ar + v.y * aim), mi = li + (v.y * ar - v.x * aim);
    worst = nanmax(worst, hypot(mr, mi));
  }
  a.iters[j] = n;
  a.resid[j] = worst;
  a.met[j] = met ? 1 : 0;
}

}  // namespace
}  // namespace tpf

extern "C" int tpf_sparse_zip_dense_max_nodes(void) { return tpf::kZipDenseMaxB; }

extern "C" size_t tpf_sparse_zip_dense_workspace_bytes(int64_t tau, int32_t b) {
  return (size_t(b) * size_t(b) + size_t(b)) * size_t(tau) * 16 + size_t(b) * size_t(tau) * 4 + 512;
}

extern "C" int tpf_sparse_zip_dense_c128(int64_t tau, int32_t b, const double* y_dense, const double* alpha,
                                         const double* src, const int32_t* y_row_ptr, const int32_t* y_col,
                                         const double* y_val, const double* S, int64_t s_node_stride,
                                         int64_t s_case_stride, double v_flat_re, double v_flat_im, const double* v0,
                                         double tol, int32_t max_iter, double* V, int64_t v_node_stride,
                                         int64_t v_case_stride, int32_t* iters, double* resid, uint8_t* step_met,
                                         int32_t* status, void* workspace, size_t workspace_bytes, void* stream) {
  using namespace tpf;
  if (tau < 0 || b < 1 || b > kZipDenseMaxB)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_zip_dense_c128: need tau >= 0, 1 <= b <= 64");
  if (!(tol > 0.0)) return set_error(TPF_ERR_INVALID, "tolerance must be positive");
  if (max_iter < 1) return set_error(TPF_ERR_INVALID, "max_iterations must be >= 1");
  if (tau == 0) return TPF_OK;
  if (!y_dense || !alpha || !src || !y_row_ptr || !y_col || !y_val || !S || !V || !iters || !resid || !step_met ||
      !status || !workspace)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_zip_dense_c128: null pointer");
  if (workspace_bytes < tpf_sparse_zip_dense_workspace_bytes(tau, b))
    return set_error(TPF_ERR_INVALID, "tpf_sparse_zip_dense_c128: workspace too small");
  ZipLuArgs a;
  memset(&a, 0, sizeof a);
  a.tau = tau;
  a.b = b;
  a.nslot = b * b;
  a.S = reinterpret_cast<const double2*>(S);
  a.s_node = s_node_stride;
  a.s_case = s_case_stride;
  a.base = reinterpret_cast<const double2*>(y_dense);
  a.alpha = alpha;
  a.src = reinterpret_cast<const double2*>(src);
  a.rp = y_row_ptr;
  a.ci = y_col;
  a.yv = reinterpret_cast<const double2*>(y_val);
  a.v_flat = make_double2(v_flat_re, v_flat_im);
  a.v0 = reinterpret_cast<const double2*>(v0);
  a.tol2 = tol * tol;
  a.max_iter = max_iter;
  a.V = reinterpret_cast<double2*>(V);
  a.v_node = v_node_stride;
  a.v_case = v_case_stride;
  a.iters = iters;
  a.resid = resid;
  a.met = step_met;
  a.status = status;
  a.F = static_cast<double2*>(workspace);
  a.Z = a.F + size_t(b) * size_t(b) * size_t(tau);
  int32_t* piv = reinterpret_cast<int32_t*>(a.Z + size_t(b) * size_t(tau));
  const int threads = 128;
  const int64_t blocks = (tau + threads - 1) / threads;
  sparse_zip_dense_kernel<<<unsigned(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(a, piv);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(sparse_zip_dense_kernel)", err);
  return TPF_OK;
}
