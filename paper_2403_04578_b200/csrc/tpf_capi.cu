// C-ABI plumbing of libtpf.so: error state, residual and summary kernels,
// and the FP64 tensor-core peak probe used as the dense roofline denominator.
#include <cstdio>
#include <string>

#include "tpf_common.cuh"
#include "tpf_internal.h"

namespace tpf {

static thread_local std::string g_last_error;

int set_error(int code, const char* msg) {
  g_last_error = msg ? msg : "";
  return code;
}

int set_cuda_error(const char* where, cudaError_t err) {
  g_last_error = std::string(where) + ": " + cudaGetErrorName(err) + ": " + cudaGetErrorString(err);
  return TPF_ERR_CUDA;
}

// residual_per_case (fpi.py:221-240): one thread per case; Y_dd rows are read
// uniformly by the warp (broadcast), V/S accesses coalesce over cases when the
// case stride is 1 (the reference's b x tau layout).
// Batches too small to fill the GPU one thread per case (C5: 8,760 cases of
// b = 1,000) split the rows over blockIdx.y: each thread takes rows [i0, i1)
// of its case and the per-case maximum is an atomicMax on the bits of the
// non-negative partial maxima (their order as unsigned integers is the numeric
// order, and NaN's patterns sort above every number, as nanmax keeps NaN), so
// the result is the same number as the single-thread row loop.
__global__ void residual_kernel(int64_t tau, int b, const double* __restrict__ S, int64_t sn, int64_t sc,
                                const double* __restrict__ V, int64_t vn, int64_t vc,
                                const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double* __restrict__ yv, const double* __restrict__ src,
                                const int32_t* __restrict__ order, double* __restrict__ resid) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= tau) return;
  const int nrb = int(gridDim.y);
  const int i0 = int(int64_t(b) * blockIdx.y / nrb), i1 = int(int64_t(b) * (blockIdx.y + 1) / nrb);
  double worst = 0.0;
  for (int ii = i0; ii < i1; ++ii) {
    // rows in `order` (a depth-first order of a radial feeder: a row's
    // neighbours were read moments ago and still sit in L1); the maximum does
    // not depend on the order of the rows
    const int i = order ? __ldg(order + ii) : ii;
    const double2 si = ldg_c128(src, i);
    double ar = si.x, ai = si.y;
    for (int k = __ldg(rp + i); k < __ldg(rp + i + 1); ++k) {
      const double2 y = ldg_c128(yv, k);
      const double2 v = ldg_c128(V, int64_t(__ldg(ci + k)) * vn + j * vc);
      ar = __fma_rn(y.x, v.x, __fma_rn(-y.y, v.y, ar));
      ai = __fma_rn(y.x, v.y, __fma_rn(y.y, v.x, ai));
    }
    const double2 v = ldg_c128(V, int64_t(i) * vn + j * vc);
    const double2 s = ldg_c128(S, int64_t(i) * sn + j * sc);
    // s + v * conj(a)
    const double mr = s.x + (v.x * ar + v.y * ai);
    const double mi = s.y + (v.y * ar - v.x * ai);
    worst = nanmax(worst, hypot(mr, mi));
  }
  if (nrb == 1) {
    resid[j] = worst;
  } else {
    atomicMax(reinterpret_cast<unsigned long long*>(resid) + j, __double_as_longlong(worst));
  }
}

__global__ void summary_kernel(int64_t tau, const int32_t* __restrict__ iters, const double* __restrict__ resid,
                               double rtol, uint8_t* __restrict__ mask, int32_t* __restrict__ out) {
  int local_max = 0, local_conv = 0;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < tau; j += int64_t(gridDim.x) * blockDim.x) {
    const double r = resid[j];
    const bool ok = isfinite(r) && r < rtol;
    if (mask) mask[j] = ok ? 1 : 0;
    local_max = max(local_max, iters[j]);
    local_conv += ok ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) {
    local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
    local_conv += __shfl_xor_sync(0xffffffffu, local_conv, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, local_max);
    atomicAdd(out + 1, local_conv);
  }
}

// DMMA-only throughput probe: 8 independent accumulators per warp.
__global__ void dmma_probe_kernel(double* out, int iters) {
  double a = 1e-3 + threadIdx.x * 1e-9, bb = 1e-3;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(bb));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace tpf

using namespace tpf;

extern "C" int tpf_version(void) { return 100; }

extern "C" const char* tpf_last_error(void) { return g_last_error.c_str(); }

extern "C" int tpf_residual_order_c128(int64_t tau, int32_t b, const double* S, int64_t s_node_stride,
                                       int64_t s_case_stride, const double* V, int64_t v_node_stride,
                                       int64_t v_case_stride, const int32_t* ydd_row_ptr, const int32_t* ydd_col,
                                       const double* ydd_val, const double* src, const int32_t* row_order,
                                       double* resid, void* stream);

extern "C" int tpf_residual_c128(int64_t tau, int32_t b, const double* S, int64_t s_node_stride,
                                 int64_t s_case_stride, const double* V, int64_t v_node_stride,
                                 int64_t v_case_stride, const int32_t* ydd_row_ptr, const int32_t* ydd_col,
                                 const double* ydd_val, const double* src, double* resid, void* stream) {
  return tpf_residual_order_c128(tau, b, S, s_node_stride, s_case_stride, V, v_node_stride, v_case_stride,
                                 ydd_row_ptr, ydd_col, ydd_val, src, nullptr, resid, stream);
}

extern "C" int tpf_residual_order_c128(int64_t tau, int32_t b, const double* S, int64_t s_node_stride,
                                       int64_t s_case_stride, const double* V, int64_t v_node_stride,
                                       int64_t v_case_stride, const int32_t* ydd_row_ptr, const int32_t* ydd_col,
                                       const double* ydd_val, const double* src, const int32_t* row_order,
                                       double* resid, void* stream) {
  if (tau < 0 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_residual_c128: need tau >= 0, b >= 1");
  if (tau == 0) return TPF_OK;
  if (!S || !V || !ydd_row_ptr || !ydd_col || !ydd_val || !src || !resid)
    return set_error(TPF_ERR_INVALID, "tpf_residual_c128: null pointer");
  const int threads = 256;
  const int64_t blocks = (tau + threads - 1) / threads;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // row blocks: enough threads for ~8 resident warps per scheduler on every SM,
  // at least 16 rows each
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t nrb = (int64_t(sms) * 2048 + tau - 1) / tau;
  if (nrb > b / 16) nrb = b / 16;
  if (const char* e = getenv("TPF_RESID_NRB")) nrb = atoi(e);  // A/B knob (tools/c2_resid_probe.py)
  if (nrb > b) nrb = b;
  if (nrb > 65535) nrb = 65535;
  if (nrb < 1) nrb = 1;
  if (nrb > 1) {
    cudaError_t e = cudaMemsetAsync(resid, 0, size_t(tau) * sizeof(double), st);  // +0.0: nanmax's start
    if (e != cudaSuccess) return set_cuda_error("cudaMemsetAsync(resid)", e);
  }
  residual_kernel<<<dim3(unsigned(blocks), unsigned(nrb)), threads, 0, st>>>(
      tau, b, S, s_node_stride, s_case_stride, V, v_node_stride, v_case_stride, ydd_row_ptr, ydd_col, ydd_val,
      src, row_order, resid);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(residual_kernel)", err);
  return TPF_OK;
}

extern "C" int tpf_batch_summary(int64_t tau, const int32_t* iters, const double* resid, double residual_tol,
                                 uint8_t* mask, int32_t* out, void* stream) {
  if (tau < 0 || !iters || !resid || !out) return set_error(TPF_ERR_INVALID, "tpf_batch_summary: bad argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t err = cudaMemsetAsync(out, 0, 2 * sizeof(int32_t), st);
  if (err != cudaSuccess) return set_cuda_error("cudaMemsetAsync(summary)", err);
  if (tau == 0) return TPF_OK;
  int64_t blocks = (tau + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  summary_kernel<<<unsigned(blocks), 256, 0, st>>>(tau, iters, resid, residual_tol, mask, out);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(summary_kernel)", err);
  return TPF_OK;
}

extern "C" int tpf_probe_fp64_tflops(double* tflops_out, double* ms_out) {
  int dev = 0, sms = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return set_cuda_error("cudaGetDevice", err);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int warps = 16, threads = 32 * warps, iters = 8000;
  double* out = nullptr;
  err = cudaMalloc(&out, sizeof(double) * size_t(sms) * threads);
  if (err != cudaSuccess) return set_cuda_error("cudaMalloc(probe)", err);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    dmma_probe_kernel<<<sms, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (err != cudaSuccess) return set_cuda_error("dmma_probe_kernel", err);
  const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * warps * sms;
  if (tflops_out) *tflops_out = flops / (double(best) * 1e-3) / 1e12;
  if (ms_out) *ms_out = best;
  return TPF_OK;
}

// ---------------------------------------------------------------------------
// Per-node voltage statistics of a solved batch (probabilistic power flow,
// config C4: the scenario batches are reduced on the device instead of being
// copied out).  Pass 1: one CTA per (node, 65,536-case block) reduces
// min / max / sum of |V| with a fixed thread-to-case mapping and a fixed
// shuffle tree; pass 2: one thread per node folds the blocks in order into
// the running arrays.  No atomics: the statistics are bit-reproducible.
namespace tpf {
namespace {
constexpr int kStatBlock = 65536;

__global__ void __launch_bounds__(256) vstats_partial_kernel(int64_t tau, const double2* __restrict__ V, int64_t vn,
                                                             int64_t vc, double* __restrict__ part) {
  const int i = blockIdx.x;
  const int64_t lo = int64_t(blockIdx.y) * kStatBlock;
  const int64_t hi = lo + kStatBlock < tau ? lo + kStatBlock : tau;
  double mn = INFINITY, mx = -INFINITY, sm = 0.0;
  for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) {
    const double2 v = V[int64_t(i) * vn + j * vc];
    const double a = hypot(v.x, v.y);  // |V| as numpy's abs (hypot)
    mn = fmin(mn, a);
    mx = fmax(mx, a);
    sm += a;
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
  }
  __shared__ double s[3][8];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s[0][w] = mn;
    s[1][w] = mx;
    s[2][w] = sm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < 8; ++k) {
      mn = fmin(mn, s[0][k]);
      mx = fmax(mx, s[1][k]);
      sm += s[2][k];
    }
    double* o = part + (int64_t(i) * gridDim.y + blockIdx.y) * 3;
    o[0] = mn;
    o[1] = mx;
    o[2] = sm;
  }
}

__global__ void vstats_fold_kernel(int b, int nblk, const double* __restrict__ part, double* vmin, double* vmax,
                                   double* vsum, int accumulate) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b) return;
  double mn = accumulate ? vmin[i] : INFINITY, mx = accumulate ? vmax[i] : -INFINITY, sm = accumulate ? vsum[i] : 0.0;
  for (int k = 0; k < nblk; ++k) {
    const double* p = part + (int64_t(i) * nblk + k) * 3;
    mn = fmin(mn, p[0]);
    mx = fmax(mx, p[1]);
    sm += p[2];
  }
  vmin[i] = mn;
  vmax[i] = mx;
  vsum[i] = sm;
}
}  // namespace
}  // namespace tpf

extern "C" size_t tpf_voltage_stats_workspace_bytes(int64_t tau, int32_t b) {
  const int64_t nblk = (tau + kStatBlock - 1) / kStatBlock;
  return size_t(b > 0 ? b : 0) * size_t(nblk > 0 ? nblk : 0) * 3 * sizeof(double) + 256;
}

extern "C" int tpf_voltage_stats_c128(int64_t tau, int32_t b, const double* V, int64_t v_node_stride,
                                      int64_t v_case_stride, double* vmin, double* vmax, double* vsum,
                                      int32_t accumulate, void* workspace, size_t workspace_bytes, void* stream) {
  if (tau < 1 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_voltage_stats_c128: need tau >= 1 and b >= 1");
  if (!V || !vmin || !vmax || !vsum || !workspace)
    return set_error(TPF_ERR_INVALID, "tpf_voltage_stats_c128: null pointer");
  if (workspace_bytes < tpf_voltage_stats_workspace_bytes(tau, b))
    return set_error(TPF_ERR_INVALID, "tpf_voltage_stats_c128: workspace too small");
  const int64_t nblk = (tau + kStatBlock - 1) / kStatBlock;
  if (nblk > 65535) return set_error(TPF_ERR_INVALID, "tpf_voltage_stats_c128: tau too large for one call");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* part = static_cast<double*>(workspace);
  vstats_partial_kernel<<<dim3(unsigned(b), unsigned(nblk)), 256, 0, st>>>(
      tau, reinterpret_cast<const double2*>(V), v_node_stride, v_case_stride, part);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(vstats_partial_kernel)", err);
  vstats_fold_kernel<<<(b + 127) / 128, 128, 0, st>>>(b, int(nblk), part, vmin, vmax, vsum, accumulate);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(vstats_fold_kernel)", err);
  return TPF_OK;
}
