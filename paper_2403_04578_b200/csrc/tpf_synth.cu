// Device scenario generator: the reference's load model
// (synth.py:131-156) for batches that only exist on the device (config C4:
// 1,000 scenarios x 525,600 cases).
//
// Per case j and node i: latent = sqrt(rho) common_j + sqrt(1 - rho) idio_ij
// (standard normals), p = base_i exp(sigma latent), power factor pf ~ U[0.9, 1]
// lagging, q = p tan(arccos pf) = p sqrt(1 - pf^2) / pf; then the whole batch
// is scaled so the worst aggregate |sum_i s_ij| is scale_num (load_scale x
// the solvability margin).  The draws come from a Philox4x32-10 counter
// generator keyed by the scenario's seed, counter (case, node pair, stream), so any
// case's loads are the same whatever the launch geometry or chunking.  Pass 1
// writes the unscaled loads (one 16-byte store per element, coalesced over
// cases) and the worst aggregate (atomicMax on the bits of non-negative
// doubles); pass 2 scales them in place (HBM-bound, cheaper than drawing
// them again).
// Statistically the reference's model, not bit-identical to numpy's PCG64.
#include "tpf_common.cuh"
#include "tpf_internal.h"

namespace tpf {
namespace {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// 53-bit uniform in the open interval (0, 1)
__device__ __forceinline__ double u01(uint32_t a, uint32_t b) {
  return (double(a >> 5) * 67108864.0 + double(b >> 6) + 0.5) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ double normal(uint4 w) {  // Box-Muller, one of the pair
  return sqrt(-2.0 * log(u01(w.x, w.y))) * cospi(2.0 * u01(w.z, w.w));
}

struct GenArgs {
  int64_t tau, case_offset;
  int b;
  const double* base;
  double a_common, a_idio, sigma, scale_num;
  uint2 key;
  double2* S;
  int64_t s_node, s_case;
  unsigned long long* worst;  // bits of the worst aggregate
};

__global__ void __launch_bounds__(256) gen_loads_kernel(const GenArgs a) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  double sr = 0.0, si = 0.0;
  if (j < a.tau) {
    const uint32_t cj = uint32_t(a.case_offset + j);
    const double common = normal(philox4x32_10(make_uint4(cj, 0xFFFFFFFFu, 2u, 0u), a.key));
    // nodes in pairs: one Box-Muller draw gives both idiosyncratic normals, one
    // Philox block both power factors
    for (int i0 = 0; i0 < a.b; i0 += 2) {
      const uint32_t pair = uint32_t(i0 >> 1);
      const uint4 wn = philox4x32_10(make_uint4(cj, pair, 0u, 0u), a.key);
      const uint4 wp = philox4x32_10(make_uint4(cj, pair, 1u, 0u), a.key);
      const double r = sqrt(-2.0 * log(u01(wn.x, wn.y)));
      double sn, cs;
      sincospi(2.0 * u01(wn.z, wn.w), &sn, &cs);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = i0 + h;
        if (i >= a.b) break;
        const double idio = r * (h == 0 ? cs : sn);
        const double pf = 0.9 + 0.1 * (h == 0 ? u01(wp.x, wp.y) : u01(wp.z, wp.w));
        const double p = __ldg(a.base + i) * exp(a.sigma * (a.a_common * common + a.a_idio * idio));
        const double q = p * (sqrt((1.0 - pf) * (1.0 + pf)) / pf);
        a.S[int64_t(i) * a.s_node + j * a.s_case] = make_double2(p, q);
        sr += p;
        si += q;
      }
    }
  }
  double m = j < a.tau ? hypot(sr, si) : 0.0;
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(a.worst, __double_as_longlong(m));
}

// s *= scale_num / worst (the reference's `s *= load_scale * margin / worst`)
__global__ void __launch_bounds__(256) scale_loads_kernel(const GenArgs a) {
  const double f = a.scale_num / __longlong_as_double(*a.worst);
  const int64_t n = a.tau * a.b;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / a.tau, j = e - i * a.tau;
    double2* p = a.S + i * a.s_node + j * a.s_case;
    const double2 v = *p;
    *p = make_double2(v.x * f, v.y * f);
  }
}

}  // namespace
}  // namespace tpf

using namespace tpf;

extern "C" size_t tpf_gen_loads_workspace_bytes(void) { return 256; }

extern "C" int tpf_gen_loads_c128(int64_t tau, int32_t b, const double* base, double rho, double sigma,
                                  uint64_t key, int64_t case_offset, double scale_num, double* S,
                                  int64_t s_node_stride, int64_t s_case_stride, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  if (tau < 1 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_gen_loads_c128: need tau >= 1, b >= 1");
  if (!(rho >= 0.0 && rho < 1.0)) return set_error(TPF_ERR_INVALID, "tpf_gen_loads_c128: correlation in [0, 1)");
  if (case_offset < 0 || case_offset + tau > (int64_t(1) << 32))
    return set_error(TPF_ERR_INVALID, "tpf_gen_loads_c128: case index beyond 2^32");
  if (!base || !S || !workspace || workspace_bytes < 256)
    return set_error(TPF_ERR_INVALID, "tpf_gen_loads_c128: null pointer or small workspace");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  GenArgs a;
  a.tau = tau;
  a.case_offset = case_offset;
  a.b = b;
  a.base = base;
  a.a_common = sqrt(rho);
  a.a_idio = sqrt(1.0 - rho);
  a.sigma = sigma;
  a.scale_num = scale_num;
  a.key = make_uint2(uint32_t(key), uint32_t(key >> 32));
  a.S = reinterpret_cast<double2*>(S);
  a.s_node = s_node_stride;
  a.s_case = s_case_stride;
  a.worst = static_cast<unsigned long long*>(workspace);
  cudaError_t err = cudaMemsetAsync(workspace, 0, 8, st);
  if (err != cudaSuccess) return set_cuda_error("cudaMemsetAsync(worst)", err);
  const unsigned blocks = unsigned((tau + 255) / 256);
  gen_loads_kernel<<<blocks, 256, 0, st>>>(a);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  scale_loads_kernel<<<unsigned(sms) * 8, 256, 0, st>>>(a);
  err = cudaGetLastError();
  return err == cudaSuccess ? TPF_OK : set_cuda_error("launch(gen_loads_kernel)", err);
}
