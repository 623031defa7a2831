// Dependent-chain latency of DFMA, MUFU.RCP64H, DADD, FFMA and an LDS pointer chase (one warp).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build_timing/lat_probe tools/lat_probe.cu
// Measured on B200: DFMA 8.5, MUFU.RCP64H 18.8, DADD 8.4, FFMA 4.9 (loop-bound), LDS 29.0 cycles.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double x = a, y = b;
  long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 125; ++i) { _Pragma("unroll") for (int u = 0; u < 8; ++u) x = __fma_rn(x, y, a); }
  long long t1 = clock64();
  double r = x;
  #pragma unroll 1
  for (int i = 0; i < 125; ++i) { _Pragma("unroll") for (int u = 0; u < 8; ++u) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(r)); }
  long long t2 = clock64();
  double s = x;
  #pragma unroll 1
  for (int i = 0; i < 125; ++i) { _Pragma("unroll") for (int u = 0; u < 8; ++u) s = s + y; }
  long long t3 = clock64();
  float f = (float)a;
  #pragma unroll 1
  for (int i = 0; i < 125; ++i) { _Pragma("unroll") for (int u = 0; u < 8; ++u) f = __fmaf_rn(f, (float)y, (float)a); }
  long long t4 = clock64();
  out[threadIdx.x] = x + r + s + f;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
// shared memory load latency chain
__global__ void k2(long long* cyc) {
  __shared__ unsigned idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  unsigned p = threadIdx.x;
  long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 125; ++i) { _Pragma("unroll") for (int u = 0; u < 8; ++u) p = idx[p]; }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[4] = t1 - t0; cyc[5] = p; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024*8); cudaMalloc(&c, 64);
  k<<<1, 32>>>(o, c, 1.0000001, 0.9999999);
  k2<<<1, 32>>>(c);
  long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("per-op latency (cycles): DFMA %.1f  MUFU.RCP64H %.1f  DADD %.1f  FFMA %.1f  LDS %.1f\n", h[0]/1000.0, h[1]/1000.0, h[2]/1000.0, h[3]/1000.0, h[4]/1000.0);
  return 0;
}
