// The persistent tail's consumer loop in isolation: per slab, 16 operand pairs
// loaded from shared memory (complex rows at the kernel's strides, one part
// read per chain) ahead of 16 dependent DMMAs.  Warps 0-2 = chains P1..P3.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_slab_bin tools/dmma_slab.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int W, int ROWA, int ROWB, bool PLANAR>
__device__ void run(const unsigned char* sm, int nslab, double& p0, double& p1) {
  const int lane = threadIdx.x & 31;
  for (int sl = 0; sl < nslab; ++sl) {
    const int s = sl & 7;
    double x[16], y[16];
#pragma unroll
    for (int ks = 0; ks < 16; ++ks) {
      if (PLANAR) {
        const double* a = reinterpret_cast<const double*>(sm + (lane >> 2) * ROWA + ((s * 16 + ks) * 4 + (lane & 3)) * 8);
        const double* b = reinterpret_cast<const double*>(sm + 65536 + (lane >> 2) * ROWB + ((s * 16 + ks) * 4 + (lane & 3)) * 8);
        x[ks] = W == 2 ? a[0] + a[4096] : a[0];
        y[ks] = W == 2 ? b[0] + b[4096] : b[0];
      } else {
        const double2 a = *reinterpret_cast<const double2*>(sm + (lane >> 2) * ROWA + ((s * 16 + ks) * 4 + (lane & 3)) * 16);
        const double2 b = *reinterpret_cast<const double2*>(sm + 65536 + (lane >> 2) * ROWB + ((s * 16 + ks) * 4 + (lane & 3)) * 16);
        x[ks] = W == 0 ? a.x : W == 1 ? a.y : a.x + a.y;
        y[ks] = W == 0 ? b.x : W == 1 ? b.y : b.x + b.y;
      }
    }
#pragma unroll
    for (int ks = 0; ks < 16; ++ks) dmma(p0, p1, x[ks], y[ks]);
  }
}

template <bool PLANAR>
__global__ void slab_kernel(double* out, long long* cyc, int nslab) {
  extern __shared__ __align__(16) unsigned char sm[];
  for (int i = threadIdx.x; i < 200 * 1024 / 8; i += blockDim.x) reinterpret_cast<double*>(sm)[i] = 1e-3 * (i % 7);
  __syncthreads();
  double p0 = 0, p1 = 0;
  const long long t0 = clock64();
  const int w = threadIdx.x >> 5;
  if (w == 0) run<0, 8192 + 64, 8192 + 64, PLANAR>(sm, nslab, p0, p1);
  else if (w == 1) run<1, 8192 + 64, 8192 + 64, PLANAR>(sm, nslab, p0, p1);
  else if (w == 2) run<2, 8192 + 64, 8192 + 64, PLANAR>(sm, nslab, p0, p1);
  const long long t1 = clock64();
  out[threadIdx.x] = p0 + p1;
  if ((threadIdx.x & 31) == 0 && w < 3) cyc[w] = t1 - t0;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 1024);
  const int nslab = 256;
  for (int planar = 0; planar < 2; ++planar) {
    auto k = planar ? slab_kernel<true> : slab_kernel<false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int rep = 0; rep < 2; ++rep) { k<<<1, 96, 200 * 1024>>>(out, cyc, nslab); cudaDeviceSynchronize(); }
    printf("%s: cycles per DMMA  P1 %.1f  P2 %.1f  P3 %.1f\n", planar ? "planar" : "complex", double(cyc[0]) / (nslab * 16),
           double(cyc[1]) / (nslab * 16), double(cyc[2]) / (nslab * 16));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
