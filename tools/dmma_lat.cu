// DMMA.8x8x4 dependent-chain latency and issue interval on one SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_lat tools/dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void chain(double* out, long long* cyc, int n, double a, double b) {
  double c[CHAINS][2];
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = 0.0;
  __syncwarp();
  const long long t0 = clock64();
  for (int k = 0; k < n; ++k) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  __syncwarp();
  const long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main2();
int main() {
  main2();
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 1024);
  const int n = 4096;
  chain<1><<<1, 32>>>(out, cyc, n, 1.0, 1e-3); cudaDeviceSynchronize();
  chain<1><<<1, 32>>>(out, cyc, n, 1.0, 1e-3); cudaDeviceSynchronize();
  printf("1 chain:  %.1f cycles per DMMA\n", double(cyc[0]) / n);
  chain<2><<<1, 32>>>(out, cyc, n, 1.0, 1e-3); cudaDeviceSynchronize();
  printf("2 chains: %.1f cycles per step (%.1f per DMMA)\n", double(cyc[0]) / n, double(cyc[0]) / n / 2);
  chain<4><<<1, 32>>>(out, cyc, n, 1.0, 1e-3); cudaDeviceSynchronize();
  printf("4 chains: %.1f cycles per step (%.1f per DMMA)\n", double(cyc[0]) / n, double(cyc[0]) / n / 4);
  chain<8><<<1, 32>>>(out, cyc, n, 1.0, 1e-3); cudaDeviceSynchronize();
  printf("8 chains: %.1f cycles per step (%.1f per DMMA)\n", double(cyc[0]) / n, double(cyc[0]) / n / 8);
  chain<1><<<1, 128>>>(out, cyc, n, 1.0, 1e-3); cudaDeviceSynchronize();
  printf("4 warps x 1 chain: %.1f cycles per DMMA per warp\n", double(cyc[0]) / n);
  return 0;
}

// operands streamed from shared memory, one load pair per DMMA (the tail chain's pattern)
__global__ void chain_lds(double* out, long long* cyc, int n) {
  __shared__ double sa[16 * 32], sb[16 * 32];
  for (int i = threadIdx.x; i < 16 * 32; i += 32) sa[i] = 1.0 + i * 1e-6, sb[i] = 1e-3;
  __syncwarp();
  double c0 = 0, c1 = 0;
  const long long t0 = clock64();
  for (int k = 0; k < n / 16; ++k) {
#pragma unroll
    for (int s = 0; s < 16; ++s) dmma(c0, c1, sa[s * 32 + threadIdx.x], sb[s * 32 + threadIdx.x]);
  }
  __syncwarp();
  const long long t1 = clock64();
  out[threadIdx.x] = c0 + c1;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// same, with the 16 operand pairs loaded into registers before the 16 DMMAs
__global__ void chain_lds_pre(double* out, long long* cyc, int n) {
  __shared__ double sa[16 * 32], sb[16 * 32];
  for (int i = threadIdx.x; i < 16 * 32; i += 32) sa[i] = 1.0 + i * 1e-6, sb[i] = 1e-3;
  __syncwarp();
  double c0 = 0, c1 = 0;
  const long long t0 = clock64();
  for (int k = 0; k < n / 16; ++k) {
    double x[16], y[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x[s]) : "r"((unsigned)__cvta_generic_to_shared(&sa[s * 32 + threadIdx.x])));
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(y[s]) : "r"((unsigned)__cvta_generic_to_shared(&sb[s * 32 + threadIdx.x])));
    }
    double acc = 0;
#pragma unroll
    for (int s = 0; s < 16; ++s) dmma(c0, c1, x[s], y[s]);
  }
  __syncwarp();
  const long long t1 = clock64();
  out[threadIdx.x] = c0 + c1;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main2() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 1024);
  const int n = 4096;
  chain_lds<<<1, 32>>>(out, cyc, n); cudaDeviceSynchronize();
  chain_lds<<<1, 32>>>(out, cyc, n); cudaDeviceSynchronize();
  printf("lds-fed chain: %.1f cycles per DMMA\n", double(cyc[0]) / n);
  chain_lds_pre<<<1, 32>>>(out, cyc, n); cudaDeviceSynchronize();
  printf("preloaded chain: %.1f cycles per DMMA\n", double(cyc[0]) / n);
  return 0;
}
