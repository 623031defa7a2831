// DMMA issue rate of ONE warp per SM sub-partition vs number of independent accumulators.
#include <cstdio>
#include <cuda_runtime.h>
template <int NACC>
__global__ void k(double* out, int iters) {
  double a = 1e-3 + threadIdx.x * 1e-9, b = 1e-3;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NACC>
void run(double* out, int warps) {
  const int iters = 32768 / NACC;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms = 0;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); k<NACC><<<148, 32 * warps>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  double dmma = double(iters) * NACC * warps * 148;
  double tf = dmma * 512 / (ms * 1e-3) / 1e12;
  printf("warps/SM %2d  acc/warp %2d  %.2f TF  clk/DMMA/SMSP %.1f\n", warps, NACC, tf, (ms * 1e-3 * 1.965e9) / (dmma / 148 / 4));
}
int main() {
  double* out; cudaMalloc(&out, 1 << 24);
  run<1>(out, 4); run<2>(out, 4); run<4>(out, 4); run<8>(out, 4); run<12>(out, 4); run<16>(out, 4); run<24>(out, 4); run<32>(out, 4);
  run<4>(out, 8); run<8>(out, 8); run<16>(out, 8);
  return 0;
}
