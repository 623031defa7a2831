// One warp per SMSP: DMMA cadence with an LDS.128 every 4 DMMAs (the dense kernel's mix).
#include <cstdio>
#include <cuda_runtime.h>
template <int NB, bool LDS>
__global__ void k(double* out, int iters) {
  __shared__ double2 sm[NB * 32 * 4];
  for (int i = threadIdx.x; i < NB * 32 * 4; i += blockDim.x) sm[i] = make_double2(1e-3 * i, 2e-3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double ur = 1e-3 + lane * 1e-9, ui = 2e-3, nui = -ui;
  double vr[NB][2], vi[NB][2];
#pragma unroll
  for (int i = 0; i < NB; ++i) vr[i][0] = vr[i][1] = vi[i][0] = vi[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int lb = 0; lb < NB; ++lb) {
      double2 kf = LDS ? sm[(lb * 4 + (it & 3)) * 32 + lane] : make_double2(ur, ui);
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(vr[lb][0]), "+d"(vr[lb][1]) : "d"(ur), "d"(kf.x));
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(vi[lb][0]), "+d"(vi[lb][1]) : "d"(ur), "d"(kf.y));
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(vr[lb][0]), "+d"(vr[lb][1]) : "d"(nui), "d"(kf.y));
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(vi[lb][0]), "+d"(vi[lb][1]) : "d"(ui), "d"(kf.x));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NB; ++i) s += vr[i][0] + vr[i][1] + vi[i][0] + vi[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NB, bool LDS>
void run(double* out, int warps) {
  const int iters = 2048;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms = 0;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); k<NB, LDS><<<148, 32 * warps>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  double dmma = double(iters) * NB * 4 * warps * 148;
  printf("warps/SM %d NB %2d lds %d: %.2f TF  clk/DMMA/SMSP %.1f\n", warps, NB, int(LDS), dmma * 512 / (ms * 1e-3) / 1e12,
         (ms * 1e-3 * 1.965e9) / (dmma / 148 / 4));
}
int main() {
  double* out; cudaMalloc(&out, 1 << 24);
  run<13, false>(out, 4); run<13, true>(out, 4); run<7, true>(out, 4); run<7, true>(out, 8); run<13, true>(out, 8);
  return 0;
}
