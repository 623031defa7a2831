// FP64 throughput probe for sm_100a: DMMA (mma.sync f64 shapes), DFMA, mixed.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int NACC>
__global__ void dmma_m8n8k4(double* out, int iters, double av, double bv) {
  double a = av + threadIdx.x * 1e-9, b = bv;
  double c[NACC][2];
  #pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template<int NACC>
__global__ void dmma_m16n8k16(double* out, int iters, double av, double bv) {
  double a[8], b[4];
  #pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = av + i * 1e-9 + threadIdx.x * 1e-12;
  #pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = bv + i * 1e-9;
  double c[NACC][4];
  #pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template<int NACC>
__global__ void dfma_loop(double* out, int iters, double av, double bv) {
  double c[NACC];
  double a = av + threadIdx.x * 1e-9, b = bv;
  #pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// warps with even id run DMMA, odd id run DFMA
template<int NACC>
__global__ void mixed(double* out, int iters_mma, int iters_fma, double av, double bv) {
  int w = threadIdx.x / 32;
  double s = 0;
  if (w % 2 == 0) {
    double a = av + threadIdx.x * 1e-9, b = bv;
    double c[NACC][2];
    #pragma unroll
    for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters_mma; ++it) {
      #pragma unroll
      for (int i = 0; i < NACC; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  } else {
    double c[NACC];
    double a = av + threadIdx.x * 1e-9, b = bv;
    #pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = i * 1e-3;
    for (int it = 0; it < iters_fma; ++it) {
      #pragma unroll
      for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], a, b);
    }
    for (int i = 0; i < NACC; ++i) s += c[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", p.name, sms, p.clockRate);
  double* out; CK(cudaMalloc(&out, sizeof(double) * 1024 * 1024 * 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int iters = 4000;
  int warps_list[] = {4, 8, 16};
  for (int wi = 0; wi < 3; ++wi) {
    int warps = warps_list[wi];
    int threads = warps * 32;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      dmma_m8n8k4<8><<<sms, threads>>>(out, iters, 1e-3, 1e-3);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * warps * sms;
    printf("{\"kernel\": \"dmma_m8n8k4\", \"warps_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", warps, ms, flops / ms / 1e9);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      dmma_m16n8k16<4><<<sms, threads>>>(out, iters / 4, 1e-3, 1e-3);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    flops = 2.0 * 16 * 8 * 16 * 4.0 * (iters / 4) * warps * sms;
    printf("{\"kernel\": \"dmma_m16n8k16\", \"warps_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", warps, ms, flops / ms / 1e9);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      dfma_loop<8><<<sms, threads>>>(out, iters * 4, 1e-3, 1e-3);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    flops = 2.0 * 8 * iters * 4.0 * threads * sms;
    printf("{\"kernel\": \"dfma\", \"warps_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", warps, ms, flops / ms / 1e9);
  }
  // mixed: 16 warps, 8 DMMA + 8 DFMA, tune iteration ratio so both halves take similar time alone
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    mixed<8><<<sms, 512>>>(out, iters, iters * 8, 1e-3, 1e-3);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  }
  double fl_mma = 2.0 * 256 * 8.0 * iters * 8 * sms;
  double fl_fma = 2.0 * 8 * iters * 8.0 * 8 * 32 * sms;
  printf("{\"kernel\": \"mixed\", \"ms\": %.4f, \"tflops_total\": %.3f, \"mma_part\": %.3e, \"fma_part\": %.3e}\n", ms, (fl_mma + fl_fma) / ms / 1e9, fl_mma, fl_fma);
  // mma-only and fma-only with the same per-warp work for comparison
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    mixed<8><<<sms, 512>>>(out, iters, 0, 1e-3, 1e-3);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("{\"kernel\": \"mixed_mma_only\", \"ms\": %.4f}\n", ms);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    mixed<8><<<sms, 512>>>(out, 0, iters * 8, 1e-3, 1e-3);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("{\"kernel\": \"mixed_fma_only\", \"ms\": %.4f}\n", ms);
  return 0;
}
