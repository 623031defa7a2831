// Shared device helpers for the TPF engine (sm_100a only).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef __CUDACC__
#error "tpf_common.cuh is CUDA-only"
#endif

namespace tpf {

// fpi.py:39-41: |v| < 1e-12 -> v := 1e-12 + 0j.  Compared on |v|^2.
constexpr double kZeroGuard = 1e-12;
constexpr double kZeroGuard2 = 1e-24;

// D = A(8x4, row) * B(4x8, col) + D, FP64 tensor core (SASS DMMA.8x8x4).
// Non-volatile: the instruction has no side effect beyond its outputs, so the
// scheduler may interleave shared-memory loads around it.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// Sign flip on the integer pipe (keeps the FP64 pipe free for DMMA).
__device__ __forceinline__ double neg_int(double x) {
  return __hiloint2double(__double2hiint(x) ^ 0x80000000, __double2loint(x));
}

// Named barrier over `count` threads (id 0 is __syncthreads).
__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ double2 ldg_c128(const double* base, int64_t idx) {
  return __ldg(reinterpret_cast<const double2*>(base) + idx);
}

__device__ __forceinline__ void stg_c128(double* base, int64_t idx, double2 v) {
  reinterpret_cast<double2*>(base)[idx] = v;
}

// NaN-propagating running max, matching numpy's max reduction.
__device__ __forceinline__ double nanmax(double m, double x) {
  return (x > m || x != x) ? x : m;
}

}  // namespace tpf
