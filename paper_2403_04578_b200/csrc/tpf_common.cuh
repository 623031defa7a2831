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

// Same, but volatile: keeps program order among DMMAs (the scheduler would
// otherwise pull dependent DMMAs together to save registers).
__device__ __forceinline__ void dmma884_v(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// 16-byte shared load that the compiler may not merge with an earlier identical load.
__device__ __forceinline__ double2 lds128_v(const double2* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
  return v;
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

// 1/x for an iterate's |v|^2 (in [1e-24, ~1e300]): MUFU seed + two Newton
// steps, faithfully rounded; 4 FP64 instructions and a short dependency chain
// instead of the IEEE divide's ~10 (on the dense path every FP64 instruction
// also costs the SMSP's DMMA stream ~9 cycles).
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = __fma_rn(-x, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-x, r, 1.0);
  return __fma_rn(r, e, r);
}

// NaN-propagating running max, matching numpy's max reduction.
__device__ __forceinline__ double nanmax(double m, double x) {
  return (x > m || x != x) ? x : m;
}

}  // namespace tpf

namespace tpf {
// ---- Tensor Memory as a per-thread register extension (sm_100a) ----------
// A warp may touch only its lane quadrant (warp % 4); with the 32x32b shape
// thread t of the warp reads/writes TMEM lane 32*(warp%4)+t, N consecutive
// 32-bit columns per instruction.
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(a), "r"(ncols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 4 doubles <-> 8 columns
__device__ __forceinline__ void tmem_st4d(uint32_t taddr, double a, double b, double c, double d) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
      "r"(__double2loint(a)), "r"(__double2hiint(a)), "r"(__double2loint(b)), "r"(__double2hiint(b)),
      "r"(__double2loint(c)), "r"(__double2hiint(c)), "r"(__double2loint(d)), "r"(__double2hiint(d))
      : "memory");
}
struct D4 {
  uint32_t r[8];
  __device__ __forceinline__ double get(int i) const { return __hiloint2double(int(r[2 * i + 1]), int(r[2 * i])); }
};
__device__ __forceinline__ void tmem_ld4d(uint32_t taddr, D4& o) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(o.r[0]), "=r"(o.r[1]), "=r"(o.r[2]), "=r"(o.r[3]), "=r"(o.r[4]), "=r"(o.r[5]), "=r"(o.r[6]),
                 "=r"(o.r[7])
               : "r"(taddr)
               : "memory");
}
}  // namespace tpf

namespace tpf {
// 1 double2 (re, im) <-> 4 TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_st2(uint32_t taddr, double2 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
               "r"(__double2loint(v.x)), "r"(__double2hiint(v.x)), "r"(__double2loint(v.y)), "r"(__double2hiint(v.y))
               : "memory");
}
struct D2 {
  uint32_t r[4];
  __device__ __forceinline__ double2 get() const {
    return make_double2(__hiloint2double(int(r[1]), int(r[0])), __hiloint2double(int(r[3]), int(r[2])));
  }
};
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, D2& o) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(o.r[0]), "=r"(o.r[1]), "=r"(o.r[2]), "=r"(o.r[3])
               : "r"(taddr)
               : "memory");
}
}  // namespace tpf

namespace tpf {
// ---- mbarrier (CTA scope) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
}  // namespace tpf
