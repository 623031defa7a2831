// complex64 twins of the hot path ("a c64 twin of each").
//
// Same update, semantics and layouts as the complex128 entry points
// (dense.py:114-126 / sparse.py:186-197, per-case freeze, flat start, zero
// guard, step test |v' - v|^2 < tol^2), evaluated in FP32.  B200 has no FP32
// tensor-core path with FP32 accuracy (TF32 keeps 10 mantissa bits), so both
// kernels are SIMT:
//
//   * dense (b <= 104): one thread per case slot, 128 slots per CTA, K^T in
//     shared memory (broadcast reads, two complex entries per LDS.128), the
//     slot's U column in shared memory (no sharing between threads, so no
//     barriers after the prologue), V' accumulated in registers 26 nodes at a
//     time, continuous batching from a global counter;
//   * sparse: the CSR forward/backward sweeps of tpf_sparse_fpi_c128, one
//     thread per case, in FP32.
//
// FP32 cannot resolve the reference's default tol = 1e-10 (|v| ~ 1, eps =
// 6e-8): callers pass a tolerance >= ~1e-6 and a residual tolerance >= ~1e-4.
// The residual post-check of a c64 solution is evaluated in FP64
// (tpf_residual_c64).
#include <climits>
#include <cstdlib>

#include "tpf_common.cuh"
#include "tpf_internal.h"

namespace tpf {
namespace {

constexpr float kGuard32 = 1e-12f;
constexpr float kGuard32Sq = 1e-24f;
constexpr int kC64Threads = 128;
constexpr int kC64MaxNodes = 104;
constexpr int kC64Chunk = 26;  // V' nodes per register chunk (4 chunks at b = 104)

struct DenseC64Args {
  int64_t tau;
  int b;
  const float2* S;
  int64_t s_node, s_case;
  const float2* K;  // b x b row-major
  const float2* W;
  float2 v_flat;
  float tol2;
  int max_iter;
  float2* V;
  int64_t v_node, v_case;
  int32_t* iters;
  unsigned long long* counter;
  float2* scratch;  // 2 x b x (grid * 128) complex64: slot-major iterate and loads
};

__device__ __forceinline__ float2 guard32(float2 v) {
  return (fmaf(v.x, v.x, v.y * v.y) < kGuard32Sq) ? make_float2(kGuard32, 0.f) : v;
}

// s* / conj(v) = conj(s) v / |v|^2 on the guarded v
__device__ __forceinline__ float2 recip32(float2 s, float2 v) {
  const float r = 1.0f / fmaf(v.x, v.x, v.y * v.y);
  return make_float2(fmaf(s.x, v.x, s.y * v.y) * r, fmaf(s.x, v.y, -(s.y * v.x)) * r);
}

#ifdef TPF_AB_VARIANTS  // A/B-only kernel, not in libtpf.so
// BP: node count padded to a multiple of the 26-node register chunk, so every
// loop over V' nodes is compile-time (padding rows of K^T and W are zero).
// 256 threads = 128 case slots, two threads per slot (lanes l and l + 16 of
// a warp), each owning half of the slot's 26-node chunks (its U entries, V'
// nodes, loads and iterate), so 8 warps per SM hide the shared-memory latency
// of the FFMA loop; only U is exchanged (shared memory, __syncwarp).
template <int BP>
__global__ void __launch_bounds__(2 * kC64Threads, 1) dense_c64_halves_kernel(const DenseC64Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = a.b;
  constexpr int bp = BP;
  constexpr int kChunks = BP / kC64Chunk;
  float2* kt = reinterpret_cast<float2*>(smem_raw);              // [b][bp]: kt[k][n] = K[n][k]
  float2* w = kt + size_t(b) * bp;                               // [bp]
  float2* us = w + bp;                                           // [b][128]: U of each slot
  const int t = threadIdx.x, lane = t & 31, h = lane >> 4;
  const int slot = (t >> 5) * 16 + (lane & 15);
  for (int idx = t; idx < b * bp; idx += 2 * kC64Threads) {
    const int k = idx / bp, n = idx % bp;
    kt[idx] = n < b ? a.K[size_t(n) * b + k] : make_float2(0.f, 0.f);
  }
  for (int n = t; n < bp; n += 2 * kC64Threads) w[n] = n < b ? a.W[n] : make_float2(0.f, 0.f);
  __syncthreads();

  // The slot's case lives in a slot-major scratch (node n of slot g at
  // [n * slots + g]), so every per-iteration access is coalesced whatever
  // cases the slots hold; S is copied in on refill and V' out on retire.
  const int64_t slots = int64_t(gridDim.x) * kC64Threads;
  const int64_t g = int64_t(blockIdx.x) * kC64Threads + slot;
  float2* vs = a.scratch + g;                 // iterate
  float2* ss = a.scratch + slots * b + g;     // loads
  constexpr int kHalf0 = (kChunks + 1) / 2;                    // chunks of half 0
  const int c0 = h ? kHalf0 : 0, c1 = h ? kChunks : kHalf0;     // this thread's chunks
  const int k0 = min(b, c0 * kC64Chunk), k1 = min(b, c1 * kC64Chunk);  // and nodes
  int n_it = 0;
  auto claim = [&](bool want) {  // every lane of the warp calls it
    int c = INT_MAX;
    if (h == 0 && want) {
      const unsigned long long x = atomicAdd(a.counter, 1ull);
      c = x < (unsigned long long)a.tau ? int(x) : INT_MAX;
    }
    return __shfl_sync(0xffffffffu, c, lane & 15);
  };
  auto load_case = [&](int cid) {
    if (cid == INT_MAX) return;
    const int64_t sb = int64_t(cid) * a.s_case;
#pragma unroll 4
    for (int k = k0; k < k1; ++k) {
      ss[k * slots] = a.S[k * a.s_node + sb];
      vs[k * slots] = a.v_flat;
    }
  };
  int cid = claim(true);
  load_case(cid);
  while (__any_sync(0xffffffffu, cid != INT_MAX)) {
    // ---- U = S* / conj(guarded v): this thread's node half of the slot ----
    __syncwarp();  // the other half has finished reading the previous U
#pragma unroll 4
    for (int k = k0; k < k1; ++k) us[k * kC64Threads + slot] = recip32(ss[k * slots], guard32(vs[k * slots]));
    __syncwarp();
    // ---- V' = W + K U on this thread's chunks, step test against the old iterate ----
    bool small = true;
#pragma unroll 1
    for (int ci = c0; ci < c1; ++ci) {
      const int n0 = ci * kC64Chunk;
      float ar[kC64Chunk], ai[kC64Chunk];
#pragma unroll
      for (int c = 0; c < kC64Chunk; ++c) {
        const float2 wc = w[n0 + c];
        ar[c] = wc.x;
        ai[c] = wc.y;
      }
#pragma unroll 4
      for (int k = 0; k < b; ++k) {
        const float2 u = us[k * kC64Threads + slot];
        const float4* kr = reinterpret_cast<const float4*>(kt + size_t(k) * bp + n0);
#pragma unroll
        for (int c = 0; c < kC64Chunk; c += 2) {
          const float4 kk = kr[c / 2];  // K[n0+c][k], K[n0+c+1][k]
          ar[c] = fmaf(kk.x, u.x, fmaf(-kk.y, u.y, ar[c]));
          ai[c] = fmaf(kk.x, u.y, fmaf(kk.y, u.x, ai[c]));
          ar[c + 1] = fmaf(kk.z, u.x, fmaf(-kk.w, u.y, ar[c + 1]));
          ai[c + 1] = fmaf(kk.z, u.y, fmaf(kk.w, u.x, ai[c + 1]));
        }
      }
#pragma unroll
      for (int c = 0; c < kC64Chunk; ++c) {
        const int n = n0 + c;
        if (n < b) {
          const float2 v = guard32(vs[n * slots]);
          const float dr = ar[c] - v.x, di = ai[c] - v.y;
          if (!(fmaf(dr, dr, di * di) < a.tol2)) small = false;  // NaN never passes
          vs[n * slots] = make_float2(ar[c], ai[c]);
        }
      }
    }
    const bool other_small = __shfl_xor_sync(0xffffffffu, small, 16);  // every lane (no short-circuit)
    small = small && other_small;
    ++n_it;
    const bool done = cid != INT_MAX && (small || n_it >= a.max_iter);
    if (done) {  // retire: V' out (this thread's node half), per-case count
      const int64_t vb = int64_t(cid) * a.v_case;
#pragma unroll 4
      for (int n = k0; n < k1; ++n) a.V[n * a.v_node + vb] = vs[n * slots];
      if (h == 0) a.iters[cid] = n_it;
    }
    if (__any_sync(0xffffffffu, done)) {  // refill the retiring slots
      const int c = claim(done);
      if (done) {
        cid = c;
        n_it = 0;
        load_case(cid);
      }
    }
  }
}
#endif  // TPF_AB_VARIANTS

// Default dense c64 kernel: 256 threads = 2 groups of 4 warps; a group owns
// 64 slot pairs (slots p and p + 64, p = lane of the group's warps) and warp q
// of the group owns node quarter q (NC nodes).  Every K^T read of a warp is
// then one broadcast address (one wavefront for two complex entries) and is
// reused by two slots, so each LDS.128 of K feeds 16 FFMAs instead of 8, and
// the U reads are contiguous.  The four quarters of a slot meet at a named
// barrier of their group (bar 1 + group, 128 threads) after U is formed and
// after the step test; the refill ids go through shared memory.  Same
// arithmetic per case as dense_c64_halves_kernel (bitwise the same V').
template <int NC>
__global__ void __launch_bounds__(2 * kC64Threads, 1) dense_c64_kernel(const DenseC64Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_cid[kC64Threads];
  __shared__ unsigned char s_small[4][kC64Threads];
  const int b = a.b;
  constexpr int bp = 4 * NC;
  float2* kt = reinterpret_cast<float2*>(smem_raw);  // [b][bp]: kt[k][n] = K[n][k]
  float2* w = kt + size_t(b) * bp;                   // [bp]
  float2* us = w + bp;                               // [b][128]: U of each slot
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int q = warp & 3, grp = warp >> 2;
  const int sA = grp * 32 + lane, sB = sA + 64;
  for (int idx = t; idx < b * bp; idx += 2 * kC64Threads) {
    const int k = idx / bp, n = idx % bp;
    kt[idx] = n < b ? a.K[size_t(n) * b + k] : make_float2(0.f, 0.f);
  }
  for (int n = t; n < bp; n += 2 * kC64Threads) w[n] = n < b ? a.W[n] : make_float2(0.f, 0.f);
  __syncthreads();

  const int64_t slots = int64_t(gridDim.x) * kC64Threads;
  const int64_t gA = int64_t(blockIdx.x) * kC64Threads + sA;
  float2* vsA = a.scratch + gA;               // iterate, slot-major
  float2* vsB = vsA + 64;
  const int n0 = q * NC;
  const int k0 = min(b, n0), k1 = min(b, n0 + NC);
  auto gbar = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(4 * 32) : "memory"); };
  // quarter 0 claims the next case ids of the group's retiring slots; the
  // other quarters read them after the group barrier
  auto claim = [&](bool wantA, bool wantB, int& cA, int& cB) {
    if (q == 0) {
      if (wantA) {
        const unsigned long long x = atomicAdd(a.counter, 1ull);
        s_cid[sA] = x < (unsigned long long)a.tau ? int(x) : INT_MAX;
      }
      if (wantB) {
        const unsigned long long x = atomicAdd(a.counter, 1ull);
        s_cid[sB] = x < (unsigned long long)a.tau ? int(x) : INT_MAX;
      }
    }
    gbar();
    if (wantA) cA = s_cid[sA];
    if (wantB) cB = s_cid[sB];
  };
  // refill = flat start only: S is read in place by form_u (L2-resident
  // while the case is active) and V' is written by the step test of the
  // iteration that may retire the slot, so neither end copies through the
  // scratch (such a copy waits one memory round trip per node)
  auto load_case = [&](int cid, float2* vs) {
    if (cid == INT_MAX) return;
#pragma unroll 4
    for (int k = k0; k < k1; ++k) vs[k * slots] = a.v_flat;
  };
  // U is formed with every load of a half-quarter issued before the first
  // dependent store (one memory round trip per half, not one per node)
  constexpr int kH = (NC + 1) / 2;  // U formed in two halves of the quarter (register budget)
  auto form_u = [&](int cid, const float2* vs, int slot) {
    const bool live = cid != INT_MAX;
    const int64_t sb = int64_t(live ? cid : 0) * a.s_case;
#pragma unroll
    for (int c0 = 0; c0 < NC; c0 += kH) {
      float2 sv[kH], vv[kH];
#pragma unroll
      for (int c = 0; c < kH; ++c)
        if (c0 + c < NC && n0 + c0 + c < b) {
          sv[c] = live ? __ldg(a.S + (n0 + c0 + c) * a.s_node + sb) : make_float2(0.f, 0.f);
          vv[c] = vs[(n0 + c0 + c) * slots];
        }
#pragma unroll
      for (int c = 0; c < kH; ++c)
        if (c0 + c < NC && n0 + c0 + c < b) us[(n0 + c0 + c) * kC64Threads + slot] = recip32(sv[c], guard32(vv[c]));
    }
  };
  int cA = INT_MAX, cB = INT_MAX;
  claim(true, true, cA, cB);
  load_case(cA, vsA);
  load_case(cB, vsB);
  int itA = 0, itB = 0;
  while (__any_sync(0xffffffffu, cA != INT_MAX || cB != INT_MAX)) {  // uniform over the group
    // ---- U = S* / conj(guarded v) on this quarter's nodes of both slots ----
    form_u(cA, vsA, sA);
    form_u(cB, vsB, sB);
    gbar();
    // ---- V' = W + K U on this quarter's nodes, two slots per K read ----
    float arA[NC], aiA[NC], arB[NC], aiB[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const float2 wc = w[n0 + c];
      arA[c] = wc.x;
      aiA[c] = wc.y;
      arB[c] = wc.x;
      aiB[c] = wc.y;
    }
#pragma unroll 2
    for (int k = 0; k < b; ++k) {
      const float2 uA = us[k * kC64Threads + sA];
      const float2 uB = us[k * kC64Threads + sB];
      const float4* kr = reinterpret_cast<const float4*>(kt + size_t(k) * bp + n0);
#pragma unroll
      for (int c = 0; c < NC; c += 2) {
        const float4 kk = kr[c / 2];  // K[n0+c][k], K[n0+c+1][k] (one broadcast address per warp)
        arA[c] = fmaf(kk.x, uA.x, fmaf(-kk.y, uA.y, arA[c]));
        aiA[c] = fmaf(kk.x, uA.y, fmaf(kk.y, uA.x, aiA[c]));
        arA[c + 1] = fmaf(kk.z, uA.x, fmaf(-kk.w, uA.y, arA[c + 1]));
        aiA[c + 1] = fmaf(kk.z, uA.y, fmaf(kk.w, uA.x, aiA[c + 1]));
        arB[c] = fmaf(kk.x, uB.x, fmaf(-kk.y, uB.y, arB[c]));
        aiB[c] = fmaf(kk.x, uB.y, fmaf(kk.y, uB.x, aiB[c]));
        arB[c + 1] = fmaf(kk.z, uB.x, fmaf(-kk.w, uB.y, arB[c + 1]));
        aiB[c + 1] = fmaf(kk.z, uB.y, fmaf(kk.w, uB.x, aiB[c + 1]));
      }
    }
    // ---- step test against the old iterate, new iterate out ----
    bool smA = true, smB = true;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int n = n0 + c;
      if (n < b) {
        const float2 va = guard32(vsA[n * slots]);
        const float dra = arA[c] - va.x, dia = aiA[c] - va.y;
        if (!(fmaf(dra, dra, dia * dia) < a.tol2)) smA = false;  // NaN never passes
        vsA[n * slots] = make_float2(arA[c], aiA[c]);
        const float2 vb = guard32(vsB[n * slots]);
        const float drb = arB[c] - vb.x, dib = aiB[c] - vb.y;
        if (!(fmaf(drb, drb, dib * dib) < a.tol2)) smB = false;
        vsB[n * slots] = make_float2(arB[c], aiB[c]);
      }
    }
    // V' out when this iteration can retire the slot (this quarter passed the
    // test, or the cap is reached); a quarter whose slot goes on rewrites it later
    if (cA != INT_MAX && (smA || itA + 1 >= a.max_iter)) {
      const int64_t vb = int64_t(cA) * a.v_case;
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (n0 + c < b) a.V[(n0 + c) * a.v_node + vb] = make_float2(arA[c], aiA[c]);
    }
    if (cB != INT_MAX && (smB || itB + 1 >= a.max_iter)) {
      const int64_t vb = int64_t(cB) * a.v_case;
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (n0 + c < b) a.V[(n0 + c) * a.v_node + vb] = make_float2(arB[c], aiB[c]);
    }
    s_small[q][sA] = smA;
    s_small[q][sB] = smB;
    gbar();  // also: every quarter has finished reading U
    smA = s_small[0][sA] & s_small[1][sA] & s_small[2][sA] & s_small[3][sA];
    smB = s_small[0][sB] & s_small[1][sB] & s_small[2][sB] & s_small[3][sB];
    ++itA;
    ++itB;
    const bool doneA = cA != INT_MAX && (smA || itA >= a.max_iter);
    const bool doneB = cB != INT_MAX && (smB || itB >= a.max_iter);
    if (q == 0) {  // retire: V' is already out
      if (doneA) a.iters[cA] = itA;
      if (doneB) a.iters[cB] = itB;
    }
    if (__any_sync(0xffffffffu, doneA || doneB)) {  // same answer in the group's 4 warps
      int nA = cA, nB = cB;
      claim(doneA, doneB, nA, nB);
      if (doneA) {
        cA = nA;
        itA = 0;
        load_case(cA, vsA);
      }
      if (doneB) {
        cB = nB;
        itB = 0;
        load_case(cB, vsB);
      }
    }
  }
}

struct SparseC64Args {
  int64_t tau;
  int b;
  const float2* S;
  int64_t s_node, s_case;
  const int32_t *l_ptr, *l_col;
  const float2* l_val;
  const int32_t *u_ptr, *u_col;
  const float2* u_val;
  const float2* u_diag_inv;
  const int32_t* row_src;
  const int32_t* col_dst;
  const float2* src;
  float2 v_flat;
  float tol2;
  int max_iter;
  float2* V;
  int64_t v_node, v_case;
  int32_t* iters;
  float2* T;
  int64_t t_ld;
};

__global__ void __launch_bounds__(128) sparse_c64_kernel(const SparseC64Args a) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= a.tau) return;
  const int b = a.b;
  for (int i = 0; i < b; ++i) a.V[i * a.v_node + j * a.v_case] = a.v_flat;
  int n = 0;
  while (n < a.max_iter) {
    for (int k = 0; k < b; ++k) {  // forward sweep
      const int i = __ldg(a.row_src + k);
      const float2 u = recip32(a.S[i * a.s_node + j * a.s_case], guard32(a.V[i * a.v_node + j * a.v_case]));
      const float2 c = a.src[i];
      float zr = -(u.x + c.x), zi = -(u.y + c.y);
      for (int p = __ldg(a.l_ptr + k); p < __ldg(a.l_ptr + k + 1); ++p) {
        const float2 l = a.l_val[p];
        const float2 z = a.T[__ldg(a.l_col + p) * a.t_ld + j];
        zr = fmaf(-l.x, z.x, fmaf(l.y, z.y, zr));
        zi = fmaf(-l.x, z.y, fmaf(-l.y, z.x, zi));
      }
      a.T[k * a.t_ld + j] = make_float2(zr, zi);
    }
    for (int k = b - 1; k >= 0; --k) {  // backward sweep
      float2 z = a.T[k * a.t_ld + j];
      for (int p = __ldg(a.u_ptr + k); p < __ldg(a.u_ptr + k + 1); ++p) {
        const float2 u = a.u_val[p];
        const float2 w = a.T[__ldg(a.u_col + p) * a.t_ld + j];
        z.x = fmaf(-u.x, w.x, fmaf(u.y, w.y, z.x));
        z.y = fmaf(-u.x, w.y, fmaf(-u.y, w.x, z.y));
      }
      const float2 d = a.u_diag_inv[k];
      a.T[k * a.t_ld + j] = make_float2(fmaf(z.x, d.x, -(z.y * d.y)), fmaf(z.x, d.y, z.y * d.x));
    }
    bool small = true;
    for (int i = 0; i < b; ++i) {  // scatter to node order, step test
      const float2 x = a.T[__ldg(a.col_dst + i) * a.t_ld + j];
      const float2 v = guard32(a.V[i * a.v_node + j * a.v_case]);
      const float dr = x.x - v.x, di = x.y - v.y;
      if (!(fmaf(dr, dr, di * di) < a.tol2)) small = false;
      a.V[i * a.v_node + j * a.v_case] = x;
    }
    ++n;
    if (small) break;
  }
  a.iters[j] = n;
}

// residual_per_case (fpi.py:221-240) of a complex64 solution, evaluated in FP64.
__global__ void residual_c64_kernel(int64_t tau, int b, const float2* __restrict__ S, int64_t sn, int64_t sc,
                                    const float2* __restrict__ V, int64_t vn, int64_t vc,
                                    const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                    const double2* __restrict__ yv, const double2* __restrict__ src,
                                    double* __restrict__ resid) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= tau) return;
  double worst = 0.0;
  for (int i = 0; i < b; ++i) {
    const double2 si = __ldg(src + i);
    double ar = si.x, ai = si.y;
    for (int k = __ldg(rp + i); k < __ldg(rp + i + 1); ++k) {
      const double2 y = __ldg(yv + k);
      const float2 vf = V[int64_t(__ldg(ci + k)) * vn + j * vc];
      const double vx = vf.x, vy = vf.y;
      ar = __fma_rn(y.x, vx, __fma_rn(-y.y, vy, ar));
      ai = __fma_rn(y.x, vy, __fma_rn(y.y, vx, ai));
    }
    const float2 vf = V[int64_t(i) * vn + j * vc];
    const float2 sf = S[int64_t(i) * sn + j * sc];
    const double vx = vf.x, vy = vf.y;
    const double mr = double(sf.x) + (vx * ar + vy * ai);
    const double mi = double(sf.y) + (vy * ar - vx * ai);
    worst = nanmax(worst, hypot(mr, mi));
  }
  resid[j] = worst;
}

}  // namespace
}  // namespace tpf

using namespace tpf;

extern "C" int tpf_dense_c64_max_nodes(void) { return kC64MaxNodes; }

static int64_t c64_grid(int64_t tau) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = sms;
  const int64_t need = (tau + kC64Threads - 1) / kC64Threads;
  if (need < grid) grid = need;
  return grid < 1 ? 1 : grid;
}

extern "C" size_t tpf_dense_c64_workspace_bytes(int64_t tau, int32_t b) {
  return 256 + size_t(2) * size_t(b) * size_t(c64_grid(tau)) * kC64Threads * sizeof(float2);
}

extern "C" int tpf_dense_fpi_c64(int64_t tau, int32_t b, const float* S, int64_t s_node_stride, int64_t s_case_stride,
                                 const float* K, const float* W, float v_flat_re, float v_flat_im, float tol,
                                 int32_t max_iter, float* V, int64_t v_node_stride, int64_t v_case_stride,
                                 int32_t* iters, void* workspace, size_t workspace_bytes, void* stream) {
  if (tau < 0 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_dense_fpi_c64: need tau >= 0 and b >= 1");
  if (b > kC64MaxNodes) return set_error(TPF_ERR_UNSUPPORTED, "tpf_dense_fpi_c64: b > 104");
  if (tau > INT_MAX - 4096) return set_error(TPF_ERR_INVALID, "tau too large for one launch; shard it");
  if (!(tol > 0.0f)) return set_error(TPF_ERR_INVALID, "tolerance must be positive");
  if (max_iter < 1) return set_error(TPF_ERR_INVALID, "max_iterations must be >= 1");
  if (tau == 0) return TPF_OK;
  if (!S || !K || !W || !V || !iters || !workspace || workspace_bytes < tpf_dense_c64_workspace_bytes(tau, b))
    return set_error(TPF_ERR_INVALID, "tpf_dense_fpi_c64: null pointer or small workspace");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t grid = c64_grid(tau);
  cudaError_t err = cudaMemsetAsync(workspace, 0, sizeof(unsigned long long), st);
  if (err != cudaSuccess) return set_cuda_error("cudaMemsetAsync(counter)", err);
  // default: quarter kernel (two slots per thread); in A/B builds
  // (-DTPF_AB_VARIANTS) TPF_C64_HALVES=1 runs the previous one-slot-per-thread kernel
  int bp;
  void (*kern)(const DenseC64Args);
#ifdef TPF_AB_VARIANTS
  static const bool halves = [] {
    const char* e = getenv("TPF_C64_HALVES");
    return e && e[0] == '1';
  }();
  if (halves) {
    bp = (b + kC64Chunk - 1) / kC64Chunk * kC64Chunk;
    kern = bp == 26 ? dense_c64_halves_kernel<26> : bp == 52 ? dense_c64_halves_kernel<52>
         : bp == 78 ? dense_c64_halves_kernel<78> : dense_c64_halves_kernel<104>;
  } else
#endif
  {  // nodes per quarter
    const int nc = b <= 32 ? 8 : b <= 40 ? 10 : b <= 56 ? 14 : b <= 80 ? 20 : 26;
    bp = 4 * nc;
    kern = nc == 8 ? dense_c64_kernel<8> : nc == 10 ? dense_c64_kernel<10> : nc == 14 ? dense_c64_kernel<14>
         : nc == 20 ? dense_c64_kernel<20> : dense_c64_kernel<26>;
  }
  const size_t smem = (size_t(b) * bp + bp + size_t(b) * kC64Threads) * sizeof(float2);
  err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (err != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(dense_c64)", err);
  DenseC64Args a;
  a.tau = tau;
  a.b = b;
  a.S = reinterpret_cast<const float2*>(S);
  a.s_node = s_node_stride;
  a.s_case = s_case_stride;
  a.K = reinterpret_cast<const float2*>(K);
  a.W = reinterpret_cast<const float2*>(W);
  a.v_flat = make_float2(v_flat_re, v_flat_im);
  a.tol2 = tol * tol;
  a.max_iter = max_iter;
  a.V = reinterpret_cast<float2*>(V);
  a.v_node = v_node_stride;
  a.v_case = v_case_stride;
  a.iters = iters;
  a.counter = static_cast<unsigned long long*>(workspace);
  a.scratch = reinterpret_cast<float2*>(static_cast<char*>(workspace) + 256);
  kern<<<unsigned(grid), 2 * kC64Threads, smem, st>>>(a);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(dense_c64_kernel)", err);
  return TPF_OK;
}

extern "C" size_t tpf_sparse_c64_workspace_bytes(int64_t tau, int32_t b) { return size_t(tau) * size_t(b) * 8 + 256; }

extern "C" int tpf_sparse_fpi_c64(int64_t tau, int32_t b, const float* S, int64_t s_node_stride,
                                  int64_t s_case_stride, const int32_t* l_ptr, const int32_t* l_col,
                                  const float* l_val, const int32_t* u_ptr, const int32_t* u_col, const float* u_val,
                                  const float* u_diag_inv, const int32_t* perm, const float* src, float v_flat_re,
                                  float v_flat_im, float tol, int32_t max_iter, float* V, int64_t v_node_stride,
                                  int64_t v_case_stride, int32_t* iters, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  if (tau < 0 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_sparse_fpi_c64: need tau >= 0, b >= 1");
  if (!(tol > 0.0f)) return set_error(TPF_ERR_INVALID, "tolerance must be positive");
  if (max_iter < 1) return set_error(TPF_ERR_INVALID, "max_iterations must be >= 1");
  if (tau == 0) return TPF_OK;
  if (!S || !l_ptr || !u_ptr || !u_diag_inv || !perm || !src || !V || !iters || !workspace)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_fpi_c64: null pointer");
  if (workspace_bytes < tpf_sparse_c64_workspace_bytes(tau, b))
    return set_error(TPF_ERR_INVALID, "tpf_sparse_fpi_c64: workspace too small");
  SparseC64Args a;
  a.tau = tau;
  a.b = b;
  a.S = reinterpret_cast<const float2*>(S);
  a.s_node = s_node_stride;
  a.s_case = s_case_stride;
  a.l_ptr = l_ptr;
  a.l_col = l_col;
  a.l_val = reinterpret_cast<const float2*>(l_val);
  a.u_ptr = u_ptr;
  a.u_col = u_col;
  a.u_val = reinterpret_cast<const float2*>(u_val);
  a.u_diag_inv = reinterpret_cast<const float2*>(u_diag_inv);
  a.row_src = perm;
  a.col_dst = perm + b;
  a.src = reinterpret_cast<const float2*>(src);
  a.v_flat = make_float2(v_flat_re, v_flat_im);
  a.tol2 = tol * tol;
  a.max_iter = max_iter;
  a.V = reinterpret_cast<float2*>(V);
  a.v_node = v_node_stride;
  a.v_case = v_case_stride;
  a.iters = iters;
  a.T = static_cast<float2*>(workspace);
  a.t_ld = tau;
  const int threads = 128;
  const int64_t blocks = (tau + threads - 1) / threads;
  sparse_c64_kernel<<<unsigned(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(a);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(sparse_c64_kernel)", err);
  return TPF_OK;
}

extern "C" int tpf_residual_c64(int64_t tau, int32_t b, const float* S, int64_t s_node_stride, int64_t s_case_stride,
                                const float* V, int64_t v_node_stride, int64_t v_case_stride,
                                const int32_t* ydd_row_ptr, const int32_t* ydd_col, const double* ydd_val,
                                const double* src, double* resid, void* stream) {
  if (tau < 0 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_residual_c64: need tau >= 0, b >= 1");
  if (tau == 0) return TPF_OK;
  if (!S || !V || !ydd_row_ptr || !ydd_col || !ydd_val || !src || !resid)
    return set_error(TPF_ERR_INVALID, "tpf_residual_c64: null pointer");
  const int threads = 256;
  const int64_t blocks = (tau + threads - 1) / threads;
  residual_c64_kernel<<<unsigned(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(
      tau, b, reinterpret_cast<const float2*>(S), s_node_stride, s_case_stride, reinterpret_cast<const float2*>(V),
      v_node_stride, v_case_stride, ydd_row_ptr, ydd_col, reinterpret_cast<const double2*>(ydd_val),
      reinterpret_cast<const double2*>(src), resid);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(residual_c64_kernel)", err);
  return TPF_OK;
}
