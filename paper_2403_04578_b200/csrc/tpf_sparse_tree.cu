// Sparse Tensor Power Flow for radial feeders: one case per CTA, all of the
// case's state on chip, level-synchronous tree sweeps.
//
// For a tree-structured Y_dd in leaf-first order the LU has no fill
// (SURVEY.md A.6): row k of L holds only k's children, row k of U only its
// parent.  Grouping nodes by depth, one fixed-point iteration
//     Y_dd v' = -(s* ./ conj(v) + src)          (sparse.py:3-14, 186-197)
// is an up-sweep (deepest level first)
//     z_k = r_k - sum_{c child of k} L_kc z_c,   r_k = -(s_k*/conj(v_k) + src_k)
// and a down-sweep (root level first)
//     w_k = (z_k - U_kp w_p) / U_kk,             v'_k = w_k.
// Both sweeps use the SAME depth levels, so one thread owns node k in both
// and keeps the node's iterate v_k and load s_k in its own Tensor Memory lane
// (4 columns each per "slot"; a slot is one node of one level for every thread
// of the CTA, so TMEM addresses stay warp-uniform).  The sweep vector z/w of
// the whole case lives in shared memory (16 B per node).  Global memory is
// touched once per case: S in, V out (the compulsory traffic).
//
// CTA = 512 threads (16 warps, 4 per TMEM lane quadrant, 128 columns each =
// 16 slots), one CTA per SM (all 512 TMEM columns), persistent over cases.
#include <climits>
#include <cstdlib>
#include <vector>

#include "tpf_common.cuh"
#include "tpf_internal.h"

namespace tpf {
namespace {

constexpr int kTreeThreads = 512;

#ifdef TPF_PHASE_TIMING
// debug build only (tools/build_timing.sh): thread 0 of every CTA accumulates
// cycles per phase: {case load, up-sweep, down-sweep, retire, residual, cases, iterations, total}
__device__ long long g_tree_cyc[148 * 8];
#define TREE_T(v) const long long v = clock64()
#define TREE_ACC(i, t0) \
  if (threadIdx.x == 0) tc[i] += clock64() - (t0)
#else
#define TREE_T(v)
#define TREE_ACC(i, t0)
#endif
constexpr int kMaxSlots = 16;
constexpr int kMaxLevels = 64;

struct TreeArgs {
  int64_t tau;
  int b, levels;
  const double2* S;
  int64_t s_node, s_case;
  double2* V;
  int64_t v_node, v_case;
  int32_t* iters;
  unsigned long long* counter;
  const int32_t* lvl;     // [levels+1] level offsets in level order (root level first), then [levels+1] slot starts
  const int4* info;       // per level-ordered node m: {original node, parent m or -1, first child m, child count}
  const double2* coef;    // planes [4][b] (level order m): e = Y[parent, m], g = U[m,parent]/U[m,m], uinv = 1/U[m,m], src
  double2 v_flat;
  const double2* v0;      // ZIP: initial iterate (original node order) or null: flat start
  double tol2;
  int max_iter;
  // optional fused residual post-check (same arithmetic as residual_kernel):
  // Y_dd rows in level order as ELL, entry r of row m at [r * b + m] (coalesced
  // over m), entries in the original CSR order, padding col = -1
  int ell_w;
  const int32_t* ell_col;
  const double2* ell_val;
  double* resid;          // or null
  // ZIP loads (fpi.py:107-206 per case): planes [3][b] alpha_z, alpha_i,
  // alpha_p and Y[m,m] in level order; per-CTA scratch [2][b] for the case's
  // own g and 1/U[m,m]; status = 1 on a zero or non-finite pivot
  const double* alpha;
  const double2* ydiag;
  double2* zcoef;
  int32_t* status;
  uint8_t* met;           // ZIP: 1 if the case stopped on the step test (or is a one-application case)
  int prefetch;           // prefetch the next case's loads into L2 (TPF_TREE_PREFETCH=1; default off)
};

__device__ __forceinline__ double2 cfma_sub(double2 acc, double2 a, double2 x) {  // acc - a*x
  return make_double2(__fma_rn(-a.x, x.x, __fma_rn(a.y, x.y, acc.x)), __fma_rn(-a.x, x.y, __fma_rn(-a.y, x.x, acc.y)));
}
__device__ __forceinline__ double2 cmul2(double2 a, double2 x) {
  return make_double2(__fma_rn(a.x, x.x, -(a.y * x.y)), __fma_rn(a.x, x.y, a.y * x.x));
}

constexpr int kLS = 6;  // max TMEM slots of one level (the host schedule guarantees it)
constexpr int kMaxRoots = 512;
constexpr int kMaxEllWidth = 16;  // widest Y_dd row the fused residual takes
constexpr int kEllChunk = 8;      // ELL entries loaded together

// Sweeps with g_m = U[m,parent] / U[m,m] (so L[p,m] z_m = g_m z_m for symmetric Y):
//   up:   z_m = r_m - sum_c g_c z_c
//   down: w_m = z_m / U[m,m] - g_m w_parent
template <bool ZIP>
__global__ void __launch_bounds__(kTreeThreads, 1) sparse_tree_kernel(const TreeArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* T = reinterpret_cast<double2*>(smem_raw);       // [b] sweep vector (zhat, then w)
  double2* P = T + a.b;                                    // [b] e_m * zhat_m, pulled by the parent
  int2* kids = reinterpret_cast<int2*>(P + a.b);           // [b] {first child, count}
  int* par = reinterpret_cast<int*>(kids + a.b);           // [b] parent (-1 at roots)
  __shared__ int s_off[kMaxLevels + 1], s_j0[kMaxLevels + 1];
  __shared__ double2 s_src[kMaxRoots];  // source injection of the root level (zero elsewhere)
  __shared__ int s_slot_lvl[kMaxSlots];
  __shared__ int s_case, s_next;
  __shared__ double s_red[kTreeThreads / 32];
  __shared__ uint32_t s_tmem;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int L = a.levels;
  for (int i = tid; i <= L; i += kTreeThreads) {
    s_off[i] = a.lvl[i];
    s_j0[i] = a.lvl[L + 1 + i];
  }
  for (int m = tid; m < a.b; m += kTreeThreads) {
    const int4 inf = __ldg(&a.info[m]);
    kids[m] = make_int2(inf.z, inf.w);
    par[m] = inf.y;
  }
  __syncthreads();
  for (int m = tid; m < s_off[1] && m < kMaxRoots; m += kTreeThreads) s_src[m] = __ldg(&a.coef[3 * a.b + m]);
  if (tid < kMaxSlots) {
    int lv = 0;
    for (int d = 0; d < L; ++d)
      if (s_j0[d] <= tid && tid < s_j0[d + 1]) lv = d;
    s_slot_lvl[tid] = lv;
  }
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tm = s_tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * 128);
  const uint32_t tm_v = tm, tm_s = tm + 4 * kMaxSlots;
  const int nslots = s_j0[L];
  // node of TMEM slot j of this thread (-1 if none): slot j belongs to level s_slot_lvl[j]
  auto slot_node = [&](int j) {
    if (j >= nslots) return -1;
    const int d = s_slot_lvl[j];
    const int m = s_off[d] + (j - s_j0[d]) * kTreeThreads + tid;
    return m < s_off[d + 1] ? m : -1;
  };

#ifdef TPF_PHASE_TIMING
  long long tc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_begin = clock64();
#endif
  // cases are claimed one ahead: while case k iterates, the loads of case
  // k + 1 are already on their way from HBM into L2 (prefetch at k's load)
  auto claim = [&]() {
    const unsigned long long c = atomicAdd(a.counter, 1ull);
    return c < (unsigned long long)a.tau ? int(c) : -1;
  };
  if (tid == 0) s_next = claim();
  for (;;) {
    TREE_T(t_load);
    if (tid == 0) {
      s_case = s_next;
      s_next = s_case < 0 ? -1 : claim();
    }
    __syncthreads();
    const int cs = s_case, nx = s_next;
    if (cs < 0) break;

    // ---- load the case: S into TMEM, flat start V (dense.py:155) ----
    // all of this thread's slots at once: the S loads are independent HBM/L2
    // round trips, so they are issued together before any TMEM store
#pragma unroll
    for (int j0 = 0; j0 < kMaxSlots; j0 += 4) {
      double2 sv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = slot_node(j0 + j);
        sv[j] = make_double2(0.0, 0.0);
        if (m >= 0) {
          const int64_t row = int64_t(__ldg(&a.info[m].x)) * a.s_node;
          sv[j] = __ldg(a.S + row + int64_t(cs) * a.s_case);
          if (nx >= 0 && a.prefetch) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.S + row + int64_t(nx) * a.s_case));
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j0 + j < nslots) {  // warp-uniform
          double2 v0 = a.v_flat;
          if (ZIP && a.v0) {  // fpi.py:141-145: opts.initial_voltage
            const int m = slot_node(j0 + j);
            if (m >= 0) v0 = __ldg(a.v0 + __ldg(&a.info[m].x));
          }
          tmem_st2(tm_s + 4 * (j0 + j), sv[j]);
          tmem_st2(tm_v + 4 * (j0 + j), v0);
        }
      }
    }
    tmem_wait_st();

    // Per level, every thread holds the data of its (at most kLS) slots of that
    // level in registers: the TMEM iterate/load and the node coefficients.  A
    // level's loads are issued right after the previous level's arithmetic,
    // BEFORE the barrier, so their latency overlaps the barrier wait.
    //   up:   z_m = r_m - sum_c P_c,  P_m = g_m z_m            (g = U[m,p] / U[m,m])
    //   down: w_m = z_m / U_mm - g_m w_p
    D2 vv[2], ss[2];
    double2 cg[kLS], cu[kLS];
    // global coefficient loads of a level, issued before the barrier that precedes it
    // node coefficients g and 1/U[m,m]: shared planes, or (ZIP) this case's own
    const double2* cgp = ZIP ? a.zcoef + size_t(blockIdx.x) * 2 * a.b : a.coef + a.b;
    const double2* cup = ZIP ? cgp + a.b : a.coef + 2 * a.b;
    auto issue_up = [&](int d) {
      const int jb = s_j0[d], je = s_j0[d + 1], off = s_off[d], end = s_off[d + 1];
#pragma unroll
      for (int u = 0; u < kLS; ++u) {
        const int m = off + u * kTreeThreads + tid;
#ifdef TPF_TREE_NOCOEF
        cg[u] = make_double2(0.01 * m, 0.0);
#else
        cg[u] = (jb + u < je && m < end) ? cgp[m] : make_double2(0.0, 0.0);
#endif
      }
    };
    auto issue_down = [&](int d) {
      const int jb = s_j0[d], je = s_j0[d + 1], off = s_off[d], end = s_off[d + 1];
#pragma unroll
      for (int u = 0; u < kLS; ++u) {
        const int m = off + u * kTreeThreads + tid;
        const bool ok = jb + u < je && m < end;
#ifdef TPF_TREE_NOCOEF
        cu[u] = make_double2(ok ? 1.0 : 0.0, 0.0);
        cg[u] = make_double2(0.01 * m, 0.0);
#else
        cu[u] = ok ? cup[m] : make_double2(0.0, 0.0);
        cg[u] = (ok && d > 0) ? cgp[m] : make_double2(0.0, 0.0);
#endif
      }
    };

    TREE_ACC(0, t_load);
#ifdef TPF_PHASE_TIMING
    if (tid == 0) tc[5] += 1;
#endif
    bool anz = true;  // ZIP: some alpha_p s != 0 (else fpi.py:150-163: one application)
    if constexpr (ZIP) {
      // this case's LU of B = Y_dd + diag(alpha_z s*) (assemble_fpi, fpi.py:107-127):
      // leaf-first, no fill, so U[m,m] = B[m,m] - sum_c e_c^2 / U[c,c] and
      // g_m = e_m / U[m,m] (e_m = Y[parent, m] = Y[m, parent]); level by level
      double2* zg = a.zcoef + size_t(blockIdx.x) * 2 * a.b;
      int any = 0, bad = 0;
      for (int d = L - 1; d >= 0; --d) {
        const int off = s_off[d], end = s_off[d + 1], jb = s_j0[d], je = s_j0[d + 1];
        for (int u = 0; u < kLS; ++u) {
          if (jb + u >= je) break;  // warp-uniform
          D2 sd;
          tmem_ld2(tm_s + 4 * (jb + u), sd);
          tmem_wait_ld();
          const int m = off + u * kTreeThreads + tid;
          if (m < end) {
            const double2 sl = sd.get();
            const double az = __ldg(a.alpha + m), ap = __ldg(a.alpha + 2 * a.b + m);
            const double2 yd = __ldg(a.ydiag + m);
            double2 piv = make_double2(__fma_rn(az, sl.x, yd.x), __fma_rn(-az, sl.y, yd.y));
            const int2 k = kids[m];
            for (int c = k.x; c < k.x + k.y; ++c) {
              const double2 pc = P[c];
              piv.x -= pc.x;
              piv.y -= pc.y;
            }
            const double n2 = __fma_rn(piv.x, piv.x, piv.y * piv.y);
            if (!(n2 > 0.0) || !isfinite(n2)) bad = 1;  // splu: "Factor is exactly singular" (also for NaN)
            const double rr = 1.0 / n2;
            const double2 ui = make_double2(piv.x * rr, -piv.y * rr);  // 1 / U[m,m]
            const double2 e = __ldg(&a.coef[m]);
            const double2 g = cmul2(e, ui);
            zg[m] = g;
            zg[a.b + m] = ui;
            P[m] = cmul2(e, g);  // e_m^2 / U[m,m], pulled by the parent
            if (ap != 0.0 && (sl.x != 0.0 || sl.y != 0.0)) any = 1;
          }
        }
        __syncthreads();
      }
      if (bad) atomicExch(a.status, 1);
      anz = __syncthreads_or(any) != 0;
      __threadfence_block();
    }
    int it = 0;
    bool met = false;  // fpi.py step_met
    issue_up(L - 1);
    while (it < a.max_iter) {
      TREE_T(t_up);
      // ---- up-sweep: deepest level first ----
      for (int d = L - 1; d >= 0; --d) {
        const int off = s_off[d], end = s_off[d + 1], jb = s_j0[d], je = s_j0[d + 1];
        // slots in pairs: both TMEM loads, one wait, two independent chains
#pragma unroll
        for (int u0 = 0; u0 < kLS; u0 += 2) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (jb + u0 + h < je) {  // warp-uniform
              tmem_ld2(tm_v + 4 * (jb + u0 + h), vv[h]);
              tmem_ld2(tm_s + 4 * (jb + u0 + h), ss[h]);
            }
          if (jb + u0 < je) tmem_wait_ld();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int u = u0 + h;
            const int m = off + u * kTreeThreads + tid;
            if (jb + u < je && m < end) {
              double2 v = vv[h].get();
              const double2 sl = ss[h].get();
              double m2 = __fma_rn(v.x, v.x, v.y * v.y);
              if (m2 < kZeroGuard2) {  // fpi.py:39-41
                v = make_double2(kZeroGuard, 0.0);
                m2 = kZeroGuard * kZeroGuard;
              }
              const double r = rcp_nr(m2);
              const double2 src = d == 0 ? s_src[m] : make_double2(0.0, 0.0);
              // r_m = -(s*/conj(v) + src),  s*/conj(v) = conj(s) v / |v|^2
              double2 z = make_double2(-(__fma_rn(sl.x, v.x, sl.y * v.y) * r + src.x),
                                       -(__fma_rn(sl.x, v.y, -(sl.y * v.x)) * r + src.y));
              if constexpr (ZIP) {  // r_m = -(alpha_p s*/conj(v) + src + alpha_i s*)
                const double ai = __ldg(a.alpha + a.b + m), ap = __ldg(a.alpha + 2 * a.b + m);
                const double ur = __fma_rn(sl.x, v.x, sl.y * v.y) * r, uim = __fma_rn(sl.x, v.y, -(sl.y * v.x)) * r;
                z = make_double2(-(ap * ur + src.x + ai * sl.x), -(ap * uim + src.y - ai * sl.y));
                if (!anz) z = make_double2(-(src.x + ai * sl.x), -(src.y - ai * sl.y));
              }
              const int2 k = kids[m];
              for (int c = k.x; c < k.x + k.y; ++c) {
                const double2 pc = P[c];
                z.x -= pc.x;
                z.y -= pc.y;
              }
              T[m] = z;
              P[m] = cmul2(cg[u], z);
            }
          }
        }
        if (d > 0)
          issue_up(d - 1);
        else
          issue_down(0);
        __syncthreads();
      }
      TREE_ACC(1, t_up);
      TREE_T(t_down);
      // ---- down-sweep: root level first, step test, iterate update ----
      bool small = true, fin = true;
      int all_small = 0, all_fin = 1;
      for (int d = 0; d < L; ++d) {
        const int off = s_off[d], end = s_off[d + 1], jb = s_j0[d], je = s_j0[d + 1];
#pragma unroll
        for (int u0 = 0; u0 < kLS; u0 += 2) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (jb + u0 + h < je) tmem_ld2(tm_v + 4 * (jb + u0 + h), vv[h]);
          if (jb + u0 < je) tmem_wait_ld();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int u = u0 + h;
            if (jb + u < je) {
              const int m = off + u * kTreeThreads + tid;
              double2 v = vv[h].get();
              double2 w = v;
              if (m < end) {
                w = cmul2(T[m], cu[u]);
                const int p = par[m];
                if (p >= 0) w = cfma_sub(w, cg[u], T[p]);
                T[m] = w;
                if (__fma_rn(v.x, v.x, v.y * v.y) < kZeroGuard2) v = make_double2(kZeroGuard, 0.0);
                const double dr = w.x - v.x, di = w.y - v.y;
                if (!(__fma_rn(dr, dr, di * di) < a.tol2)) small = false;  // NaN never passes
                if (ZIP && !(isfinite(w.x) && isfinite(w.y))) fin = false;
              }
              tmem_st2(tm_v + 4 * (jb + u), w);
            }
          }
        }
        tmem_wait_st();
        if (d + 1 < L) {
          issue_down(d + 1);
          __syncthreads();
        } else {
          all_small = __syncthreads_and(small);
          if constexpr (ZIP) all_fin = __syncthreads_and(fin);
        }
      }
      TREE_ACC(2, t_down);
      ++it;
      if (ZIP && !anz) {  // fpi.py:150-163: A = 0, one application, no step requirement
        met = true;
        break;
      }
      if (ZIP && !all_fin) break;  // fpi.py:178-181: diverged, not converged
      if (all_small) {
        met = true;
        break;
      }
      issue_up(L - 1);
    }

    TREE_T(t_ret);
    // ---- retire: V out, per-case count; with the fused residual V also goes
    // to T (the sweeps are done with it) ----
#pragma unroll
    for (int j0 = 0; j0 < kMaxSlots; j0 += 4) {
      D2 vo[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j0 + j < nslots) tmem_ld2(tm_v + 4 * (j0 + j), vo[j]);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = slot_node(j0 + j);
        if (m >= 0) {
          const double2 v = vo[j].get();
          a.V[__ldg(&a.info[m].x) * a.v_node + int64_t(cs) * a.v_case] = v;
          if (a.resid) T[m] = v;
        }
      }
    }
    TREE_ACC(3, t_ret);
    TREE_T(t_res);
    if (a.resid) {
      // residual_per_case (fpi.py:221-240): max_i |s_i + v_i conj(src_i + (Y_dd v)_i)|,
      // the operations of residual_kernel in the same order (bit-identical)
      __syncthreads();
      double worst = 0.0;
      // per slot: every ELL entry load is issued at once (one L2 round trip),
      // only the T[col] shared-memory reads depend on them
#pragma unroll 2
      for (int j = 0; j < nslots; ++j) {  // warp-uniform bound
        D2 sd;
        tmem_ld2(tm_s + 4 * j, sd);
        const int m = slot_node(j);
        double ar = 0.0, ai = 0.0;
        int len = 0;  // row length = diagonal + parent + children (checked by tpf_sparse_tree_build_ell)
        if (m >= 0) {
          const double2 si = __ldg(&a.coef[3 * a.b + m]);
          ar = si.x;
          ai = si.y;
          len = 1 + (par[m] >= 0) + kids[m].y;
        }
        for (int r0 = 0; r0 < a.ell_w; r0 += kEllChunk) {
          int c[kEllChunk];
          double2 y[kEllChunk];
#pragma unroll
          for (int r = 0; r < kEllChunk; ++r) {
            const bool ok = r0 + r < len;  // padding entries are not loaded
            c[r] = ok ? __ldg(a.ell_col + (r0 + r) * a.b + m) : -1;
            y[r] = ok ? __ldg(a.ell_val + (r0 + r) * a.b + m) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int r = 0; r < kEllChunk; ++r) {
            if (c[r] >= 0) {
              const double2 v = T[c[r]];
              ar = __fma_rn(y[r].x, v.x, __fma_rn(-y[r].y, v.y, ar));
              ai = __fma_rn(y[r].x, v.y, __fma_rn(y[r].y, v.x, ai));
            }
          }
        }
        tmem_wait_ld();
        if (m >= 0) {
          const double2 v = T[m];
          const double2 sl = sd.get();
          double2 sload = sl;
          if constexpr (ZIP) {  // fpi.py:229-235: az s |v|^2 + ai s v + ap s
            const double az = __ldg(a.alpha + m), zi = __ldg(a.alpha + a.b + m), zp = __ldg(a.alpha + 2 * a.b + m);
            const double v2 = v.x * v.x + v.y * v.y;
            const double2 sv = cmul2(sl, v);
            sload = make_double2(az * sl.x * v2 + zi * sv.x + zp * sl.x, az * sl.y * v2 + zi * sv.y + zp * sl.y);
          }
          const double mr = sload.x + (v.x * ar + v.y * ai);
          const double mi = sload.y + (v.y * ar - v.x * ai);
          worst = nanmax(worst, hypot(mr, mi));
        }
      }
      for (int o = 16; o > 0; o >>= 1) worst = nanmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
      if ((tid & 31) == 0) s_red[warp] = worst;
      __syncthreads();
      if (tid == 0) {
        double w = 0.0;
        for (int k = 0; k < kTreeThreads / 32; ++k) w = nanmax(w, s_red[k]);
        a.resid[cs] = w;
      }
    }
    TREE_ACC(4, t_res);
#ifdef TPF_PHASE_TIMING
    if (tid == 0) tc[6] += it;
#endif
    if (tid == 0) a.iters[cs] = it;
    if constexpr (ZIP) {
      if (tid == 0) a.met[cs] = met ? 1 : 0;
    }
  }
#ifdef TPF_PHASE_TIMING
  if (tid == 0 && blockIdx.x < 148) {
    tc[7] = clock64() - t_begin;
    for (int i = 0; i < 8; ++i) g_tree_cyc[blockIdx.x * 8 + i] = tc[i];
  }
#endif
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(s_tmem, 512);
}

}  // namespace
}  // namespace tpf

using namespace tpf;

extern "C" int tpf_sparse_tree_max_slots(void) { return kMaxSlots; }

#ifdef TPF_PHASE_TIMING
extern "C" int tpf_debug_tree_phase_cycles(long long* out) {
  return cudaMemcpyFromSymbol(out, g_tree_cyc, sizeof(g_tree_cyc)) == cudaSuccess ? 0 : 1;
}
#endif

static int tree_launch(int64_t tau, int32_t b, int32_t levels, const int32_t* level_info, const int32_t* node_info,
                       const double* node_coef, const double* S, int64_t s_node_stride, int64_t s_case_stride,
                       double v_flat_re, double v_flat_im, double tol, int32_t max_iter, double* V,
                       int64_t v_node_stride, int64_t v_case_stride, int32_t* iters, int32_t ell_w,
                       const int32_t* ell_col, const double* ell_val, double* resid, void* workspace,
                       size_t workspace_bytes, void* stream, const double* alpha = nullptr,
                       const double* ydiag = nullptr, int32_t* status = nullptr, uint8_t* met = nullptr,
                       const double* v0 = nullptr) {
  const bool zip = alpha != nullptr;
  if (tau < 0 || b < 1 || levels < 1 || levels > kMaxLevels)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_fpi_c128: bad shape");
  if (!(tol > 0.0)) return set_error(TPF_ERR_INVALID, "tolerance must be positive");
  if (max_iter < 1) return set_error(TPF_ERR_INVALID, "max_iterations must be >= 1");
  if (tau == 0) return TPF_OK;
  if (!level_info || !node_info || !node_coef || !S || !V || !iters || !workspace || workspace_bytes < 256)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_fpi_c128: null pointer or small workspace");
  if (resid && (!ell_col || !ell_val || ell_w < 1 || ell_w > kMaxEllWidth))
    return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_fpi_resid_c128: bad ELL rows");
  const size_t smem = size_t(b) * (2 * sizeof(double2) + sizeof(int2) + sizeof(int));
  if (smem > 220 * 1024) return set_error(TPF_ERR_UNSUPPORTED, "tpf_sparse_tree_fpi_c128: b too large for one SM");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto kern = zip ? sparse_tree_kernel<true> : sparse_tree_kernel<false>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (err != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(tree)", err);
  err = cudaMemsetAsync(workspace, 0, sizeof(unsigned long long), st);
  if (err != cudaSuccess) return set_cuda_error("cudaMemsetAsync(counter)", err);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = sms;
  if (tau < grid) grid = tau;
  if (zip && workspace_bytes < 256 + size_t(grid) * 2 * size_t(b) * sizeof(double2))
    return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_zip_fpi_c128: workspace too small");
  TreeArgs a;
  a.tau = tau;
  a.b = b;
  a.levels = levels;
  a.S = reinterpret_cast<const double2*>(S);
  a.s_node = s_node_stride;
  a.s_case = s_case_stride;
  a.V = reinterpret_cast<double2*>(V);
  a.v_node = v_node_stride;
  a.v_case = v_case_stride;
  a.iters = iters;
  a.counter = static_cast<unsigned long long*>(workspace);
  a.lvl = level_info;
  a.info = reinterpret_cast<const int4*>(node_info);
  a.coef = reinterpret_cast<const double2*>(node_coef);
  a.v_flat = make_double2(v_flat_re, v_flat_im);
  a.v0 = reinterpret_cast<const double2*>(v0);
  a.tol2 = tol * tol;
  a.max_iter = max_iter;
  a.ell_w = ell_w;
  a.ell_col = ell_col;
  a.ell_val = reinterpret_cast<const double2*>(ell_val);
  a.resid = resid;
  a.alpha = alpha;
  a.ydiag = reinterpret_cast<const double2*>(ydiag);
  a.zcoef = reinterpret_cast<double2*>(static_cast<char*>(workspace) + 256);
  a.status = status;
  a.met = met;
  static const int pf = [] {
    const char* e = getenv("TPF_TREE_PREFETCH");
    return e ? atoi(e) : 0;  // off: measured neutral at 1 MB node stride, -10% at 8 MB (TLB reach)
  }();
  a.prefetch = pf;
  kern<<<unsigned(grid), kTreeThreads, smem, st>>>(a);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error("launch(sparse_tree_kernel)", err);
  return TPF_OK;
}

extern "C" int tpf_sparse_tree_fpi_c128(int64_t tau, int32_t b, int32_t levels, const int32_t* level_info,
                                        const int32_t* node_info, const double* node_coef, const double* S,
                                        int64_t s_node_stride, int64_t s_case_stride, double v_flat_re,
                                        double v_flat_im, double tol, int32_t max_iter, double* V,
                                        int64_t v_node_stride, int64_t v_case_stride, int32_t* iters,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  return tree_launch(tau, b, levels, level_info, node_info, node_coef, S, s_node_stride, s_case_stride, v_flat_re,
                     v_flat_im, tol, max_iter, V, v_node_stride, v_case_stride, iters, 0, nullptr, nullptr, nullptr,
                     workspace, workspace_bytes, stream);
}

extern "C" int tpf_sparse_tree_fpi_resid_c128(int64_t tau, int32_t b, int32_t levels, const int32_t* level_info,
                                              const int32_t* node_info, const double* node_coef, const double* S,
                                              int64_t s_node_stride, int64_t s_case_stride, double v_flat_re,
                                              double v_flat_im, double tol, int32_t max_iter, double* V,
                                              int64_t v_node_stride, int64_t v_case_stride, int32_t* iters,
                                              int32_t ell_width, const int32_t* ell_col, const double* ell_val,
                                              double* resid, void* workspace, size_t workspace_bytes, void* stream) {
  if (!resid) return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_fpi_resid_c128: null resid");
  return tree_launch(tau, b, levels, level_info, node_info, node_coef, S, s_node_stride, s_case_stride, v_flat_re,
                     v_flat_im, tol, max_iter, V, v_node_stride, v_case_stride, iters, ell_width, ell_col, ell_val,
                     resid, workspace, workspace_bytes, stream);
}

extern "C" size_t tpf_sparse_tree_zip_workspace_bytes(int64_t tau, int32_t b) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = sms;
  if (tau < grid) grid = tau;
  if (grid < 1) grid = 1;
  return 256 + size_t(grid) * 2 * size_t(b) * sizeof(double2);
}

extern "C" int tpf_sparse_tree_zip_fpi_c128(int64_t tau, int32_t b, int32_t levels, const int32_t* level_info,
                                            const int32_t* node_info, const double* node_coef, const double* alpha,
                                            const double* ydiag, const double* S, int64_t s_node_stride,
                                            int64_t s_case_stride, double v_flat_re, double v_flat_im,
                                            const double* v0, double tol, int32_t max_iter, double* V, int64_t v_node_stride,
                                            int64_t v_case_stride, int32_t* iters, int32_t ell_width,
                                            const int32_t* ell_col, const double* ell_val, double* resid,
                                            uint8_t* step_met, int32_t* status, void* workspace,
                                            size_t workspace_bytes, void* stream) {
  if (!alpha || !ydiag || !resid || !status || !step_met)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_zip_fpi_c128: null alpha / ydiag / resid / step_met / status");
  return tree_launch(tau, b, levels, level_info, node_info, node_coef, S, s_node_stride, s_case_stride, v_flat_re,
                     v_flat_im, tol, max_iter, V, v_node_stride, v_case_stride, iters, ell_width, ell_col, ell_val,
                     resid, workspace, workspace_bytes, stream, alpha, ydiag, status, step_met, v0);
}

extern "C" int tpf_sparse_tree_ell_width(int32_t b, const int32_t* ydd_row_ptr) {
  if (b < 1 || !ydd_row_ptr) {
    set_error(TPF_ERR_INVALID, "tpf_sparse_tree_ell_width: bad argument");
    return -1;
  }
  int w = 0;
  for (int i = 0; i < b; ++i) w = ydd_row_ptr[i + 1] - ydd_row_ptr[i] > w ? ydd_row_ptr[i + 1] - ydd_row_ptr[i] : w;
  return w;
}

extern "C" int tpf_sparse_tree_build_ell(int32_t b, int32_t width, const int32_t* node_info,
                                         const int32_t* ydd_row_ptr, const int32_t* ydd_col, const double* ydd_val,
                                         int32_t* ell_col, double* ell_val) {
  if (b < 1 || width < 1 || !node_info || !ydd_row_ptr || !ydd_col || !ydd_val || !ell_col || !ell_val)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_build_ell: bad argument");
  std::vector<int32_t> m_of(size_t(b), -1);
  for (int m = 0; m < b; ++m) {
    const int i = node_info[4 * m];
    if (i < 0 || i >= b || m_of[i] >= 0) return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_build_ell: bad node_info");
    m_of[i] = m;
  }
  for (int m = 0; m < b; ++m) {
    const int i = node_info[4 * m];
    const int lo = ydd_row_ptr[i], n = ydd_row_ptr[i + 1] - lo;
    if (n > width) return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_build_ell: row wider than width");
    // the kernel reads row m's length from the tree (diagonal + parent + children)
    if (n != 1 + (node_info[4 * m + 1] >= 0 ? 1 : 0) + node_info[4 * m + 3])
      return set_error(TPF_ERR_UNSUPPORTED, "tpf_sparse_tree_build_ell: Y_dd row is not diagonal + tree edges");
    for (int r = 0; r < width; ++r) {
      const size_t at = size_t(r) * b + m;
      if (r < n) {
        const int c = ydd_col[lo + r];
        if (c < 0 || c >= b) return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_build_ell: bad column");
        ell_col[at] = m_of[c];
        ell_val[2 * at] = ydd_val[2 * (lo + r)];
        ell_val[2 * at + 1] = ydd_val[2 * (lo + r) + 1];
      } else {
        ell_col[at] = -1;
        ell_val[2 * at] = ell_val[2 * at + 1] = 0.0;
      }
    }
  }
  return TPF_OK;
}

extern "C" int tpf_sparse_tree_max_ell_width(void) { return kMaxEllWidth; }
