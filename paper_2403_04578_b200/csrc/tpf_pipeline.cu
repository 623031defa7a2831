// End-to-end host pipeline: the C-ABI entry points that take HOST buffers.
//
// A full reference-sized batch (C2: 841 MB of loads in, 841 MB of voltages out)
// is moved over PCIe in tau-chunks on three streams so that the H2D copy of
// chunk i+1, the solve of chunk i and the D2H copy of chunk i-1 overlap:
//
//   in   : [H2D 0][H2D 1][H2D 2] ...
//   comp :        [solve 0][solve 1] ...      (iteration kernel + residual)
//   out  :                 [D2H 0 ][D2H 1 ] ...
//
// Two device slots per stream stage; events order slot reuse.  Per-case
// outputs (iters, residuals, mask) stay device-resident until one final
// summary kernel and copy.  Pageable host buffers are page-locked in place for
// the duration of the call (cudaHostRegister) so every copy is a DMA.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <thread>
#include <vector>

#include "tpf_common.cuh"
#include "tpf_internal.h"

namespace tpf {
namespace {

struct HostPin {
  void* ptr = nullptr;
  bool registered = false;
  int pin(const void* p, size_t bytes, bool read_only) {
    cudaPointerAttributes attr;
    cudaError_t err = cudaPointerGetAttributes(&attr, p);
    if (err == cudaSuccess && (attr.type == cudaMemoryTypeHost || attr.type == cudaMemoryTypeManaged)) return TPF_OK;
    cudaGetLastError();  // clear a pageable-pointer query error
    unsigned flags = cudaHostRegisterPortable | (read_only ? cudaHostRegisterReadOnly : 0u);
    err = cudaHostRegister(const_cast<void*>(p), bytes, flags);
    if (err != cudaSuccess) {
      cudaGetLastError();
      return TPF_OK;  // fall back to pageable copies (correct, slower)
    }
    ptr = const_cast<void*>(p);
    registered = true;
    return TPF_OK;
  }
  ~HostPin() {
    if (registered) cudaHostUnregister(ptr);
  }
};

bool host_pinned(const void* p) {
  cudaPointerAttributes attr;
  cudaError_t err = cudaPointerGetAttributes(&attr, p);
  if (err != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost || attr.type == cudaMemoryTypeManaged;
}

// Page-locked staging for pageable loads: registering a caller's 841 MB array
// costs ~75 ms per call (page pinning at ~11 GB/s), more than the whole C2
// transfer; instead each chunk is copied by host threads into one of two
// pinned staging buffers (grow-only, per calling thread) while the GPU works
// on the previous chunk.
struct Staging {
  void* p = nullptr;
  size_t bytes = 0;
  ~Staging() {
    if (p) cudaFreeHost(p);
  }
  cudaError_t ensure(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaHostAlloc(&p, n, cudaHostAllocPortable);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
};
thread_local Staging g_staging;

// Copy `rows` rows of `row_bytes` (source pitch src_pitch) into dst (pitch
// dst_pitch) with a few host threads.
void parallel_copy2d(char* dst, size_t dst_pitch, const char* src, size_t src_pitch, size_t row_bytes,
                     int64_t rows) {
  int nt = int(std::thread::hardware_concurrency());
  if (nt > 16) nt = 16;
  const size_t total = row_bytes * size_t(rows);
  if (total < (size_t(8) << 20) || nt < 2) nt = 1;
  if (int64_t(nt) > rows) nt = int(rows > 0 ? rows : 1);
  auto work = [&](int w) {
    const int64_t lo = rows * w / nt, hi = rows * (w + 1) / nt;
    for (int64_t r = lo; r < hi; ++r) memcpy(dst + size_t(r) * dst_pitch, src + size_t(r) * src_pitch, row_bytes);
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < nt; ++w) pool.emplace_back(work, w);
  work(0);
  for (auto& t : pool) t.join();
}

// Layout of a b x tau complex host matrix: either node-major (case stride 1,
// the reference LoadMatrix / VoltageBatch layout) or case-major (node stride 1).
struct HostLayout {
  bool case_contig;  // case stride == 1
  int64_t ld;        // stride of the other index
  int ok(int64_t b, int64_t tau, int64_t node_stride, int64_t case_stride) {
    if (case_stride == 1 && node_stride >= tau) {
      case_contig = true;
      ld = node_stride;
      return 1;
    }
    if (node_stride == 1 && case_stride >= b) {
      case_contig = false;
      ld = case_stride;
      return 1;
    }
    return 0;
  }
  size_t span_bytes(int64_t b, int64_t tau) const {
    return case_contig ? size_t(ld) * (b - 1) * 16 + size_t(tau) * 16 : size_t(ld) * (tau - 1) * 16 + size_t(b) * 16;
  }
};

// Copy cases [lo, hi) between a host matrix and a device chunk buffer laid out
// the same way (node-major chunk: ld = chunk; case-major chunk: ld = b).
cudaError_t copy_chunk(bool h2d, const HostLayout& L, double* host, double* dev, int64_t b, int64_t lo, int64_t n,
                       int64_t chunk, cudaStream_t st) {
  if (L.case_contig) {
    char* h = reinterpret_cast<char*>(host) + size_t(lo) * 16;
    if (n == L.ld && n == chunk)  // the whole batch in one chunk: one contiguous block
      return h2d ? cudaMemcpyAsync(dev, h, size_t(n) * b * 16, cudaMemcpyHostToDevice, st)
                 : cudaMemcpyAsync(h, dev, size_t(n) * b * 16, cudaMemcpyDeviceToHost, st);
    if (h2d)
      return cudaMemcpy2DAsync(dev, size_t(chunk) * 16, h, size_t(L.ld) * 16, size_t(n) * 16, size_t(b),
                               cudaMemcpyHostToDevice, st);
    return cudaMemcpy2DAsync(h, size_t(L.ld) * 16, dev, size_t(chunk) * 16, size_t(n) * 16, size_t(b),
                             cudaMemcpyDeviceToHost, st);
  }
  char* h = reinterpret_cast<char*>(host) + size_t(lo) * size_t(L.ld) * 16;
  if (L.ld == b) {
    return h2d ? cudaMemcpyAsync(dev, h, size_t(n) * b * 16, cudaMemcpyHostToDevice, st)
               : cudaMemcpyAsync(h, dev, size_t(n) * b * 16, cudaMemcpyDeviceToHost, st);
  }
  if (h2d)
    return cudaMemcpy2DAsync(dev, size_t(b) * 16, h, size_t(L.ld) * 16, size_t(b) * 16, size_t(n),
                             cudaMemcpyHostToDevice, st);
  return cudaMemcpy2DAsync(h, size_t(L.ld) * 16, dev, size_t(b) * 16, size_t(b) * 16, size_t(n),
                           cudaMemcpyDeviceToHost, st);
}

// Device buffer carved from a caller workspace (no allocation) or, when the
// caller passes none, owned via cudaMalloc/cudaFree.
struct Arena {
  char* base = nullptr;
  size_t size = 0, used = 0;
};
thread_local Arena* g_arena = nullptr;

struct DevBuf {
  void* p = nullptr;
  bool owned = false;
  ~DevBuf() {
    if (owned && p) cudaFree(p);
  }
  cudaError_t alloc(size_t n) {
    n = (n ? n : 16);
    if (g_arena) {
      const size_t need = (n + 255) / 256 * 256;
      if (g_arena->used + need > g_arena->size) return cudaErrorMemoryAllocation;
      p = g_arena->base + g_arena->used;
      g_arena->used += need;
      return cudaSuccess;
    }
    owned = true;
    return cudaMalloc(&p, n);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct Streams {
  cudaStream_t s[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t in_done[2], comp_done[2], out_done[2];
  bool ok = false;
  cudaError_t init() {
    for (auto& x : s) {
      cudaError_t e = cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
      if (e != cudaSuccess) return e;
    }
    for (int k = 0; k < 2; ++k) {
      cudaEventCreateWithFlags(&in_done[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&comp_done[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&out_done[k], cudaEventDisableTiming);
    }
    ok = true;
    return cudaSuccess;
  }
  ~Streams() {
    if (!ok) return;
    for (int k = 0; k < 2; ++k) {
      cudaEventDestroy(in_done[k]);
      cudaEventDestroy(comp_done[k]);
      cudaEventDestroy(out_done[k]);
    }
    for (auto& x : s)
      if (x) cudaStreamDestroy(x);
  }
};

// Streams and events of the pipeline, created once per (thread, device) and
// reused: creating 3 streams + 6 events per call costs ~0.1 ms, a visible
// share of a small batch's end-to-end time.
Streams* cached_streams(int device) {
  thread_local std::map<int, std::unique_ptr<Streams>> cache;
  std::unique_ptr<Streams>& p = cache[device];
  if (!p) {
    p.reset(new Streams);
    if (p->init() != cudaSuccess) {
      p.reset();
      return nullptr;
    }
  }
  return p.get();
}

#define TPF_CK(expr, where)                           \
  do {                                                \
    cudaError_t _e = (expr);                          \
    if (_e != cudaSuccess) return set_cuda_error(where, _e); \
  } while (0)

// Inside the chunk loop: record the error and leave the loop, so the streams
// are still synchronised (queued copies may target the caller's host buffers,
// which HostPin unregisters on return) and the setup event is destroyed.
#define TPF_CK_LOOP(expr, where)                \
  {                                             \
    cudaError_t _e = (expr);                    \
    if (_e != cudaSuccess) {                    \
      rc = set_cuda_error(where, _e);           \
      break;                                    \
    }                                           \
  }

template <class T>
cudaError_t upload(DevBuf& d, const T* h, size_t n, cudaStream_t st) {
  cudaError_t e = d.alloc(n * sizeof(T));
  if (e != cudaSuccess || n == 0) return e;
  return cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyDefault, st);  // host or device source (UVA)
}

// Solver callback: run the iteration on device chunk (S_dev -> V_dev) for n cases.
struct ChunkSolver {
  virtual ~ChunkSolver() = default;
  virtual int solve(int64_t n, const double* S, int64_t sn, int64_t sc, double* V, int64_t vn, int64_t vc,
                    int32_t* iters, cudaStream_t st) = 0;
  // solvers whose kernel also computes the residual post-check override this
  // (returning 1 = done, the separate residual kernel is skipped)
  virtual int solve_resid(int64_t, const double*, int64_t, int64_t, double*, int64_t, int64_t, int32_t*,
                          const int32_t*, const int32_t*, const double*, const double*, double*, cudaStream_t) {
    return -1;
  }
};

int run_pipeline(ChunkSolver& solver, int64_t tau, int b, const double* S, int64_t s_node, int64_t s_case,
                 const int32_t* rp, const int32_t* ci, const double* yv, const double* src, double residual_tol,
                 double* V, int64_t v_node, int64_t v_case, int32_t* iters, double* resid, uint8_t* mask,
                 int32_t* summary, int64_t chunk, const Streams& ss, cudaStream_t setup) {
  const auto h0 = std::chrono::steady_clock::now();
  auto hms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count(); };
  double h_mark = 0, h_loop = 0;
  HostLayout LS, LV;
  if (!LS.ok(b, tau, s_node, s_case)) return set_error(TPF_ERR_INVALID, "host S must be node-major or case-major");
  if (!LV.ok(b, tau, v_node, v_case)) return set_error(TPF_ERR_INVALID, "host V must be node-major or case-major");
  HostPin pin_s, pin_v, pin_i, pin_r, pin_m;
  const bool stage_s = !host_pinned(S);  // pageable loads: staged (registering costs ms even for one chunk)
  if (stage_s) {
    TPF_CK(g_staging.ensure(size_t(2) * size_t(chunk) * b * 16), "cudaHostAlloc(staging)");
  } else {
    pin_s.pin(S, LS.span_bytes(b, tau), true);
  }
  pin_v.pin(V, LV.span_bytes(b, tau), false);
  if (iters) pin_i.pin(iters, size_t(tau) * 4, false);
  if (resid) pin_r.pin(resid, size_t(tau) * 8, false);
  if (mask) pin_m.pin(mask, size_t(tau), false);

  const int nnz = 0;
  (void)nnz;
  DevBuf d_rp, d_ci, d_yv, d_src, d_it, d_res, d_mask, d_sum, d_S[2], d_V[2];
  int64_t ynnz = 0;
  {
    // row_ptr lives on the host: read nnz from it
    ynnz = rp[b];
  }
  TPF_CK(upload(d_rp, rp, size_t(b) + 1, setup), "upload(row_ptr)");
  TPF_CK(upload(d_ci, ci, size_t(ynnz), setup), "upload(col)");
  TPF_CK(upload(d_yv, yv, size_t(ynnz) * 2, setup), "upload(val)");
  TPF_CK(upload(d_src, src, size_t(b) * 2, setup), "upload(src)");
  TPF_CK(d_it.alloc(size_t(tau) * 4), "cudaMalloc(iters)");
  TPF_CK(d_res.alloc(size_t(tau) * 8), "cudaMalloc(resid)");
  TPF_CK(d_mask.alloc(size_t(tau)), "cudaMalloc(mask)");
  TPF_CK(d_sum.alloc(64), "cudaMalloc(summary)");
  for (int k = 0; k < 2; ++k) {
    TPF_CK(d_S[k].alloc(size_t(chunk) * b * 16), "cudaMalloc(S chunk)");
    TPF_CK(d_V[k].alloc(size_t(chunk) * b * 16), "cudaMalloc(V chunk)");
  }
  cudaEvent_t setup_done;
  TPF_CK(cudaEventCreateWithFlags(&setup_done, cudaEventDisableTiming), "cudaEventCreate");
  cudaEventRecord(setup_done, setup);
  cudaStream_t sin = ss.s[0], scomp = ss.s[1], sout = ss.s[2];
  cudaStreamWaitEvent(scomp, setup_done, 0);
  // device chunk strides mirror the host layout so each chunk copy is one 2-D DMA
  const int64_t dsn_S = LS.case_contig ? chunk : 1, dsc_S = LS.case_contig ? 1 : b;
  const int64_t dsn_V = LV.case_contig ? chunk : 1, dsc_V = LV.case_contig ? 1 : b;
  // chunk boundaries: with more than 4 chunks the first and the last are a
  // quarter chunk, which shortens the pipeline fill (first H2D, nothing to
  // overlap it with) and drain (last D2H); the rest are full chunks
  std::vector<int64_t> bnd{0};
  {
    static const bool no_ramp = [] {  // TPF_PIPE_NORAMP=1: equal chunks (A/B only)
      const char* e = getenv("TPF_PIPE_NORAMP");
      return e && e[0] == '1';
    }();
    static const int64_t div = [] {  // TPF_PIPE_RAMP_DIV: ramp chunk = chunk / div (A/B only)
      const char* e = getenv("TPF_PIPE_RAMP_DIV");
      const long v = e ? atol(e) : 0;
      return int64_t(v >= 2 && v <= 64 ? v : 4);
    }();
    const int64_t small =
        tau > 4 * chunk && !no_ramp ? std::max<int64_t>(chunk / div / 256 * 256, 256) : chunk;
    int64_t at = 0;
    if (small < chunk) bnd.push_back(at = small);
    while (tau - at > chunk + (small < chunk ? small : 0)) bnd.push_back(at += chunk);
    if (small < chunk && tau - at > small) bnd.push_back(at = tau - small);
    if (at < tau) bnd.push_back(tau);
  }
  const int64_t nchunks = int64_t(bnd.size()) - 1;
  // TPF_PIPE_TRACE=1 (diagnostics only): per-chunk timeline on stderr
  static const bool trace = [] {
    const char* e = getenv("TPF_PIPE_TRACE");
    return e && e[0] == '1';
  }();
  std::vector<cudaEvent_t> tev;
  auto mark = [&](cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tev.push_back(e);
  };
  mark(setup);
  h_mark = hms();
  std::vector<double> h_chunk;
  int rc = TPF_OK;
  for (int64_t c = 0; c < nchunks && rc == TPF_OK; ++c) {
    const int k = int(c & 1);
    const int64_t lo = bnd[c], n = bnd[c + 1] - bnd[c];
    if (trace) h_chunk.push_back(hms());
    if (c >= 2) cudaStreamWaitEvent(sin, ss.comp_done[k], 0);
    if (stage_s) {
      // staging slot k was last read by the H2D of chunk c - 2
      if (c >= 2) TPF_CK_LOOP(cudaEventSynchronize(ss.in_done[k]), "staging reuse");
      char* stg = static_cast<char*>(g_staging.p) + size_t(k) * size_t(chunk) * b * 16;
      const char* hs = reinterpret_cast<const char*>(S);
      if (LS.case_contig) {  // b rows of n cases -> [b][chunk] pitch chunk
        parallel_copy2d(stg, size_t(chunk) * 16, hs + size_t(lo) * 16, size_t(LS.ld) * 16, size_t(n) * 16, b);
        TPF_CK_LOOP(cudaMemcpy2DAsync(d_S[k].as<double>(), size_t(chunk) * 16, stg, size_t(chunk) * 16, size_t(n) * 16,
                                 size_t(b), cudaMemcpyHostToDevice, sin),
               "H2D(S chunk)");
      } else {  // n cases of b nodes -> [n][b]
        parallel_copy2d(stg, size_t(b) * 16, hs + size_t(lo) * size_t(LS.ld) * 16, size_t(LS.ld) * 16,
                        size_t(b) * 16, n);
        TPF_CK_LOOP(cudaMemcpyAsync(d_S[k].as<double>(), stg, size_t(n) * b * 16, cudaMemcpyHostToDevice, sin),
               "H2D(S chunk)");
      }
    } else {
      TPF_CK_LOOP(copy_chunk(true, LS, const_cast<double*>(S), d_S[k].as<double>(), b, lo, n, chunk, sin),
             "H2D(S chunk)");
    }
    cudaEventRecord(ss.in_done[k], sin);
    mark(sin);
    cudaStreamWaitEvent(scomp, ss.in_done[k], 0);
    if (c >= 2) cudaStreamWaitEvent(scomp, ss.out_done[k], 0);
    rc = solver.solve_resid(n, d_S[k].as<double>(), dsn_S, dsc_S, d_V[k].as<double>(), dsn_V, dsc_V,
                            d_it.as<int32_t>() + lo, d_rp.as<int32_t>(), d_ci.as<int32_t>(), d_yv.as<double>(),
                            d_src.as<double>(), d_res.as<double>() + lo, scomp);
    if (rc == TPF_OK) {
      cudaEventRecord(ss.comp_done[k], scomp);
      mark(scomp);
      cudaStreamWaitEvent(sout, ss.comp_done[k], 0);
      TPF_CK_LOOP(copy_chunk(false, LV, V, d_V[k].as<double>(), b, lo, n, chunk, sout), "D2H(V chunk)");
      cudaEventRecord(ss.out_done[k], sout);
      mark(sout);
      continue;
    }
    if (rc > 0) break;  // a real error from the fused solver
    rc = solver.solve(n, d_S[k].as<double>(), dsn_S, dsc_S, d_V[k].as<double>(), dsn_V, dsc_V,
                      d_it.as<int32_t>() + lo, scomp);
    if (rc != TPF_OK) break;
    rc = tpf_residual_c128(n, b, d_S[k].as<double>(), dsn_S, dsc_S, d_V[k].as<double>(), dsn_V, dsc_V,
                           d_rp.as<int32_t>(), d_ci.as<int32_t>(), d_yv.as<double>(), d_src.as<double>(),
                           d_res.as<double>() + lo, scomp);
    if (rc != TPF_OK) break;
    cudaEventRecord(ss.comp_done[k], scomp);
    mark(scomp);
    cudaStreamWaitEvent(sout, ss.comp_done[k], 0);
    TPF_CK_LOOP(copy_chunk(false, LV, V, d_V[k].as<double>(), b, lo, n, chunk, sout), "D2H(V chunk)");
    cudaEventRecord(ss.out_done[k], sout);
    mark(sout);
  }
  if (rc == TPF_OK) {
    rc = tpf_batch_summary(tau, d_it.as<int32_t>(), d_res.as<double>(), residual_tol, d_mask.as<uint8_t>(),
                           d_sum.as<int32_t>(), scomp);
  }
  if (rc == TPF_OK) {
    cudaEvent_t fin;
    cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
    cudaEventRecord(fin, scomp);
    cudaStreamWaitEvent(sout, fin, 0);
    if (iters) cudaMemcpyAsync(iters, d_it.p, size_t(tau) * 4, cudaMemcpyDeviceToHost, sout);
    if (resid) cudaMemcpyAsync(resid, d_res.p, size_t(tau) * 8, cudaMemcpyDeviceToHost, sout);
    if (mask) cudaMemcpyAsync(mask, d_mask.p, size_t(tau), cudaMemcpyDeviceToHost, sout);
    if (summary) cudaMemcpyAsync(summary, d_sum.p, 8, cudaMemcpyDeviceToHost, sout);
    cudaEventDestroy(fin);
  }
  mark(sout);
  h_loop = hms();
  cudaError_t e1 = cudaStreamSynchronize(sin), e2 = cudaStreamSynchronize(scomp), e3 = cudaStreamSynchronize(sout);
  if (trace) {
    fprintf(stderr, "[tpf pipe] host: setup mark enqueued %.2f ms, loop enqueued %.2f ms, synced %.2f ms; chunk starts:", h_mark, h_loop, hms());
    for (double t : h_chunk) fprintf(stderr, " %.2f", t);
    fprintf(stderr, "\n");
  }
  if (trace && !tev.empty()) {  // in / compute / out completion times of each chunk, ms after the setup mark
    fprintf(stderr, "[tpf pipe] %lld chunks, chunk %lld:", (long long)nchunks, (long long)chunk);
    for (size_t i = 1; i < tev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[0], tev[i]);
      fprintf(stderr, " %.2f", ms);
    }
    fprintf(stderr, "\n");
    for (auto e : tev) cudaEventDestroy(e);
  }
  cudaEventDestroy(setup_done);
  if (rc != TPF_OK) return rc;
  if (e1 != cudaSuccess) return set_cuda_error("pipeline(in)", e1);
  if (e2 != cudaSuccess) return set_cuda_error("pipeline(compute)", e2);
  if (e3 != cudaSuccess) return set_cuda_error("pipeline(out)", e3);
  return TPF_OK;
}

struct ArenaScope {
  Arena a;
  ArenaScope(void* ws, size_t bytes) {
    if (ws) {
      a.base = static_cast<char*>(ws);
      a.size = bytes;
      g_arena = &a;
    }
  }
  ~ArenaScope() { g_arena = nullptr; }
};

// Device bytes a host pipeline call carves from its workspace (see the
// run_pipeline allocations): per-case outputs, two S and V chunk slots,
// model arrays and the solver workspace.
size_t pipeline_bytes(int64_t tau, int b, int64_t chunk, size_t model_bytes, size_t solver_ws) {
  auto r = [](size_t n) { return (n + 255) / 256 * 256 + 256; };
  return r(size_t(tau) * 4) + r(size_t(tau) * 8) + r(size_t(tau)) + r(64) + 4 * r(size_t(chunk) * b * 16) +
         model_bytes + r(solver_ws) + 4096;
}

int64_t pick_chunk(int64_t tau, int b, int64_t requested) {
  if (requested > 0) return requested < tau ? requested : (tau > 0 ? tau : 1);
  int64_t c = (tau + 15) / 16;  // ~16 chunks: fill/drain costs ~1/8 of the transfer time
  if (c < 16384) c = 16384;     // enough cases per launch to fill 148 SMs
  c = (c + 4095) / 4096 * 4096;
  // but at most ~192 MB of S per chunk: the first H2D and the last D2H are
  // not overlapped, so a chunk's transfer time is the pipeline's fill+drain
  int64_t cap = (int64_t(192) << 20) / (int64_t(b) * 16);
  if (cap < 1024) cap = 1024;
  cap = cap / 256 * 256;
  if (c > cap) c = cap;
  return c < tau ? c : (tau > 0 ? tau : 1);
}

struct DenseChunk : ChunkSolver {
  int b;
  const double *K, *W;
  double vre, vim, tol;
  int max_iter;
  void* ws;
  size_t ws_bytes;
  int solve(int64_t n, const double* S, int64_t sn, int64_t sc, double* V, int64_t vn, int64_t vc, int32_t* it,
            cudaStream_t st) override {
    return tpf_dense_fpi_c128(n, b, S, sn, sc, K, W, vre, vim, tol, max_iter, V, vn, vc, it, ws, ws_bytes, st);
  }
};

struct SparseChunk : ChunkSolver {
  int b;
  const int32_t *lp, *lc, *up, *uc, *perm;
  const double *lv, *uv, *ud, *src;
  double vre, vim, tol;
  int max_iter;
  void* ws;
  size_t ws_bytes;
  int solve(int64_t n, const double* S, int64_t sn, int64_t sc, double* V, int64_t vn, int64_t vc, int32_t* it,
            cudaStream_t st) override {
    return tpf_sparse_fpi_c128(n, b, S, sn, sc, lp, lc, lv, up, uc, uv, ud, perm, src, vre, vim, tol, max_iter, V,
                               vn, vc, it, ws, ws_bytes, st);
  }
};

struct TreeChunk : ChunkSolver {
  int b, levels;
  const int32_t *lvl, *info;
  const double* coef;
  double vre, vim, tol;
  int max_iter;
  void* ws;
  size_t ws_bytes;
  int solve(int64_t n, const double* S, int64_t sn, int64_t sc, double* V, int64_t vn, int64_t vc, int32_t* it,
            cudaStream_t st) override {
    return tpf_sparse_tree_fpi_c128(n, b, levels, lvl, info, coef, S, sn, sc, vre, vim, tol, max_iter, V, vn, vc, it,
                                    ws, ws_bytes, st);
  }
  int ell_w = 0;  // 0: Y_dd rows too wide for the fused residual
  const int32_t* ell_col = nullptr;
  const double* ell_val = nullptr;
  int solve_resid(int64_t n, const double* S, int64_t sn, int64_t sc, double* V, int64_t vn, int64_t vc, int32_t* it,
                  const int32_t*, const int32_t*, const double*, const double*, double* resid,
                  cudaStream_t st) override {
    if (ell_w < 1) return -1;
    return tpf_sparse_tree_fpi_resid_c128(n, b, levels, lvl, info, coef, S, sn, sc, vre, vim, tol, max_iter, V, vn,
                                          vc, it, ell_w, ell_col, ell_val, resid, ws, ws_bytes, st);
  }
};

// warp-per-subtree kernel (tpf_sparse_subtree_fpi_c128) with the fused residual
struct SubtreeChunk : ChunkSolver {
  int b, ns, nt, rmax, rw, nkids;
  const int32_t *pinfo, *slotinfo;
  const uint16_t* kids;
  const double *coef, *ell_val;
  const int32_t* ell_col;
  double vre, vim, tol;
  int max_iter;
  void* ws;
  size_t ws_bytes;
  int solve(int64_t n, const double* S, int64_t sn, int64_t sc, double* V, int64_t vn, int64_t vc, int32_t* it,
            cudaStream_t st) override {
    return tpf_sparse_subtree_fpi_c128(n, b, ns, nt, rmax, rw, nkids, pinfo, slotinfo, kids, coef, ell_col, ell_val,
                                       S, sn, sc, vre, vim, tol, max_iter, V, vn, vc, it, nullptr, ws, ws_bytes, st);
  }
  int solve_resid(int64_t n, const double* S, int64_t sn, int64_t sc, double* V, int64_t vn, int64_t vc, int32_t* it,
                  const int32_t*, const int32_t*, const double*, const double*, double* resid,
                  cudaStream_t st) override {
    return tpf_sparse_subtree_fpi_c128(n, b, ns, nt, rmax, rw, nkids, pinfo, slotinfo, kids, coef, ell_col, ell_val,
                                       S, sn, sc, vre, vim, tol, max_iter, V, vn, vc, it, resid, ws, ws_bytes, st);
  }
};

}  // namespace
}  // namespace tpf

using namespace tpf;

extern "C" size_t tpf_sparse_subtree_solve_host_workspace_bytes(int64_t tau, int32_t b, int32_t ns, int32_t nt,
                                                                int32_t rw, int32_t nkids, int64_t chunk_cases,
                                                                int64_t ydd_nnz) {
  const int64_t chunk = pick_chunk(tau, b, chunk_cases);
  const int64_t P = int64_t(tpf_sparse_subtree_warps()) * (ns + nt) * 32;
  const size_t model = size_t(P) * (8 + 48 + size_t(rw) * 20) + size_t(12) * ns * 4 + size_t(nkids) * 2 +
                       size_t(ydd_nnz) * 24 + size_t(b) * 32 + 64 * 1024;
  return pipeline_bytes(tau, b, chunk, model, tpf_sparse_subtree_workspace_bytes(chunk, b));
}

extern "C" int tpf_sparse_subtree_solve_host_c128(int64_t tau, int32_t b, int32_t ns, int32_t nt, int32_t rmax,
                                                  int32_t rw, int32_t nkids, const int32_t* pinfo,
                                                  const int32_t* slotinfo, const uint16_t* kids, const double* coef,
                                                  const int32_t* ell_col, const double* ell_val, const double* S,
                                                  int64_t s_node_stride, int64_t s_case_stride,
                                                  const int32_t* ydd_row_ptr, const int32_t* ydd_col,
                                                  const double* ydd_val, const double* src, double v_flat_re,
                                                  double v_flat_im, double tol, int32_t max_iter, double residual_tol,
                                                  double* V, int64_t v_node_stride, int64_t v_case_stride,
                                                  int32_t* iters, double* resid, uint8_t* mask, int32_t* summary,
                                                  int64_t chunk_cases, int32_t device, void* workspace,
                                                  size_t workspace_bytes) {
  if (tau < 0 || b < 1 || ns < 1 || nt < 1)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_subtree_solve_host_c128: bad shape");
  if (!S || !pinfo || !slotinfo || !kids || !coef || !ell_col || !ell_val || !ydd_row_ptr || !src || !V)
    return set_error(TPF_ERR_INVALID, "null pointer");
  TPF_CK(cudaSetDevice(device), "cudaSetDevice");
  if (summary) summary[0] = summary[1] = 0;
  if (tau == 0) return TPF_OK;
  if (workspace && workspace_bytes < tpf_sparse_subtree_solve_host_workspace_bytes(tau, b, ns, nt, rw, nkids,
                                                                                  chunk_cases, ydd_row_ptr[b]))
    return set_error(TPF_ERR_INVALID, "tpf_sparse_subtree_solve_host_c128: workspace too small");
  ArenaScope arena(workspace, workspace_bytes);
  Streams* ssp = cached_streams(device);
  if (!ssp) return set_cuda_error("cudaStreamCreate", cudaGetLastError());
  const Streams& ss = *ssp;
  const int64_t chunk = pick_chunk(tau, b, chunk_cases);
  cudaStream_t st = ss.s[1];
  const int64_t P = int64_t(tpf_sparse_subtree_warps()) * (ns + nt) * 32;
  DevBuf dpi, dsi, dk, dc, dec, dev_, dws;
  TPF_CK(upload(dpi, pinfo, size_t(P) * 2, st), "upload(pinfo)");
  TPF_CK(upload(dsi, slotinfo, size_t(tpf_sparse_subtree_warps()) * ns, st), "upload(slotinfo)");
  TPF_CK(upload(dk, kids, size_t(nkids), st), "upload(kids)");
  TPF_CK(upload(dc, coef, size_t(P) * 6, st), "upload(coef)");
  TPF_CK(upload(dec, ell_col, size_t(rw) * P, st), "upload(ell_col)");
  TPF_CK(upload(dev_, ell_val, size_t(rw) * P * 2, st), "upload(ell_val)");
  const size_t wsb = tpf_sparse_subtree_workspace_bytes(chunk, b);
  TPF_CK(dws.alloc(wsb), "cudaMalloc(workspace)");
  SubtreeChunk sv;
  sv.b = b;
  sv.ns = ns;
  sv.nt = nt;
  sv.rmax = rmax;
  sv.rw = rw;
  sv.nkids = nkids;
  sv.pinfo = dpi.as<int32_t>();
  sv.slotinfo = dsi.as<int32_t>();
  sv.kids = static_cast<const uint16_t*>(dk.p);
  sv.coef = dc.as<double>();
  sv.ell_col = dec.as<int32_t>();
  sv.ell_val = dev_.as<double>();
  sv.vre = v_flat_re;
  sv.vim = v_flat_im;
  sv.tol = tol;
  sv.max_iter = max_iter;
  sv.ws = dws.p;
  sv.ws_bytes = wsb;
  return run_pipeline(sv, tau, b, S, s_node_stride, s_case_stride, ydd_row_ptr, ydd_col, ydd_val, src, residual_tol,
                      V, v_node_stride, v_case_stride, iters, resid, mask, summary, chunk, ss, st);
}

extern "C" int tpf_host_pin(void* ptr, size_t bytes) {
  if (!ptr || bytes == 0) return 0;
  cudaPointerAttributes attr;
  cudaError_t err = cudaPointerGetAttributes(&attr, ptr);
  if (err == cudaSuccess && (attr.type == cudaMemoryTypeHost || attr.type == cudaMemoryTypeManaged)) return 0;
  cudaGetLastError();
  err = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable);
  if (err != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return 1;
}

extern "C" int tpf_host_unpin(void* ptr) {
  cudaError_t err = cudaHostUnregister(ptr);
  if (err != cudaSuccess) {
    cudaGetLastError();
    return set_cuda_error("cudaHostUnregister", err);
  }
  return TPF_OK;
}

extern "C" size_t tpf_sparse_tree_solve_host_workspace_bytes(int64_t tau, int32_t b, int64_t chunk_cases,
                                                             int64_t ydd_nnz) {
  const int64_t chunk = pick_chunk(tau, b, chunk_cases);
  const size_t model = size_t(b) * 256 + size_t(ydd_nnz) * 24 + size_t(b) * 16 * 20 + 64 * 1024;
  return pipeline_bytes(tau, b, chunk, model, 256);
}

extern "C" int tpf_sparse_tree_solve_host_c128(int64_t tau, int32_t b, int32_t levels, const int32_t* level_info,
                                               const int32_t* node_info, const double* node_coef, const double* S,
                                               int64_t s_node_stride, int64_t s_case_stride,
                                               const int32_t* ydd_row_ptr, const int32_t* ydd_col,
                                               const double* ydd_val, const double* src, double v_flat_re,
                                               double v_flat_im, double tol, int32_t max_iter, double residual_tol,
                                               double* V, int64_t v_node_stride, int64_t v_case_stride,
                                               int32_t* iters, double* resid, uint8_t* mask, int32_t* summary,
                                               int64_t chunk_cases, int32_t device, void* workspace,
                                               size_t workspace_bytes) {
  if (tau < 0 || b < 1 || levels < 1)
    return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_solve_host_c128: bad shape");
  if (!S || !level_info || !node_info || !node_coef || !ydd_row_ptr || !src || !V)
    return set_error(TPF_ERR_INVALID, "null pointer");
  TPF_CK(cudaSetDevice(device), "cudaSetDevice");
  if (summary) summary[0] = summary[1] = 0;
  if (tau == 0) return TPF_OK;
  if (workspace && workspace_bytes < tpf_sparse_tree_solve_host_workspace_bytes(tau, b, chunk_cases, ydd_row_ptr[b]))
    return set_error(TPF_ERR_INVALID, "tpf_sparse_tree_solve_host_c128: workspace too small");
  ArenaScope arena(workspace, workspace_bytes);
  Streams* ssp = cached_streams(device);
  if (!ssp) return set_cuda_error("cudaStreamCreate", cudaGetLastError());
  const Streams& ss = *ssp;
  const int64_t chunk = pick_chunk(tau, b, chunk_cases);
  cudaStream_t st = ss.s[1];
  DevBuf dl, di, dc, dws;
  TPF_CK(upload(dl, level_info, size_t(levels + 1) * 2, st), "upload(levels)");
  TPF_CK(upload(di, node_info, size_t(b) * 4, st), "upload(node_info)");
  TPF_CK(upload(dc, node_coef, size_t(b) * 8, st), "upload(node_coef)");
  TPF_CK(dws.alloc(256), "cudaMalloc(workspace)");
  // level-ordered ELL rows of Y_dd for the residual fused into the tree kernel
  const int ell_w = tpf_sparse_tree_ell_width(b, ydd_row_ptr);
  std::vector<int32_t> h_ec;
  std::vector<double> h_ev;
  DevBuf dec, dev_;
  bool fuse = ydd_col && ydd_val && ell_w >= 1 && ell_w <= tpf_sparse_tree_max_ell_width();
  if (fuse) {
    h_ec.resize(size_t(ell_w) * b);
    h_ev.resize(size_t(ell_w) * b * 2);
    if (tpf_sparse_tree_build_ell(b, ell_w, node_info, ydd_row_ptr, ydd_col, ydd_val, h_ec.data(), h_ev.data()) ==
        TPF_OK) {
      TPF_CK(upload(dec, h_ec.data(), h_ec.size(), st), "upload(ell_col)");
      TPF_CK(upload(dev_, h_ev.data(), h_ev.size(), st), "upload(ell_val)");
    } else {
      fuse = false;  // not a plain tree pattern: separate residual kernel
    }
  }
  TreeChunk sv;
  if (fuse) {
    sv.ell_w = ell_w;
    sv.ell_col = dec.as<int32_t>();
    sv.ell_val = dev_.as<double>();
  }
  sv.b = b;
  sv.levels = levels;
  sv.lvl = dl.as<int32_t>();
  sv.info = di.as<int32_t>();
  sv.coef = dc.as<double>();
  sv.vre = v_flat_re;
  sv.vim = v_flat_im;
  sv.tol = tol;
  sv.max_iter = max_iter;
  sv.ws = dws.p;
  sv.ws_bytes = 256;
  return run_pipeline(sv, tau, b, S, s_node_stride, s_case_stride, ydd_row_ptr, ydd_col, ydd_val, src, residual_tol,
                      V, v_node_stride, v_case_stride, iters, resid, mask, summary, chunk, ss, st);
}

extern "C" size_t tpf_dense_solve_host_workspace_bytes(int64_t tau, int32_t b, int64_t chunk_cases,
                                                       int64_t ydd_nnz) {
  const int64_t chunk = pick_chunk(tau, b, chunk_cases);
  const bool large = b > tpf_dense_max_nodes();
  const size_t solver = large ? tpf_dense_large_workspace_bytes(chunk, b) : tpf_dense_workspace_bytes(b);
  const size_t model = size_t(b) * b * 16 + size_t(b) * 128 + size_t(ydd_nnz) * 24 + 64 * 1024;
  return pipeline_bytes(tau, b, chunk, model, solver);
}

extern "C" size_t tpf_sparse_solve_host_workspace_bytes(int64_t tau, int32_t b, int64_t chunk_cases,
                                                        int64_t ydd_nnz, int64_t l_nnz, int64_t u_nnz) {
  const int64_t chunk = pick_chunk(tau, b, chunk_cases);
  const size_t model = size_t(b) * 128 + size_t(ydd_nnz + l_nnz + u_nnz) * 24 + 64 * 1024;
  return pipeline_bytes(tau, b, chunk, model, tpf_sparse_workspace_bytes(chunk, b));
}

extern "C" int tpf_dense_solve_host_c128(int64_t tau, int32_t b, const double* S, int64_t s_node_stride,
                                         int64_t s_case_stride, const double* K, const double* W,
                                         const int32_t* ydd_row_ptr, const int32_t* ydd_col,
                                         const double* ydd_val, const double* src, double v_flat_re,
                                         double v_flat_im, double tol, int32_t max_iter, double residual_tol,
                                         double* V, int64_t v_node_stride, int64_t v_case_stride, int32_t* iters,
                                         double* resid, uint8_t* mask, int32_t* summary, int64_t chunk_cases,
                                         int32_t device, void* workspace, size_t workspace_bytes) {
  if (tau < 0 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_dense_solve_host_c128: need tau >= 0, b >= 1");
  if (!S || !K || !W || !ydd_row_ptr || !src || !V) return set_error(TPF_ERR_INVALID, "null pointer");
  TPF_CK(cudaSetDevice(device), "cudaSetDevice");
  if (summary) summary[0] = summary[1] = 0;
  if (tau == 0) return TPF_OK;
  if (workspace && workspace_bytes < tpf_dense_solve_host_workspace_bytes(tau, b, chunk_cases, ydd_row_ptr[b]))
    return set_error(TPF_ERR_INVALID, "tpf_dense_solve_host_c128: workspace too small");
  ArenaScope arena(workspace, workspace_bytes);
  Streams* ssp = cached_streams(device);
  if (!ssp) return set_cuda_error("cudaStreamCreate", cudaGetLastError());
  const Streams& ss = *ssp;
  const bool large = b > tpf_dense_max_nodes();
  const int64_t chunk = pick_chunk(tau, b, chunk_cases);
  DevBuf dK, dW, dws;
  TPF_CK(upload(dK, K, size_t(b) * b * 2, ss.s[1]), "upload(K)");
  TPF_CK(upload(dW, W, size_t(b) * 2, ss.s[1]), "upload(W)");
  size_t wsb = large ? tpf_dense_large_workspace_bytes(chunk, b) : tpf_dense_workspace_bytes(b);
  TPF_CK(dws.alloc(wsb), "cudaMalloc(workspace)");
  struct LargeChunk : DenseChunk {
    int solve(int64_t n, const double* S, int64_t sn, int64_t sc, double* V, int64_t vn, int64_t vc, int32_t* it,
              cudaStream_t st) override {
      return tpf_dense_fpi_large_c128(n, b, S, sn, sc, K, W, vre, vim, tol, max_iter, V, vn, vc, it, ws, ws_bytes,
                                      st);
    }
  };
  DenseChunk small_solver;
  LargeChunk large_solver;
  DenseChunk& sv = large ? static_cast<DenseChunk&>(large_solver) : small_solver;
  sv.b = b;
  sv.K = dK.as<double>();
  sv.W = dW.as<double>();
  sv.vre = v_flat_re;
  sv.vim = v_flat_im;
  sv.tol = tol;
  sv.max_iter = max_iter;
  sv.ws = dws.p;
  sv.ws_bytes = wsb;
  return run_pipeline(sv, tau, b, S, s_node_stride, s_case_stride, ydd_row_ptr, ydd_col, ydd_val, src, residual_tol,
                      V, v_node_stride, v_case_stride, iters, resid, mask, summary, chunk, ss, ss.s[1]);
}

extern "C" int tpf_sparse_solve_host_c128(int64_t tau, int32_t b, const double* S, int64_t s_node_stride,
                                          int64_t s_case_stride, const int32_t* l_ptr, const int32_t* l_col,
                                          const double* l_val, const int32_t* u_ptr, const int32_t* u_col,
                                          const double* u_val, const double* u_diag_inv, const int32_t* perm,
                                          const int32_t* ydd_row_ptr, const int32_t* ydd_col,
                                          const double* ydd_val, const double* src, double v_flat_re,
                                          double v_flat_im, double tol, int32_t max_iter, double residual_tol,
                                          double* V, int64_t v_node_stride, int64_t v_case_stride, int32_t* iters,
                                          double* resid, uint8_t* mask, int32_t* summary, int64_t chunk_cases,
                                          int32_t device, void* workspace, size_t workspace_bytes) {
  if (tau < 0 || b < 1) return set_error(TPF_ERR_INVALID, "tpf_sparse_solve_host_c128: need tau >= 0, b >= 1");
  if (!S || !l_ptr || !u_ptr || !perm || !ydd_row_ptr || !src || !V) return set_error(TPF_ERR_INVALID, "null pointer");
  TPF_CK(cudaSetDevice(device), "cudaSetDevice");
  if (summary) summary[0] = summary[1] = 0;
  if (tau == 0) return TPF_OK;
  if (workspace && workspace_bytes < tpf_sparse_solve_host_workspace_bytes(tau, b, chunk_cases, ydd_row_ptr[b],
                                                                            l_ptr[b], u_ptr[b]))
    return set_error(TPF_ERR_INVALID, "tpf_sparse_solve_host_c128: workspace too small");
  ArenaScope arena(workspace, workspace_bytes);
  Streams* ssp = cached_streams(device);
  if (!ssp) return set_cuda_error("cudaStreamCreate", cudaGetLastError());
  const Streams& ss = *ssp;
  const int64_t chunk = pick_chunk(tau, b, chunk_cases);
  const int64_t lnnz = l_ptr[b], unnz = u_ptr[b];
  DevBuf dlp, dlc, dlv, dup, duc, duv, dud, dperm, dsrc, dws;
  cudaStream_t st = ss.s[1];
  TPF_CK(upload(dlp, l_ptr, size_t(b) + 1, st), "upload(L)");
  TPF_CK(upload(dlc, l_col, size_t(lnnz), st), "upload(L)");
  TPF_CK(upload(dlv, l_val, size_t(lnnz) * 2, st), "upload(L)");
  TPF_CK(upload(dup, u_ptr, size_t(b) + 1, st), "upload(U)");
  TPF_CK(upload(duc, u_col, size_t(unnz), st), "upload(U)");
  TPF_CK(upload(duv, u_val, size_t(unnz) * 2, st), "upload(U)");
  TPF_CK(upload(dud, u_diag_inv, size_t(b) * 2, st), "upload(U)");
  TPF_CK(upload(dperm, perm, size_t(b) * 2, st), "upload(perm)");
  TPF_CK(upload(dsrc, src, size_t(b) * 2, st), "upload(src)");
  const size_t wsb = tpf_sparse_workspace_bytes(chunk, b);
  TPF_CK(dws.alloc(wsb), "cudaMalloc(workspace)");
  SparseChunk sv;
  sv.b = b;
  sv.lp = dlp.as<int32_t>();
  sv.lc = dlc.as<int32_t>();
  sv.lv = dlv.as<double>();
  sv.up = dup.as<int32_t>();
  sv.uc = duc.as<int32_t>();
  sv.uv = duv.as<double>();
  sv.ud = dud.as<double>();
  sv.perm = dperm.as<int32_t>();
  sv.src = dsrc.as<double>();
  sv.vre = v_flat_re;
  sv.vim = v_flat_im;
  sv.tol = tol;
  sv.max_iter = max_iter;
  sv.ws = dws.p;
  sv.ws_bytes = wsb;
  return run_pipeline(sv, tau, b, S, s_node_stride, s_case_stride, ydd_row_ptr, ydd_col, ydd_val, src, residual_tol,
                      V, v_node_stride, v_case_stride, iters, resid, mask, summary, chunk, ss, st);
}
