/*
 * tpf.h -- C ABI of the B200-native Tensor Power Flow engine (libtpf.so).
 *
 * The reference (`tpflow`, pure Python) has no FFI: its hot-path "operator
 * API" is the Python pair batch_solve_dense / batch_solve_sparse
 * (pkg/src/tpflow/dense.py:129-134, sparse.py:167-172) dispatched by
 * solve_batch (bench.py:96-111).  The Python package
 * `paper_2403_04578_b200` re-exposes those signatures and calls the entry
 * points below through ctypes; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - complex128 data are interleaved (re, im) doubles; strides are counted in
 *    complex elements.  Element (node i, case j) of a b x tau matrix lives at
 *    index i*node_stride + j*case_stride.  The reference's LoadMatrix layout
 *    (b x tau, C order, dense.py:57-78) is node_stride = tau, case_stride = 1.
 *  - "_c128" entry points take DEVICE pointers, are stream-ordered on the
 *    given cudaStream_t (NULL = legacy default stream) and never synchronize.
 *    "_host" entry points take HOST pointers and return after completion.
 *  - Every entry point returns TPF_OK (0) or an error code; the message of
 *    the last failure on the calling thread is tpf_last_error().
 *  - Stateless; safe to call concurrently on different devices/streams.
 *
 * Semantics (both solvers): flat start v = v_flat for every node; each
 * iteration applies the zero-voltage guard (|v| < 1e-12 -> 1e-12, fpi.py:39-41),
 * the fixed-point update, and a per-case step test max_i |v'_i - v_i| < tol
 * (dense.py:125-126, 189-193).  A case stops at its first passing step or at
 * max_iter ("per-case freeze"); iters[j] is its update count.  The reference's
 * batch `iterations` equals max_j iters[j] (test_dense.py:72-79).  Non-finite
 * steps never pass, so diverging cases run to max_iter, as in the reference.
 */
#ifndef TPF_H_
#define TPF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPF_OK 0
#define TPF_ERR_INVALID 1     /* bad argument (ValueError in the reference) */
#define TPF_ERR_CUDA 2        /* CUDA runtime failure */
#define TPF_ERR_UNSUPPORTED 3 /* shape not supported by this entry point */
#define TPF_ERR_SINGULAR 4    /* zero pivot (SingularSystemError, fpi.py:44) */
#define TPF_ERR_MEMORY 5      /* allocation failure (MemoryGuardError, sparse.py:55) */

/* ABI version (major*10000 + minor*100 + patch). */
int tpf_version(void);
/* Message of the last failed call on this thread ("" if none). */
const char* tpf_last_error(void);

/* ------------------------------------------------------ scenario loads --
 * Device scenario generator (replaces synth.py:131-156 for batches that only
 * exist on the device): per case j, node i: p = base[i] exp(sigma (sqrt(rho)
 * common_j + sqrt(1 - rho) idio_ij)), power factor U[0.9, 1] lagging, then
 * the batch scaled so max_j |sum_i s_ij| = scale_num (load_scale x margin).
 * Draws: Philox4x32-10 keyed by `key`, counter (case_offset + j, node pair,
 * stream): the same loads for a case whatever the launch or chunking.  S b x
 * tau complex (any strides), device; workspace >= tpf_gen_loads_workspace_bytes(). */
size_t tpf_gen_loads_workspace_bytes(void);
int tpf_gen_loads_c128(int64_t tau, int32_t b, const double* base, double rho, double sigma, uint64_t key,
                       int64_t case_offset, double scale_num, double* S, int64_t s_node_stride,
                       int64_t s_case_stride, void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- dense --
 * Replaces the hot loop of batch_solve_dense (dense.py:166-193) and its
 * per-iteration op chain _iterate_chunk (dense.py:114-126):
 *     V <- K (S* ./ conj(V)) + W,   K = -inv(Y_dd) (dense.py:151),
 *                                   W = K (Y_ds v_s) (dense.py:152).
 * K, W of the host pipelines (*_solve_host_c128) may be host or device
 * pointers (unified addressing).
 * FP64 tensor-core (DMMA) kernel with K resident in shared memory:
 * requires b <= tpf_dense_max_nodes() (104); larger b: the _large_ entry below.
 *   S      b x tau complex loads (consumption positive), device
 *   K      b x b complex, row-major, device
 *   W      b complex, device
 *   V      b x tau complex output, device
 *   iters  int32[tau] per-case update counts, device
 *   workspace >= tpf_dense_workspace_bytes(b) device bytes
 */
/* Dense setup on the device for radial feeders (replaces dense.py:150-152,
 * K = -inv(Y_dd) and W = K src on the host by LAPACK): column j of K is the
 * tree-LU solve Y_dd x = -e_j (one thread per column, O(b) each), then
 * W = K src.  The tree LU is the sparse path's (sparse.py:186; layout of
 * tpf_sparse_tree_fpi_c128: level offsets int32[levels + 1], node_info
 * int32[4 b] {original node, parent, first child, child count} in level
 * order, node_coef complex[4 b] planes e, g, 1/U[m,m], src).  K agrees with
 * LAPACK's inverse to rounding (not bitwise).  All pointers device; K b x b
 * row-major complex, W b complex, src b complex (original order).
 * Stream-ordered. */
int tpf_dense_setup_tree_c128(int32_t b, int32_t levels, const int32_t* level_off, const int32_t* node_info,
                              const double* node_coef, const double* src, double* K, double* W, void* stream);
int tpf_dense_max_nodes(void);
size_t tpf_dense_workspace_bytes(int32_t b);
int tpf_dense_fpi_c128(int64_t tau, int32_t b,
                       const double* S, int64_t s_node_stride, int64_t s_case_stride,
                       const double* K, const double* W,
                       double v_flat_re, double v_flat_im,
                       double tol, int32_t max_iter,
                       double* V, int64_t v_node_stride, int64_t v_case_stride,
                       int32_t* iters, void* workspace, size_t workspace_bytes,
                       void* stream);

/* The two b <= 104 kernels behind tpf_dense_fpi_c128 (same arguments, same
 * bits; tpf_dense_fpi_c128 picks pairs for batches of at most two waves of
 * ws slots, ws above; TPF_DENSE_KERNEL=pairs forces the second):
 *   _ws_    warp-specialised: per SM sub-partition one DMMA warp alternating
 *           between two slot groups and two elementwise warps (default);
 *   _pairs_ pairs of warps sharing 8 slots, each doing GEMM and elementwise. */
int tpf_dense_ws_fpi_c128(int64_t tau, int32_t b,
                          const double* S, int64_t s_node_stride, int64_t s_case_stride,
                          const double* K, const double* W, double v_flat_re, double v_flat_im,
                          double tol, int32_t max_iter, double* V, int64_t v_node_stride, int64_t v_case_stride,
                          int32_t* iters, void* workspace, size_t workspace_bytes, void* stream);
int tpf_dense_pairs_fpi_c128(int64_t tau, int32_t b,
                             const double* S, int64_t s_node_stride, int64_t s_case_stride,
                             const double* K, const double* W, double v_flat_re, double v_flat_im,
                             double tol, int32_t max_iter, double* V, int64_t v_node_stride, int64_t v_case_stride,
                             int32_t* iters, void* workspace, size_t workspace_bytes, void* stream);

/* Dense TPF for b > 104 (K streamed from L2; config C5, b = 1,000): an
 * iteration-synchronous loop over a compacted active set of unconverged cases,
 * tiled FP64-DMMA GEMM per iteration.  Same arguments and semantics as
 * tpf_dense_fpi_c128; works for any b >= 1.
 *   workspace >= tpf_dense_large_workspace_bytes(tau, b) device bytes      */
size_t tpf_dense_large_workspace_bytes(int64_t tau, int32_t b);
int tpf_dense_fpi_large_c128(int64_t tau, int32_t b,
                             const double* S, int64_t s_node_stride, int64_t s_case_stride,
                             const double* K, const double* W,
                             double v_flat_re, double v_flat_im,
                             double tol, int32_t max_iter,
                             double* V, int64_t v_node_stride, int64_t v_case_stride,
                             int32_t* iters, void* workspace, size_t workspace_bytes,
                             void* stream);

/* --------------------------------------------------------------- sparse --
 * Replaces the hot loop of batch_solve_sparse (sparse.py:186-197), which
 * re-solves a tau-block-diagonal SuperLU system per iteration.  Every block
 * is the equation Y_dd v'_j = -(s_j* ./ conj(v_j) + src), so one host LU
 * Pr Y_dd Pc = L U (factorized once) serves all cases:
 *   l_ptr/l_col/l_val   strictly-lower part of unit-diagonal L, CSR (int32, complex)
 *   u_ptr/u_col/u_val   strictly-upper part of U, CSR
 *   u_diag_inv          complex[b] = 1 / U[k,k]
 *   perm                int32[2b]: perm[k] = node whose right-hand side feeds
 *                       forward row k (row permutation), perm[b+i] = index of
 *                       node i's solution in the permuted unknowns (column perm.)
 *   src                 complex[b] = Y_ds v_s
 *   workspace >= tpf_sparse_workspace_bytes(tau, b) device bytes            */
size_t tpf_sparse_workspace_bytes(int64_t tau, int32_t b);
int tpf_sparse_fpi_c128(int64_t tau, int32_t b,
                        const double* S, int64_t s_node_stride, int64_t s_case_stride,
                        const int32_t* l_ptr, const int32_t* l_col, const double* l_val,
                        const int32_t* u_ptr, const int32_t* u_col, const double* u_val,
                        const double* u_diag_inv, const int32_t* perm, const double* src,
                        double v_flat_re, double v_flat_im, double tol, int32_t max_iter,
                        double* V, int64_t v_node_stride, int64_t v_case_stride,
                        int32_t* iters, void* workspace, size_t workspace_bytes,
                        void* stream);

/* Radial-feeder sparse solver, warp-per-subtree (default for radial feeders
 * whose schedule fits; paper_2403_04578_b200.subtree.subtree_schedule): the
 * tree LU is cut at depth D, the subtrees are packed onto 12 warps and
 * list-scheduled into slots of 32 independent nodes swept with __syncwarp
 * only (two slots at a time where independent), the top (depth < D) is swept
 * by every warp on a private copy; one CTA barrier per iteration.  One case
 * per SM; per thread and slot the iterate, the load and z / U_mm live in
 * Tensor Memory.  Per case the loads come in by TMA (one column of
 * node-major S, cp.async.bulk.tensor, or one case-major column,
 * cp.async.bulk), the next case's column is prefetched into L2, V goes out
 * by TMA, and the residual post-check (fpi.py:221-240) is fused when
 * resid != null.  Same arithmetic and bits as tpf_sparse_tree_fpi_c128.
 *   ns, nt      subtree slots (8 * ns + 4 * y-slots <= 168) and top slots
 *   rmax, rw    root slots per warp, residual row width (<= 8)
 *   pinfo       int32[2 * P] (P = 12 * (ns + nt) * 32 positions),
 *   slotinfo    int32[12 * ns], kids uint16[nkids], coef complex[3 * P]
 *               (g, 1/U[m,m], src), ell_col int32[P / 32][rw][32] and
 *               ell_val complex[P / 32][rw][32] (Y_dd rows in CSR order, blocked
 *               by slot; padding: X's zero entry, value 0): device arrays of
 *               the schedule
 *   S, V        node-major (case stride 1) or case-major (node stride 1), 16-B aligned
 *   workspace  >= 256 device bytes; with tpf_sparse_subtree_workspace_bytes(tau, b)
 *               a node-major batch is solved in case-major chunks of 65,536
 *               cases (transposed in and out on the device: contiguous
 *               per-case columns instead of b scattered rows)
 * tpf_sparse_subtree_smem_bytes: the kernel's shared memory for a schedule. */
int tpf_sparse_subtree_warps(void);
size_t tpf_sparse_subtree_workspace_bytes(int64_t tau, int32_t b);
size_t tpf_sparse_subtree_smem_bytes(int32_t b, int32_t ns, int32_t nt, int32_t rmax, int32_t nkids);
int tpf_sparse_subtree_fpi_c128(int64_t tau, int32_t b, int32_t ns, int32_t nt, int32_t rmax, int32_t rw,
                                int32_t nkids, const int32_t* pinfo, const int32_t* slotinfo,
                                const uint16_t* kids, const double* coef, const int32_t* ell_col,
                                const double* ell_val, const double* S, int64_t s_node_stride,
                                int64_t s_case_stride, double v_flat_re, double v_flat_im, double tol,
                                int32_t max_iter, double* V, int64_t v_node_stride, int64_t v_case_stride,
                                int32_t* iters, double* resid, void* workspace, size_t workspace_bytes,
                                void* stream);

/* Radial-feeder fast path of the sparse solver: one case per SM with the
 * whole case on chip (sweep vector in shared memory, iterate and loads in
 * Tensor Memory), level-synchronous up/down sweeps over the depth levels of
 * the zero-fill tree LU.  Inputs come from the host-built schedule
 * (paper_2403_04578_b200.sparse.tree_schedule):
 *   level_info  int32[2*(levels+1)]: node offsets per depth level (root level
 *               first), then the first TMEM slot of each level
 *   node_info   int32[4*b]: per level-ordered node {original node, parent,
 *               first child, child count} (parent -1 at the roots)
 *   node_coef   complex[4*b], four planes of b (coalesced per level):
 *               [0*b + m] e = Y[parent,m], [1*b + m] g = U[m,parent]/U[m,m],
 *               [2*b + m] 1/U[m,m], [3*b + m] src (symmetric Y_dd; src nonzero only at the
 *               root level, at most 512 root-level nodes, at most 6 slots
 *               (ceil(level size / 512)) per level)
 * Limits: b <= 5,120 (44 B of shared memory per node) and sum over levels of ceil(n_level/512) <=
 * tpf_sparse_tree_max_slots() (16); otherwise use tpf_sparse_fpi_c128.
 *   workspace >= 256 device bytes                                          */
int tpf_sparse_tree_max_slots(void);
int tpf_sparse_tree_fpi_c128(int64_t tau, int32_t b, int32_t levels,
                             const int32_t* level_info, const int32_t* node_info, const double* node_coef,
                             const double* S, int64_t s_node_stride, int64_t s_case_stride,
                             double v_flat_re, double v_flat_im, double tol, int32_t max_iter,
                             double* V, int64_t v_node_stride, int64_t v_case_stride,
                             int32_t* iters, void* workspace, size_t workspace_bytes,
                             void* stream);
/* Same solve with the residual post-check (tpf_residual_c128, below) fused
 * into the kernel's retire step: resid[j] is bit-identical to what
 * tpf_residual_c128 computes from this call's V, and no second pass over
 * S and V is made.  Y_dd is passed as level-ordered ELL rows built on the
 * host by tpf_sparse_tree_build_ell (width <= tpf_sparse_tree_max_ell_width()):
 *   ell_col int32[width*b], ell_val complex[width*b], entry r of level-ordered
 *   row m at [r*b + m], columns level-ordered, -1 = padding.              */
int tpf_sparse_tree_fpi_resid_c128(int64_t tau, int32_t b, int32_t levels,
                                   const int32_t* level_info, const int32_t* node_info, const double* node_coef,
                                   const double* S, int64_t s_node_stride, int64_t s_case_stride,
                                   double v_flat_re, double v_flat_im, double tol, int32_t max_iter,
                                   double* V, int64_t v_node_stride, int64_t v_case_stride,
                                   int32_t* iters, int32_t ell_width, const int32_t* ell_col,
                                   const double* ell_val, double* resid,
                                   void* workspace, size_t workspace_bytes, void* stream);
int tpf_sparse_tree_max_ell_width(void);
/* ZIP loads on radial feeders (the reference's per-case fpi_solve route,
 * dense.py:214-230 / fpi.py:107-206): per case the tree LU of
 * B = Y_dd + diag(alpha_z s*) (no fill, leaf-first), then
 *   B v' = -(alpha_p s* ./ conj(v) + src + alpha_i s*)
 * with fpi_solve's rules: one application when alpha_p s = 0 everywhere,
 * stop on a non-finite iterate, stop on the step test; the residual uses the
 * ZIP load power.  alpha = float64 planes [3][b] (z, i, p), ydiag = Y[m,m]
 * (complex[b]), both in level order; Y_dd must be exactly symmetric with
 * rows = diagonal + tree edges (ELL as above).  step_met[j] = 1 when case j
 * stopped on the step test (or was a one-application case); *status = 1
 * if some case's B had a zero pivot (SingularSystemError in the reference).
 * workspace >= tpf_sparse_tree_zip_workspace_bytes(tau, b).
 * All three ZIP entry points take v0: null = flat start v_flat for every
 * node (fpi.py:130-131), else b complex values in ORIGINAL node order, the
 * start of every case (opts.initial_voltage, fpi.py:141-145).            */
/* The same ZIP route for radial feeders the tree kernel does not take (deep,
 * wide or > 5,120 nodes): one thread per case, nodes in leaf-first order
 * (orig = original node of position k, parent = position of k's parent or
 * -1, e = Y[k, parent], ydiag, alpha [3][b], src all in that order); the
 * residual sums Y v over the tree edges.  workspace >=
 * tpf_sparse_zip_chain_workspace_bytes(tau, b) (64 B per node and case). */
size_t tpf_sparse_zip_chain_workspace_bytes(int64_t tau, int32_t b);
int tpf_sparse_zip_chain_c128(int64_t tau, int32_t b, const int32_t* orig, const int32_t* parent,
                              const double* e, const double* ydiag, const double* alpha, const double* src,
                              const double* S, int64_t s_node_stride, int64_t s_case_stride,
                              double v_flat_re, double v_flat_im, const double* v0, double tol, int32_t max_iter,
                              double* V, int64_t v_node_stride, int64_t v_case_stride, int32_t* iters,
                              double* resid, uint8_t* step_met, int32_t* status,
                              void* workspace, size_t workspace_bytes, void* stream);
/* ZIP loads on meshed (or non-symmetric) networks, the reference's per-case
 * SuperLU route (dense.py:214-230 -> fpi.py:107-206): one thread per case,
 * per-case LU of B = Y_dd + diag(alpha_z s*) on a fixed fill pattern without
 * pivoting.  Step k eliminates original node orig[k]; kinfo[k] = (m_k, off)
 * with idx[off..] = the m_k later positions, their L slots, U slots and the
 * m_k x m_k update targets; base = Y_dd at the nslot factor slots (slot k < b
 * the pivot of step k).  alpha [3][b] and src in elimination order; the
 * residual reads Y_dd in CSR (original order).  workspace >=
 * tpf_sparse_zip_lu_workspace_bytes(tau, b, nslot) (16 B per slot, node and
 * case).  *status = 1 on a zero pivot.                                   */
size_t tpf_sparse_zip_lu_workspace_bytes(int64_t tau, int32_t b, int32_t nslot);
int tpf_sparse_zip_lu_c128(int64_t tau, int32_t b, int32_t nslot, const int32_t* orig, const int32_t* kinfo,
                           const int32_t* idx, const double* base, const double* alpha, const double* src,
                           const int32_t* y_row_ptr, const int32_t* y_col, const double* y_val,
                           const double* S, int64_t s_node_stride, int64_t s_case_stride,
                           double v_flat_re, double v_flat_im, const double* v0, double tol, int32_t max_iter,
                           double* V, int64_t v_node_stride, int64_t v_case_stride, int32_t* iters,
                           double* resid, uint8_t* step_met, int32_t* status,
                           void* workspace, size_t workspace_bytes, void* stream);
/* ZIP loads on small meshed networks (b <= tpf_sparse_zip_dense_max_nodes(),
 * 64) with partial pivoting, as the reference's per-case splu (fpi.py:119):
 * one thread per case, dense LU of B = Y_dd + diag(alpha_z s*) with row
 * pivoting (largest |.| in the column), then fpi_solve's iteration and ZIP
 * residual as tpf_sparse_zip_lu_c128.  y_dense = Y_dd b x b row-major; alpha
 * [3][b], src, S, V, v0 in original node order; the residual reads Y_dd in
 * CSR.  workspace >= tpf_sparse_zip_dense_workspace_bytes(tau, b).
 * *status = 1 on a zero pivot (a singular B).                             */
int tpf_sparse_zip_dense_max_nodes(void);
size_t tpf_sparse_zip_dense_workspace_bytes(int64_t tau, int32_t b);
int tpf_sparse_zip_dense_c128(int64_t tau, int32_t b, const double* y_dense, const double* alpha, const double* src,
                              const int32_t* y_row_ptr, const int32_t* y_col, const double* y_val, const double* S,
                              int64_t s_node_stride, int64_t s_case_stride, double v_flat_re, double v_flat_im,
                              const double* v0, double tol, int32_t max_iter, double* V, int64_t v_node_stride,
                              int64_t v_case_stride, int32_t* iters, double* resid, uint8_t* step_met,
                              int32_t* status, void* workspace, size_t workspace_bytes, void* stream);
size_t tpf_sparse_tree_zip_workspace_bytes(int64_t tau, int32_t b);
int tpf_sparse_tree_zip_fpi_c128(int64_t tau, int32_t b, int32_t levels,
                                 const int32_t* level_info, const int32_t* node_info, const double* node_coef,
                                 const double* alpha, const double* ydiag,
                                 const double* S, int64_t s_node_stride, int64_t s_case_stride,
                                 double v_flat_re, double v_flat_im, const double* v0, double tol, int32_t max_iter,
                                 double* V, int64_t v_node_stride, int64_t v_case_stride, int32_t* iters,
                                 int32_t ell_width, const int32_t* ell_col, const double* ell_val,
                                 double* resid, uint8_t* step_met, int32_t* status,
                                 void* workspace, size_t workspace_bytes, void* stream);
/* Host helpers (no device work): widest CSR row of Y_dd (-1 on bad input),
 * and the ELL rows above from the ORIGINAL-order CSR and node_info.        */
int tpf_sparse_tree_ell_width(int32_t b, const int32_t* ydd_row_ptr);
int tpf_sparse_tree_build_ell(int32_t b, int32_t width, const int32_t* node_info,
                              const int32_t* ydd_row_ptr, const int32_t* ydd_col, const double* ydd_val,
                              int32_t* ell_col, double* ell_val);

/* ------------------------------------------------------- complex64 twins --
 * Same contracts as the c128 entry points above, in FP32 (complex64 arrays,
 * float scalars).  FP32 cannot resolve tol = 1e-10: use tol >= ~1e-6.
 *   tpf_dense_fpi_c64:  b <= tpf_dense_c64_max_nodes() (104); K, W complex64;
 *                       workspace >= tpf_dense_c64_workspace_bytes(tau, b).
 *   tpf_sparse_fpi_c64: L/U values, 1/U[k,k] and src complex64; workspace
 *                       >= tpf_sparse_c64_workspace_bytes(tau, b).
 *   tpf_residual_c64:   the post-check of a complex64 solution, in FP64
 *                       (Y_dd, src complex128; resid float64).            */
int tpf_dense_c64_max_nodes(void);
size_t tpf_dense_c64_workspace_bytes(int64_t tau, int32_t b);
int tpf_dense_fpi_c64(int64_t tau, int32_t b, const float* S, int64_t s_node_stride, int64_t s_case_stride,
                      const float* K, const float* W, float v_flat_re, float v_flat_im, float tol,
                      int32_t max_iter, float* V, int64_t v_node_stride, int64_t v_case_stride,
                      int32_t* iters, void* workspace, size_t workspace_bytes, void* stream);
size_t tpf_sparse_c64_workspace_bytes(int64_t tau, int32_t b);
int tpf_sparse_fpi_c64(int64_t tau, int32_t b, const float* S, int64_t s_node_stride, int64_t s_case_stride,
                       const int32_t* l_ptr, const int32_t* l_col, const float* l_val,
                       const int32_t* u_ptr, const int32_t* u_col, const float* u_val,
                       const float* u_diag_inv, const int32_t* perm, const float* src,
                       float v_flat_re, float v_flat_im, float tol, int32_t max_iter,
                       float* V, int64_t v_node_stride, int64_t v_case_stride, int32_t* iters,
                       void* workspace, size_t workspace_bytes, void* stream);
int tpf_residual_c64(int64_t tau, int32_t b, const float* S, int64_t s_node_stride, int64_t s_case_stride,
                     const float* V, int64_t v_node_stride, int64_t v_case_stride,
                     const int32_t* ydd_row_ptr, const int32_t* ydd_col, const double* ydd_val,
                     const double* src, double* resid, void* stream);

/* -------------------------------------------------------------- residual --
 * residual_per_case (fpi.py:221-240, constant-power branch) as used by
 * _safe_residuals (dense.py:208-211):
 *     resid[j] = max_i | s_ij + v_ij * conj(src_i + (Y_dd v_j)_i) |
 * Y_dd in CSR (int32 row_ptr[b+1], int32 col[nnz], complex val[nnz]).
 * NaN propagates as in numpy's max.                                        */
int tpf_residual_c128(int64_t tau, int32_t b,
                      const double* S, int64_t s_node_stride, int64_t s_case_stride,
                      const double* V, int64_t v_node_stride, int64_t v_case_stride,
                      const int32_t* ydd_row_ptr, const int32_t* ydd_col, const double* ydd_val,
                      const double* src, double* resid, void* stream);
/* The same with the rows visited in row_order (a permutation of 0..b-1, e.g.
 * a depth-first order of a radial feeder, so a row's neighbours are read
 * while still cached); the per-case maximum does not depend on the order. */
int tpf_residual_order_c128(int64_t tau, int32_t b,
                            const double* S, int64_t s_node_stride, int64_t s_case_stride,
                            const double* V, int64_t v_node_stride, int64_t v_case_stride,
                            const int32_t* ydd_row_ptr, const int32_t* ydd_col, const double* ydd_val,
                            const double* src, const int32_t* row_order, double* resid, void* stream);

/* --------------------------------------------------------------- summary --
 * converged mask (dense.py:198-199): mask[j] = isfinite(resid[j]) && resid[j] < residual_tol.
 * out[0] = max_j iters[j] (the reference's joint iteration count),
 * out[1] = number of converged cases.  out must be 2 int32 of device memory. */
int tpf_batch_summary(int64_t tau, const int32_t* iters, const double* resid,
                      double residual_tol, uint8_t* mask, int32_t* out, void* stream);

/* ------------------------------------------------------- host pipelines --
 * The whole batch_solve_dense / batch_solve_sparse call on HOST buffers
 * (the reference's LoadMatrix in, VoltageBatch arrays out): H2D of S, the
 * iteration, the residual post-check and the D2H of V run in tau-chunks on
 * three CUDA streams so PCIe transfers overlap the solve.  Host S and V must be
 * node-major (case stride 1, the reference layout) or case-major (node stride
 * 1); pageable buffers are page-locked for the duration of the call.
 * K, W, Y_dd CSR, src and the LU arrays are host arrays (as in the _c128
 * entry points).  iters/resid/mask may be NULL; summary (2 int32, host) gets
 * {max iterations, converged count}.  chunk_cases <= 0 picks a default.
 * workspace: device scratch of >= tpf_*_solve_host_workspace_bytes(...)
 * bytes, or NULL to let the call cudaMalloc/cudaFree its own.
 * Synchronous: returns when every output is on the host.                  */
/* ------------------------------------------------------------ file tables --
 * Host-only, multi-threaded (threads <= 0: all hardware threads).
 * Load table (reference fileio.py:196-234): header p_1,q_1,...,p_b,q_b, one
 * row per case, blank lines skipped.  tpf_loads_csv_scan validates the
 * header and counts the cases; tpf_loads_csv_read parses them (correctly
 * rounded) into values = complex128 b x tau node-major.  A malformed row gives
 * TPF_ERR_INVALID and *bad_line (1-based); a field whose float() reading
 * could differ from strtod (inf/nan words, hex, underscores, > 63 chars)
 * gives TPF_ERR_UNSUPPORTED.
 * tpf_write_pairs_csv: the header line, then per case j one row
 * x[0,j],y[0,j],...,x[b-1,j],y[b-1,j][,flag[j]] with "%.17g" cells ("nan"
 * for every NaN): the voltage table (x = |V|, y = angle V, flag = converged;
 * fileio.py:237-253) and the load table writer (fileio.py:184-193).       */
int tpf_loads_csv_scan(const char* path, int32_t* b, int64_t* tau);
int tpf_loads_csv_read(const char* path, int32_t b, int64_t tau, double* values, int64_t* bad_line,
                       int32_t threads);
int tpf_write_pairs_csv(const char* path, const char* header, int32_t b, int64_t tau, const double* x,
                        const double* y, int64_t node_stride, int64_t case_stride, const uint8_t* flag,
                        int32_t threads);

/* Page-lock a host range for the duration of several concurrent host-pipeline
 * calls (multi-device use): returns 1 if this call registered it (release with
 * tpf_host_unpin), 0 if it was already page-locked or cannot be.          */
int tpf_host_pin(void* ptr, size_t bytes);
int tpf_host_unpin(void* ptr);
/* Per-node statistics of a solved batch (probabilistic PF, config C4):
 * vmin/vmax/vsum[i] = min / max / sum over the tau cases of |V[i, j]|
 * (accumulate != 0: folded into the arrays' current values, e.g. over
 * scenario batches).  Deterministic (fixed reduction order, no atomics).
 * workspace >= tpf_voltage_stats_workspace_bytes(tau, b).                 */
size_t tpf_voltage_stats_workspace_bytes(int64_t tau, int32_t b);
int tpf_voltage_stats_c128(int64_t tau, int32_t b, const double* V, int64_t v_node_stride, int64_t v_case_stride,
                           double* vmin, double* vmax, double* vsum, int32_t accumulate, void* workspace,
                           size_t workspace_bytes, void* stream);
/* Host-buffer pipeline of the warp-per-subtree kernel (schedule arrays on the
 * HOST, uploaded once per call; same chunked H2D / solve + fused residual /
 * D2H streams as tpf_sparse_tree_solve_host_c128).                        */
size_t tpf_sparse_subtree_solve_host_workspace_bytes(int64_t tau, int32_t b, int32_t ns, int32_t nt, int32_t rw,
                                                     int32_t nkids, int64_t chunk_cases, int64_t ydd_nnz);
int tpf_sparse_subtree_solve_host_c128(int64_t tau, int32_t b, int32_t ns, int32_t nt, int32_t rmax, int32_t rw,
                                       int32_t nkids, const int32_t* pinfo, const int32_t* slotinfo,
                                       const uint16_t* kids, const double* coef, const int32_t* ell_col,
                                       const double* ell_val, const double* S, int64_t s_node_stride,
                                       int64_t s_case_stride, const int32_t* ydd_row_ptr, const int32_t* ydd_col,
                                       const double* ydd_val, const double* src, double v_flat_re, double v_flat_im,
                                       double tol, int32_t max_iter, double residual_tol, double* V,
                                       int64_t v_node_stride, int64_t v_case_stride, int32_t* iters, double* resid,
                                       uint8_t* mask, int32_t* summary, int64_t chunk_cases, int32_t device,
                                       void* workspace, size_t workspace_bytes);
size_t tpf_sparse_tree_solve_host_workspace_bytes(int64_t tau, int32_t b, int64_t chunk_cases, int64_t ydd_nnz);
int tpf_sparse_tree_solve_host_c128(int64_t tau, int32_t b, int32_t levels,
                                    const int32_t* level_info, const int32_t* node_info, const double* node_coef,
                                    const double* S, int64_t s_node_stride, int64_t s_case_stride,
                                    const int32_t* ydd_row_ptr, const int32_t* ydd_col, const double* ydd_val,
                                    const double* src, double v_flat_re, double v_flat_im,
                                    double tol, int32_t max_iter, double residual_tol,
                                    double* V, int64_t v_node_stride, int64_t v_case_stride,
                                    int32_t* iters, double* resid, uint8_t* mask, int32_t* summary,
                                    int64_t chunk_cases, int32_t device, void* workspace, size_t workspace_bytes);
size_t tpf_dense_solve_host_workspace_bytes(int64_t tau, int32_t b, int64_t chunk_cases, int64_t ydd_nnz);
size_t tpf_sparse_solve_host_workspace_bytes(int64_t tau, int32_t b, int64_t chunk_cases, int64_t ydd_nnz,
                                             int64_t l_nnz, int64_t u_nnz);
int tpf_dense_solve_host_c128(int64_t tau, int32_t b,
                              const double* S, int64_t s_node_stride, int64_t s_case_stride,
                              const double* K, const double* W,
                              const int32_t* ydd_row_ptr, const int32_t* ydd_col, const double* ydd_val,
                              const double* src, double v_flat_re, double v_flat_im,
                              double tol, int32_t max_iter, double residual_tol,
                              double* V, int64_t v_node_stride, int64_t v_case_stride,
                              int32_t* iters, double* resid, uint8_t* mask, int32_t* summary,
                              int64_t chunk_cases, int32_t device, void* workspace, size_t workspace_bytes);
int tpf_sparse_solve_host_c128(int64_t tau, int32_t b,
                               const double* S, int64_t s_node_stride, int64_t s_case_stride,
                               const int32_t* l_ptr, const int32_t* l_col, const double* l_val,
                               const int32_t* u_ptr, const int32_t* u_col, const double* u_val,
                               const double* u_diag_inv, const int32_t* perm,
                               const int32_t* ydd_row_ptr, const int32_t* ydd_col, const double* ydd_val,
                               const double* src, double v_flat_re, double v_flat_im,
                               double tol, int32_t max_iter, double residual_tol,
                               double* V, int64_t v_node_stride, int64_t v_case_stride,
                               int32_t* iters, double* resid, uint8_t* mask, int32_t* summary,
                               int64_t chunk_cases, int32_t device, void* workspace, size_t workspace_bytes);

/* ----------------------------------------------------------------- probe --
 * FP64 tensor-core peak of the current device, measured with a DMMA-only
 * kernel (used as the dense roofline denominator).  Synchronous.           */
int tpf_probe_fp64_tflops(double* tflops_out, double* ms_out);

#ifdef __cplusplus
}
#endif
#endif /* TPF_H_ */
