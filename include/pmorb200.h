/* libpmorb200 -- C ABI of the B200 (sm_100a) SPAI / SPAI-update / block-solve
 * path of "Preconditioned Linear Solves for Parametric Model Order Reduction"
 * (arXiv 1809.06574).
 *
 * The reference (`pmorprec`, pure Python over numpy/scipy) has no FFI layer:
 * its boundary for this path is the Python API.  Each entry point below is
 * the native replacement of one reference function (or of the numpy/scipy
 * call inside it) and cites it as file:line under /root/reference/pkg/src/
 * pmorprec.  The Python package paper_1809_06574_b200 binds them with ctypes
 * (see INTEGRATION.md for the binding a reference maintainer would add).
 *
 * Conventions
 *  - every pointer argument named d_* is DEVICE memory owned by the caller;
 *    h_* pointers are host memory read during the call;
 *  - indices are int32, values float64 (the reference's complex128 carries
 *    only zero imaginary parts on the real BASELINE inputs);
 *  - dense blocks are ROW-MAJOR n x k with a leading dimension (ld >= k);
 *  - every call is asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *    default stream) and never synchronises;
 *  - the library never allocates: scratch comes in via (d_ws, ws_bytes),
 *    sized by the matching *_workspace() query;
 *  - return codes: PMP_OK, PMP_ERR_ARG (-> ValueError), PMP_ERR_CUDA
 *    (-> RuntimeError with pmp_last_error()), PMP_ERR_WORKSPACE;
 *  - all reductions are fixed-order: repeated calls are bitwise identical.
 */
#ifndef PMORB200_H
#define PMORB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PMP_OK 0
#define PMP_ERR_ARG (-1)
#define PMP_ERR_CUDA (-2)
#define PMP_ERR_WORKSPACE (-3)

#define PMP_MAX_TERMS 16

const char* pmp_last_error(void);
int pmp_version(void);

/* ---- kernel 1: assembly ------------------------------------------------
 * Replaces SecondOrderModel.assemble (rpmor.py:92-107, _eval_terms :41-49)
 * when mode == 0, and AffineFamily.evaluate (affine.py:118-134) when
 * mode == 1, over a precomputed union pattern (affine.py:97-116).
 * Term t contributes h_coef[t] * value; h_first[t] == 1 marks the constant
 * term that opens its group (coefficient ignored).  Groups (h_group):
 * 0 = mass (scaled by s^2), 1 = damping (scaled by s), 2 = stiffness.
 * h_kind[t] == 0: d_term_vals[t] holds one value per union entry;
 * h_kind[t] == 1: it holds a length-nrows diagonal (needs d_rowid).
 * Per entry the arithmetic is the reference's exactly (no FMA), so the
 * result is bit-identical.  Exact zeros (mode 0) / |v| < 1e-300 (mode 1)
 * are written as 0.0 and counted into *d_zero_count (int, accumulated). */
int pmp_assemble(int nnz, int nterms, const double* const* h_term_vals, const int32_t* h_kind,
                 const int32_t* h_group, const int32_t* h_first, const double* h_coef, int mode,
                 double s, const int32_t* d_rowid, const int32_t* d_colidx, double* d_out,
                 const int32_t* d_perm, double* d_out_perm, int32_t* d_zero_count, void* stream);
/* Several systems of one recipe shape at once (a parameter sweep: the same
 * terms, groups and opening terms; system q's coefficients are
 * h_coef[q * nterms + t] and its shift h_s[q]).  Every term value is read
 * once for all systems; system q's result goes to h_out[q] (and, with
 * d_perm, permuted to h_out_perm[q]) -- HOST arrays of device pointers --
 * and its exact-zero count is added to d_zero_counts[q].  Bit-identical to
 * nsys pmp_assemble calls. */
int pmp_assemble_multi(int nnz, int nterms, const double* const* h_term_vals,
                       const int32_t* h_kind, const int32_t* h_group, const int32_t* h_first,
                       int nsys, const double* h_coef, const double* h_s, int mode,
                       const int32_t* d_rowid, const int32_t* d_colidx, double* const* h_out,
                       const int32_t* d_perm, double* const* h_out_perm,
                       int32_t* d_zero_counts, void* stream);

/* Drop entries whose value is exactly 0.0 (as_csr eliminate_zeros,
 * sparsecore.py:43).  Output arrays have capacity nnz; d_out_rowptr[n]
 * holds the new nnz. */
size_t pmp_compact_workspace(int n);
int pmp_compact_zeros(int n, const int32_t* d_rowptr, const int32_t* d_colidx,
                      const double* d_vals, int32_t* d_out_rowptr, int32_t* d_out_colidx,
                      double* d_out_vals, void* d_ws, size_t ws_bytes, void* stream);

/* ---- structure: CSR <-> CSC ---------------------------------------------
 * Transposed structure of an n x n CSR plus the permutation
 * d_perm[e_in] = e_out (A.tocsc() at spai.py:320; _assemble_and_stats COO
 * -> CSR at spai.py:307).  Rows of the output are sorted.  When drop_zeros
 * is set and d_vals is given, entries equal to 0.0 are skipped (their
 * d_perm is -1) and values are transposed into d_out_vals. */
size_t pmp_transpose_workspace(int n, int nnz);
int pmp_transpose(int n, int nnz, const int32_t* d_ptr, const int32_t* d_idx,
                  const double* d_vals, int drop_zeros, int32_t* d_out_ptr, int32_t* d_out_idx,
                  double* d_out_vals, int32_t* d_perm, void* d_ws, size_t ws_bytes,
                  void* stream);
/* d_dst[d_perm[e]] = d_src[e] for d_perm[e] >= 0 */
int pmp_permute(int nnz, const int32_t* d_perm, const double* d_src, double* d_dst, void* stream);
/* pmp_permute over k value arrays in one launch (the factors of a window of
 * SPAI updates sharing one pattern, spai.py:307 per factor):
 * d_dst[q*dst_stride + d_perm[e]] = d_src[q*src_stride + e], 0 <= q < k <= 65535 */
int pmp_permute_batch(int nnz, const int32_t* d_perm, int k, const double* d_src,
                      long long src_stride, double* d_dst, long long dst_stride, void* stream);

/* ---- kernel 2: SPAI pattern gather (spai_pattern level 0, spai.py:182-207)
 * I_j = rows(A(:, j)) U {j} for an n x n matrix in CSC. */
size_t pmp_pattern_l0_workspace(int n);
int pmp_pattern_l0(int n, const int32_t* d_colptr, const int32_t* d_rowidx, int32_t* d_iptr,
                   int32_t* d_iidx, void* d_ws, size_t ws_bytes, void* stream);
/* Size pass only: d_iptr[0..n] (exclusive scan of |I_j|); d_iptr[n] = total. */
int pmp_pattern_l0_ptr(int n, const int32_t* d_colptr, const int32_t* d_rowidx, int32_t* d_iptr,
                       void* d_ws, size_t ws_bytes, void* stream);

/* ---- kernels 3/4: batched column least squares (spai.py:229-292) --------
 * For each listed column j: J = unique(rows(T(:,j)) U rows(A(:,k)), k in I_j)
 * (spai.py:237-240); dense A(J, I_j) with the target scattered on J;
 * column-pivoted Householder QR; rank by |R_kk| > eps |R_00|; minimum-norm
 * complete-orthogonal solve when rank deficient (LAPACK gelsy semantics,
 * spai.py:250); explicit residual ||t - A(J,I) z||_2 (spai.py:252).
 * T == NULL (d_tcolptr NULL) means the identity target (SPAI build,
 * spai.py:362); otherwise T is the reference matrix (update, update.py:75).
 *
 * team: 32 (warp per column), 128 or 256 (CTA per column).  Team scratch is
 * sized from (lcap, mcap, ncap) = (pow2 bound on the gathered row list,
 * max |J|, max |I|) -- see pmp_ls_team_bytes.  use_global != 0 keeps the
 * team scratch in d_ws (for columns whose dense block exceeds shared
 * memory); otherwise it lives in shared memory.
 * mode 0: solve (writes d_coef at the I_j slots, d_resid[j], d_flags[j] bit 0
 *         = rank deficient);
 * mode 1: plan (writes |J_j| into d_msize[j] only);
 * mode 2: export J (writes J_j into d_jidx at d_jptr[j]; tests only). */
size_t pmp_ls_team_bytes(int team, int lcap, int mcap, int ncap);
int pmp_ls_bound(int ncols, const int32_t* d_cols, const int32_t* d_iptr, const int32_t* d_iidx,
                 const int32_t* d_acolptr, const int32_t* d_tcolptr, int32_t* d_lsize,
                 void* stream);
int pmp_ls_columns(int mode, int team, int use_global, int lcap, int mcap, int ncap, int ncols,
                   const int32_t* d_cols, int n, const int32_t* d_iptr, const int32_t* d_iidx,
                   const int32_t* d_acolptr, const int32_t* d_arowidx, const double* d_avals,
                   const int32_t* d_tcolptr, const int32_t* d_trowidx, const double* d_tvals,
                   double* d_coef, double* d_resid, int32_t* d_flags, int32_t* d_msize,
                   const int32_t* d_jptr, int32_t* d_jidx, void* d_ws, size_t ws_bytes,
                   void* stream);

/* Same least squares with the per-column symbolic work (the sorted J, the
 * positions of every A(J, I) entry and target entry) recorded once and
 * replayed: every system of a parameter sweep shares one CSR structure, so
 * only the values change between updates.  mode 4 solves and records into
 * d_plan at d_plan_ptr[c] (c = position in the column list; size of column
 * c: 4 + |I_j| + 2 * (pmp_ls_bound's list length)); mode 5 solves from the
 * record (A / T values may differ, structures must be the recorded ones).
 * Results are bitwise those of mode 0. */
int pmp_ls_columns_planned(int mode, int team, int use_global, int lcap, int mcap, int ncap,
                           int ncols, const int32_t* d_cols, int n, const int32_t* d_iptr,
                           const int32_t* d_iidx, const int32_t* d_acolptr,
                           const int32_t* d_arowidx, const double* d_avals,
                           const int32_t* d_tcolptr, const int32_t* d_trowidx,
                           const double* d_tvals, double* d_coef, double* d_resid,
                           int32_t* d_flags, int32_t* d_plan, const int32_t* d_plan_ptr,
                           void* d_ws, size_t ws_bytes, void* stream);

/* Several systems that share the plan's structures (the SPAI updates of a
 * parameter sweep: same pattern, same A_l structure, same target A1):
 * system q's values are h_avals[q], its outputs h_coef[q] / h_resid[q] /
 * h_flags[q] -- HOST arrays of nsys DEVICE pointers.  mode 4 records the
 * plan on system 0 and replays it for the others, mode 5 replays for all.
 * Small columns (the segmented register tier: |J| <= 32, |I| <= 15) are
 * solved for up to PMP_LS_MAX_SYSTEMS systems per launch; other tiers one
 * launch per system.  Results are bitwise those of pmp_ls_columns_planned
 * per system. */
#define PMP_LS_MAX_SYSTEMS 64
int pmp_ls_columns_multi(int mode, int team, int use_global, int lcap, int mcap, int ncap,
                         int ncols, const int32_t* d_cols, int n, const int32_t* d_iptr,
                         const int32_t* d_iidx, const int32_t* d_acolptr,
                         const int32_t* d_arowidx, int nsys, const double* const* h_avals,
                         const int32_t* d_tcolptr, const int32_t* d_trowidx,
                         const double* d_tvals, double* const* h_coef, double* const* h_resid,
                         int32_t* const* h_flags, int32_t* d_plan, const int32_t* d_plan_ptr,
                         void* d_ws, size_t ws_bytes, void* stream);

/* ---- level-1 augmentation (_augmented_column, spai.py:210-222) ----------
 * Weights w_r = sum over k ascending of |a_rk| |a_kj| (no FMA; scipy's
 * csc_matmat order); candidates outside the base support
 * ranked by (w desc, row asc), top max(max_fill - |base|, 0) kept, union
 * with base.  For each listed column j = d_cols[c], mode 0 writes the new
 * support size to d_newsize[j]; mode 1 writes the support at d_newptr[j]
 * into d_newidx. */
size_t pmp_augment_team_bytes(int lcap);
int pmp_augment(int mode, int lcap, int use_global, int ncols, const int32_t* d_cols,
                int max_fill, const int32_t* d_iptr, const int32_t* d_iidx,
                const int32_t* d_acolptr, const int32_t* d_arowidx, const double* d_avals,
                int32_t* d_newsize, const int32_t* d_newptr, int32_t* d_newidx, void* d_ws,
                size_t ws_bytes, void* stream);

/* ---- kernel 5a: CSR SpMM (Preconditioner.apply spai.py:82-89; op and true
 * residual krylov.py:140-147, :231) -----------------------------------------
 * Y = alpha * A X + beta * Y0 over s <= 32 columns.  Y0 may alias Y; beta
 * == 0 ignores Y0. */
int pmp_spmm(int n, const int32_t* d_rowptr, const int32_t* d_colidx, const double* d_vals,
             int s, const double* d_x, int ldx, double alpha, double beta, const double* d_y0,
             int ldy0, double* d_y, int ldy, void* stream);

/* ---- kernel 5b: block orthogonalisation (krylov.py:160-161, :189-196) ---
 * G = V^T W (kv x nw, row-major, device), fixed-order two-level reduction. */
size_t pmp_gram_workspace(int n, int kv, int nw);
int pmp_gram(int n, int kv, const double* d_v, int ldv, int nw, const double* d_w, int ldw,
             double* d_g, void* d_ws, size_t ws_bytes, void* stream);
/* Out = beta * Out + alpha * V H, H kv x nc row-major on the device
 * (W - V H, dXt = V Y, images = V G Y: krylov.py:195, :221-223, :246). */
int pmp_tsmm(int n, int kv, const double* d_v, int ldv, int nc, const double* d_h, double alpha,
             double beta, double* d_out, int ldo, void* stream);

/* ---- kernel 5c: TSQR, R factor only (the geqp3 inside _qr_deflate,
 * krylov.py:79-95).  Householder QR per row chunk + in-order reduction of
 * the chunk R factors; writes the nz x nz upper-triangular R (row-major). */
size_t pmp_tsqr_workspace(int n, int nz);
int pmp_tsqr_r(int n, int nz, const double* d_z, int ldz, double* d_r, void* d_ws,
               size_t ws_bytes, void* stream);

/* ---- kernel 5b+5c fused: one block-Arnoldi orthogonalisation step -------
 * (krylov.py:189-202) in one cooperative launch:
 *   W -= C (C^T W)  [k > 0];  npass x { H = V^T W; W -= V H }  (npass 0 or 2)
 *   W = Q R by Cholesky-QR2 with symmetric pivoting; Q written to
 *   V[:, qout : qout + sb].
 * Outputs (device): outB = C^T W (k x sb), outH1 / outH2 = the two CGS
 * coefficient blocks (total x sb), outR (sb x sb, row-major, un-pivoted),
 * *outFlag = 0.  When the pivoted Cholesky finds min|R_kk|/|R_00| <= 1e-5
 * (too close to the 1e-12 deflation threshold for Cholesky to decide),
 * *outFlag = 1, V is untouched and W holds the projected block for the
 * Householder fallback (pmp_tsqr_r + pmp_host_deflate).  sb <= 16. */
size_t pmp_orth_workspace(int n, int total_max, int k_max, int sb);
int pmp_orth_step(int n, const double* d_C, int ldc, int k, double* d_V, int ldv, int total,
                  int npass, double* d_W, int ldw, int sb, int qout, double* d_outB,
                  double* d_outH1, double* d_outH2, double* d_outR, double* d_outFlag,
                  void* d_ws, size_t ws_bytes, void* stream);

/* ---- outer-space fold (krylov.py:244-269), one cooperative launch --------
 * For col = 0..na-1: w = img[:, col], z = dz[:, col]; two passes of
 * { h = C^T w; w -= C h; z -= U h } against the current C (k columns);
 * drop when ||w|| <= 1e-10 ||img[:, col]|| (or ||img[:, col]|| == 0), else
 * append C[:, k] = w / ||w||, U[:, k] = z / ||w||, k++.  Writes out[0] =
 * final k and out[1 + col] = 1 / 0 (kept).  C, U: n x ldc row-major with
 * k0 + na <= kc <= ldc. */
size_t pmp_fold_workspace(int n, int kc);
int pmp_fold(int n, int na, const double* d_img, int ldi, const double* d_dz, int ldz,
             double* d_C, double* d_U, int ldc, int kc, int k0, double* d_out, void* d_ws,
             size_t ws_bytes, void* stream);

/* ---- native block-step driver (krylov.py:184-216) ------------------------
 * Pinned, device-mapped host memory for zero-copy step results. */
int pmp_host_alloc_mapped(size_t bytes, void** h_ptr);
int pmp_host_free_mapped(void* h_ptr);
int pmp_host_device_ptr(void* h_ptr, void** d_ptr);
/* Spin until *h_flag != sentinel (written last by the step kernel); after
 * timeout_us, synchronise the stream instead. */
int pmp_host_wait_flag(const double* h_flag, double sentinel, long long timeout_us, void* stream);
/* Enqueue one block step: W = A F_0 ... F_{nfac-1} V[:, q0:q0+sb] (host
 * arrays of the factors' device CSR pointers, outermost first), then
 * pmp_orth_step with its small outputs at d_small + off* (device), mirrored
 * at the end of the kernel to the same offsets of h_mirror (mapped host
 * memory, flag written last); h_mirror[offFlag] is set to -1 first.
 * ev_begin / ev_end (cudaEvent_t, may be NULL) bracket the orthogonalisation
 * kernel alone, for per-kernel timing. */
int pmp_gcro_step(int n, int s, int nfac, const int32_t* const* h_fac_rowptr,
                  const int32_t* const* h_fac_colidx, const double* const* h_fac_vals,
                  const int32_t* d_a_rowptr, const int32_t* d_a_colidx, const double* d_a_vals,
                  double* d_V, int cap, int q0, int sb, double* d_W, double* d_T0, double* d_T1,
                  double* d_T2, const double* d_C, int kc, int k, int total, double* d_small,
                  double* h_mirror, int offB, int offH1, int offH2, int offR, int offFlag,
                  void* d_ws, size_t ws_bytes, void* stream, void* ev_begin, void* ev_end);
/* End of a GCRO cycle (krylov.py:221-234), enqueued natively:
 *   dX = V[:, :m] Yv + U[:, :k] Yu ; Xt[:, act] += dX ; Xa = P Xt[:, act] ;
 *   X[:, act] = Xa ; Rb = B[:, act] - A Xa ; R[:, act] = Rb ; nrm = Rb^T Rb. */
int pmp_gcro_cycle_end(int n, int s, int na, const int32_t* d_act, const double* d_V, int cap,
                       int m, const double* d_Yv, const double* d_U, int kc, int k,
                       const double* d_Yu, double* d_dX, double* d_Xt, double* d_Z,
                       double* d_Xa, double* d_X, const double* d_B, double* d_Rb, double* d_R,
                       int nfac, const int32_t* const* h_fac_rowptr,
                       const int32_t* const* h_fac_colidx, const double* const* h_fac_vals,
                       const int32_t* d_a_rowptr, const int32_t* d_a_colidx,
                       const double* d_a_vals, double* d_T0, double* d_T1, double* d_nrm,
                       void* d_gram_ws, size_t gram_ws_bytes, void* stream);
/* State of the native inner loop of one GCRO cycle (pmp_gcro_inner).  The
 * caller owns every buffer; the loop runs full-rank block steps
 * (pmp_gcro_step + wait + pmp_gcro_absorb, with the next step launched
 * speculatively) until
 *   status 0: all estimates <= tol (cycle converged)
 *   status 2: m >= inner_restart      status 3: iterations >= max_iters
 *   status 4: G rank deficient after an absorb (caller: min-norm solve)
 *   status 5: the pending step needs the Householder deflation fallback
 * Estimates of each completed step are written row by row to hist. */
typedef struct PmpGcroInner {
  int n, s, na, k, cap, kc, ldq;
  double tol;
  int max_iters, inner_restart;
  int nfac;
  const int32_t* const* fac_rowptr;
  const int32_t* const* fac_colidx;
  const double* const* fac_vals;
  const int32_t* a_rowptr;
  const int32_t* a_colidx;
  const double* a_vals;
  double *V, *W, *T0, *T1, *T2;
  const double* C;
  double* d_small;
  double* mirror[2];
  int offB, offH1, offH2, offR, offFlag;
  void* orth_ws;
  size_t orth_ws_bytes;
  void* stream;
  double *Bmat, *Hb, *QR, *tau;
  int* ext;
  double *Cq, *Y, *res, *colsbuf;
  const double* bn;
  double* hist;
  int m, total, ncols, iterations, launched, buf;
  double prev_max;
  int matvecs, precond_applies, status, steps_done;
} PmpGcroInner;
int pmp_gcro_inner(PmpGcroInner* state);
/* Fold a finished full-rank step into Bmat / Hb (krylov.py:190-200) and the
 * incremental QR of G (pmp_host_hls_append). */
int pmp_gcro_absorb(const double* h_small, int offB, int offH1, int offH2, int offR, int cap,
                    int k, int q0, int sb, int total, double* h_Bmat, double* h_Hb, int ldq,
                    int nrhs, int ncols_old, double* h_QR, double* h_tau, int* h_ext,
                    double* h_C, double* h_Y, double* h_resnorm, double* h_colsbuf);

/* Device-resident inner loop of one GCRO cycle (krylov.py:184-216): ONE
 * persistent cooperative kernel runs every block step of the cycle -- the
 * operator chain W = A F_0 .. F_{nfac-1} V[:, q0:q0+sb], the fused
 * projection + CGS2 + Cholesky-QR2, and the incremental Householder QR of
 * the projected least-squares problem with the stopping test -- with grid
 * barriers instead of host round trips.  Block 0 is the control block (it
 * owns no rows; it keeps the projected QR in shared memory).
 * The projected state lives in d_proj (doubles, offsets o*; Bmat k x cap
 * and Hb cap x cap row-major, QR ldq x ldq and Cq ldq x na column-major,
 * Y na x n1 rhs-major, hist one row of na estimates per completed step) and
 * d_istate (int32: [0] m, [1] total, [2] ncols, [3] iterations, [4] status,
 * [5] history rows written, [6] scratch; ext[] of the QR at [16..16+ldq)).
 * On entry d_istate[0..3] and Cq / bn must be set (ncols == 0: the kernel
 * zeroes Bmat / Hb).  Exit status as pmp_gcro_inner: 0 converged,
 * 2 restart length, 3 max_iters, 4 G rank deficient (state after the
 * absorb), 5 the pending step needs the Householder deflation (W holds W2,
 * its B / H1 / H2 are copied to `mirror` at offB / offH1 / offH2). */
typedef struct PmpGcroCycle {
  int n, s, cap, kc, ldq, nfac;
  const int32_t* const* fac_rowptr;
  const int32_t* const* fac_colidx;
  const double* const* fac_vals;
  const int32_t* a_rowptr;
  const int32_t* a_colidx;
  const double* a_vals;
  double *V, *W, *T0, *T1;
  const double* C;
  double* d_small;
  double* mirror;
  int offB, offH1, offH2, offR;
  void* ws;
  size_t ws_bytes;
  void* stream;
  int k, na, sb, max_iters, inner_restart, hist_cap;
  double tol;
  double* d_proj;
  int oBmat, oHb, oQR, oTau, oCq, oY, oRes, oBn, oHist, blocks_per_sm;
  int32_t* d_istate;
} PmpGcroCycle;
size_t pmp_cycle_workspace(int n, int cap, int kc, int s);
int pmp_gcro_cycle_dev(PmpGcroCycle* cycle);
/* Diagnostics only: the next `records` cycle kernels write %globaltimer
 * stamps of blocks 0 and 1 into d_stamps[4096 * launch + (32 * step + phase)
 * * 2 + block] (device memory, zero-initialised by the caller). */
int pmp_cycle_debug_stamps(unsigned long long* d_stamps, int records);

/* Whole block-GCRO solves on the device (krylov.py:105-275), `groups`
 * independent systems per launch (one group of gsz blocks each; query
 * pmp_solve_geometry).  One PmpSysDesc per system, in DEVICE memory at
 * d_sys: the factor chain (nfac <= 3 CSR factors, applied right to left), A, the
 * right-hand side block B (n x s) and the output X (n x s).  Each system
 * gets wsz doubles of d_ws and isz ints of d_istate (offsets below, in
 * doubles, inside one system's block; p* offsets inside its projected-
 * state block at oProj).  Per system the int state reports: [144] active
 * columns left (0 = converged), [146] iterations, [147] status (0 ok,
 * 10 = needs the host path: deflation, rank-deficient projected problem or
 * an ambiguous drop test), [148] rows of the residual log (s doubles per
 * row at oLog), [149] matvecs, [150] preconditioner applications. */
typedef struct PmpSysDesc {
  int nfac;
  const int32_t* fac_rowptr[3];
  const int32_t* fac_colidx[3];
  const double* fac_vals[3];
  const int32_t* a_rowptr;
  const int32_t* a_colidx;
  const double* a_vals;
  const double* B;
  double* X;
} PmpSysDesc;
typedef struct PmpSolveBatch {
  int n, s, cap, kc, outer_dim, inner_restart, max_iters;
  int groups, gsz, rows_per_block, hist_cap, log_cap, isz;
  double tol;
  const PmpSysDesc* d_sys;
  double* d_ws;
  size_t wsz;
  int32_t* d_istate;
  size_t oV, oC, oU, oW, oT0, oT1, oQ1, oXt, oR, oDX, oRB, oZ, oPart, oGout, oSbuf, oProj, oLog,
      oAux;
  int pBmat, pHb, pCq, pY, pRes, pBn, pHist;
  /* pCtl: pmp_solve_ctl_doubles(s, kc, cap, inner_restart) doubles inside the
   * projected-state block for the control block's state when the geometry
   * keeps it in global memory (rows beyond shared memory: c4 / c5). */
  int pCtl;
  /* queue of systems: d_sys holds nsys descriptors; `groups` block groups
   * solve them, each taking the next unsolved system when it finishes one
   * (d_queue: one int32 of scratch, reset by the call).  Per system i:
   * d_result[8 i + 0..6] = status (0 ok, 10 host fallback), fallback reason,
   * iterations, columns still active (0 = converged), residual-log rows,
   * matvec count, preconditioner-apply count; d_result_log[i (2 + log_cap s)]
   * = algorithmic HBM bytes of its block steps -- [0] every operand once
   * per step, [1] SURVEY.md 8(d)'s unit (the operator chain + 32 n total +
   * 48 n s_b + 16 n k per step: block CGS2 reads [C | V] four times) --
   * then the residual log (log rows x s, row-major). */
  int nsys;
  int32_t* d_queue;
  int32_t* d_result;
  double* d_result_log;
  void* stream;
} PmpSolveBatch;
int pmp_solve_geometry(int n, int s, int cap, int kc, int inner_restart, int groups, int* gsz,
                       int* rows_per_block, int* cached, size_t* smem_bytes);
size_t pmp_solve_ctl_doubles(int s, int kc, int cap, int inner_restart);
int pmp_solve_batch(PmpSolveBatch* batch);

/* Route every cooperative launch (pmp_orth_step, pmp_fold, pmp_gcro_step's
 * orthogonalisation) through one shared stream, with event handoffs to and
 * from the caller's stream, so concurrent workers never run two grid-barrier
 * kernels at once.  NULL restores launching on the caller's stream. */
int pmp_set_coop_stream(void* stream);

/* Diagnostics only: block 0 of each of the next `records` orthogonalisation
 * kernels writes the device %globaltimer (ns) at its 11 phase boundaries
 * into d_stamps[16 * launch + 0..10] (device memory, zero-initialised by
 * the caller; unreached phases stay 0).  NULL (the default) disables it. */
int pmp_orth_debug_stamps(unsigned long long* d_stamps, int records);
/* Micro-benchmark: `iters` cooperative grid barriers over blocks_per_sm x
 * #SMs CTAs (diagnostic; time with events around the call). */
int pmp_bench_grid_sync(int blocks_per_sm, int iters, void* stream);

/* ---- helpers ------------------------------------------------------------ */
/* dst[:, dst_cols[c]] = src[:, src_cols[c]] for c < nc (NULL = identity). */
int pmp_copy_cols(int n, int nc, const double* d_src, int lds, const int32_t* d_src_cols,
                  double* d_dst, int ldd, const int32_t* d_dst_cols, void* stream);
/* dst[:, dst_cols[c]] = beta * dst[:, dst_cols[c]] + alpha * src[:, src_cols[c]]
 * (beta == 0 ignores dst). */
int pmp_axpby_cols(int n, int nc, double alpha, const double* d_src, int lds,
                   const int32_t* d_src_cols, double beta, double* d_dst, int ldd,
                   const int32_t* d_dst_cols, void* stream);
/* *d_count += #{j < n : d_flags[j] & mask}; *d_count must be zeroed. */
int pmp_count_flags(int n, const int32_t* d_flags, int mask, int32_t* d_count, void* stream);
/* d_out[c] = #{j in list: d_resid[d_cols? d_cols[c]: c] > ep}; compaction
 * of the columns whose residual exceeds ep (spai.py:287) into d_out_cols,
 * count into *d_count (zeroed by caller); order preserved. */
size_t pmp_select_workspace(int ncols);
int pmp_select_gt(int ncols, const int32_t* d_cols, const double* d_resid, double ep,
                  int32_t* d_out_cols, int32_t* d_count, void* d_ws, size_t ws_bytes,
                  void* stream);
/* exclusive scan of n int32 counts into n+1 outputs (d_out[n] = total) */
size_t pmp_scan_workspace(int n);
int pmp_scan(int n, const int32_t* d_in, int32_t* d_out, void* d_ws, size_t ws_bytes,
             void* stream);
/* Final SPAI/update column layout after the level-1 pass (spai.py:287-291):
 * column j keeps its augmented support and coefficients when the augmented
 * pattern has a non-empty column j, its base ones otherwise. */
int pmp_merge_sizes(int n, const int32_t* d_base_ptr, const int32_t* d_aug_ptr, int32_t* d_size,
                    void* stream);
int pmp_merge_columns(int n, const int32_t* d_base_ptr, const int32_t* d_base_idx,
                      const double* d_base_coef, const int32_t* d_aug_ptr,
                      const int32_t* d_aug_idx, const double* d_aug_coef,
                      const int32_t* d_out_ptr, int32_t* d_out_idx, double* d_out_coef,
                      void* stream);

/* ---- host-side small dense algebra of block GCRO (no device) -----------
 * Rank-revealing QR of the mz x mz TSQR factor rt (row-major, upper): LAPACK
 * geqp3 semantics with exact column norms; rank = #{|R_kk| > tol |R_00|}
 * (krylov.py:89-95).  Writes T (mz x rank, row-major) = Pi R11^-1, so the
 * orthonormal block is Z T, and Rout (rank x mz rows of an mz x mz
 * row-major buffer) = R[:rank] un-pivoted; *cond = |R_00| / |R_{r-1,r-1}|. */
int pmp_host_deflate(int mz, const double* h_rt, double tol, int* h_rank, double* h_T,
                     double* h_Rout, double* h_cond);
/* Incremental Householder QR least squares for min ||rhs - G Y||
 * (krylov.py:204-212): appends nnew columns (nrows x nnew, column-major) to
 * the factorisation held in h_QR (ldq x ldq column-major), h_tau, h_ext,
 * applies the new reflectors to h_C (ldq x nrhs, column-major, = Q^T rhs),
 * and writes Y ((ncols_old + nnew) x nrhs, column-major) and the residual
 * norms.  Returns 1 when R is (near) rank deficient (caller falls back to
 * a minimum-norm solve). */
int pmp_host_hls_append(int ldq, int nrhs, int ncols_old, int nnew, int nrows,
                        const double* h_newcols, double* h_QR, double* h_tau, int* h_ext,
                        double* h_C, double* h_Y, double* h_resnorm);

/* ---- measurement --------------------------------------------------------- */
/* Live FP64 pipe peak of this device (kind 0: DFMA, 8 independent fma
 * chains per thread; kind 1: DMMA, mma.sync m8n8k4 f64): 4 x #SMs blocks of
 * 256 threads, `iters` x 128 (DFMA) / 32 (DMMA) instructions per thread,
 * timed with CUDA events on `stream` after one warm-up launch (this call
 * synchronises).  *tflops = achieved TFLOP/s.  The denominator of the
 * least-squares roofline (bench.py roofline_ls). */
int pmp_fp64_peak(int kind, int iters, double* tflops, void* stream);

/* ---- complex128 through the real form ---------------------------------------
 * The reference computes in complex128 (sparsecore.py:8-10).  Complex
 * matrices run on the real kernels as R(A) (2n x 2n, entry (r, c) -> block
 * [[Re, -Im], [Im, Re]], every block stored in full, every row holding its
 * diagonal block); complex vectors as R(x) = (re_0, im_0, re_1, im_1, ...).
 * Complex least squares over a support I is exactly real least squares over
 * R(A)'s columns {2k, 2k+1 : k in I}; the complex block Krylov space of B is
 * the real one of [R(b_0), R(i b_0), R(b_1), ...] (see csrc/cplx.cu). */
/* Real form of an n x n complex CSR (rows sorted, diagonal present): writes
 * d_rowptr2[2n+1], d_colidx2[4 nnz] (may be NULL: values only), d_vals2[4 nnz].
 * d_im may be NULL (zero imaginary part). */
int pmp_realify(int n, const int32_t* d_rowptr, const int32_t* d_colidx, const double* d_re,
                const double* d_im, int32_t* d_rowptr2, int32_t* d_colidx2, double* d_vals2,
                void* stream);
/* n x s complex block (row-major re / im, ld ldx) -> 2n x 2s real block
 * (ld ldy >= 2s): column 2c = R(x_c), column 2c+1 = R(i x_c). */
int pmp_realify_block(int n, int s, const double* d_re, const double* d_im, int ldx, double* d_y,
                      int ldy, void* stream);
/* inverse: x_c = column stride*c of the 2n-row real block. */
int pmp_derealify_block(int n, int s, const double* d_y, int ldy, int stride, double* d_re,
                        double* d_im, int ldx, void* stream);
/* d_out[e] = |re[e] + i im[e]| (level-1 weights use |A|, spai.py:212). */
int pmp_modulus(int nnz, const double* d_re, const double* d_im, double* d_out, void* stream);
/* complex supports (iptr[n+1], iidx) -> real-form supports of columns 2j and
 * 2j+1: {2k, 2k+1 : k in I_j} (optr[2n+1], oidx[4 nnz]). */
int pmp_pattern_realify(int n, const int32_t* d_iptr, const int32_t* d_iidx, int32_t* d_optr,
                        int32_t* d_oidx, void* stream);

/* Complex assembly (rpmor.py:92-107 mode 0 / affine.py:118-134 mode 1) over
 * a union pattern: as pmp_assemble, with complex coefficients (h_cr + i h_ci),
 * complex shift s and s^2 (computed by the caller as the reference does,
 * Python complex s * s), term values h_re[t] (+ i h_im[t]; h_im or an entry
 * NULL: real term).  Writes the complex result (d_re, d_im) per union
 * entry, counts exact 0 + 0i entries; mode 1 prunes |v| < 1e-300. */
int pmp_assemble_cplx(int nnz, int nterms, const double* const* h_re, const double* const* h_im,
                      const int32_t* h_kind, const int32_t* h_group, const int32_t* h_first,
                      const double* h_cr, const double* h_ci, int mode, double sr, double si,
                      double s2r, double s2i, const int32_t* d_rowid, const int32_t* d_colidx,
                      double* d_re, double* d_im, int32_t* d_zero_count, void* stream);

/* ---- multi-GPU collectives (NCCL over NVLink / NVSwitch) ------------------
 * The sequence driver's two exchanges: replicate the base
 * SPAI P1 (rpmor.py:205-210: every first-approach system depends only on
 * (A1, P1)) and gather the per-system scalars.  libnccl.so.2 is opened at run
 * time (no link dependency); pmp_nccl_available() reports whether it loads.
 * The 128-byte unique id from rank 0 reaches the other ranks out of band
 * (the Python driver sends it through the torch.distributed store). */
int pmp_nccl_available(void);
int pmp_nccl_unique_id(unsigned char* h_out128);
int pmp_nccl_init(int rank, int world, const unsigned char* h_id128, void** comm);
int pmp_nccl_destroy(void* comm);
/* d_buf[0, bytes) from `root` to every rank (P1's CSR arrays). */
int pmp_nccl_bcast(void* d_buf, size_t bytes, int root, void* comm, void* stream);
/* In-place variable all-gather: rank r's bytes [h_displs[r], h_displs[r] +
 * h_counts[r]) of d_buf are replicated on every rank (one grouped broadcast
 * per rank; the column-sharded base build, spai.py:328-336). */
int pmp_nccl_allgatherv(void* d_buf, const size_t* h_counts, const size_t* h_displs, int world,
                        void* comm, void* stream);
/* Element-wise sum over ranks of `count` doubles, in place (per-system
 * scalar records, each system owned by exactly one rank). */
int pmp_nccl_allreduce_f64(double* d_buf, size_t count, void* comm, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PMORB200_H */
