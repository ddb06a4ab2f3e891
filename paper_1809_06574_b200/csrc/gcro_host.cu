// Native per-step driver of block GCRO (krylov.py:184-216).
//
// At BASELINE sizes a block step is ~50 us of device work, so the host side
// of a step -- launching the operator and the orthogonalisation, waiting for
// the small results, and folding them into the projected least-squares
// problem -- must cost about as much or less.  Through Python + numpy it
// cost ~150 us.  These entry points keep the reference's control flow in
// the Python caller but make each step two native calls:
//   pmp_gcro_step   : enqueue W = A P V[:, q0:q0+sb] (chain of SpMMs) and the
//                     fused orthogonalisation (pmp_orth_step) whose small
//                     outputs land directly in mapped (zero-copy) host memory;
//   pmp_gcro_absorb : spin on the step's flag in that memory, then update
//                     Bmat / Hb (krylov.py:190-202) and append the new block
//                     columns to the incremental QR of G (pmp_host_hls_append).
#include <atomic>
#include <chrono>

#include "common.cuh"

extern "C" {

int pmp_host_alloc_mapped(size_t bytes, void** host) {
  void* p = nullptr;
  cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess) {
    pmp::set_error("pmp_host_alloc_mapped: %s", cudaGetErrorString(e));
    return PMP_ERR_CUDA;
  }
  *host = p;
  return PMP_OK;
}

int pmp_host_free_mapped(void* host) {
  cudaError_t e = cudaFreeHost(host);
  if (e != cudaSuccess) {
    pmp::set_error("pmp_host_free_mapped: %s", cudaGetErrorString(e));
    return PMP_ERR_CUDA;
  }
  return PMP_OK;
}

// device-side address of mapped host memory (identical under UVA)
int pmp_host_device_ptr(void* host, void** dev) {
  cudaError_t e = cudaHostGetDevicePointer(dev, host, 0);
  if (e != cudaSuccess) {
    pmp::set_error("pmp_host_device_ptr: %s", cudaGetErrorString(e));
    return PMP_ERR_CUDA;
  }
  return PMP_OK;
}

// Spin until *flag != sentinel (the kernel writes it last, after a
// system-scope fence).  After `timeout_us` fall back to synchronising the
// stream; returns PMP_OK when the flag arrived, PMP_ERR_CUDA otherwise.
int pmp_host_wait_flag(const double* flag, double sentinel, long long timeout_us, void* stream) {
  const volatile double* f = flag;
  auto t0 = std::chrono::steady_clock::now();
  unsigned spins = 0;
  while (*f == sentinel) {
    if ((++spins & 1023u) == 0) {
      auto us = std::chrono::duration_cast<std::chrono::microseconds>(
                    std::chrono::steady_clock::now() - t0)
                    .count();
      if (us > timeout_us) {
        cudaError_t e = cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) {
          pmp::set_error("pmp_host_wait_flag: %s", cudaGetErrorString(e));
          return PMP_ERR_CUDA;
        }
        if (*f == sentinel) {
          pmp::set_error("pmp_host_wait_flag: stream finished without writing the flag");
          return PMP_ERR_CUDA;
        }
        break;
      }
    }
  }
  // the flag is written last: order every later read of the mirror after
  // the flag observation (weakly ordered hosts, compiler reordering)
  std::atomic_thread_fence(std::memory_order_acquire);
  return PMP_OK;
}

int pmp_spmm(int n, const int32_t* rowptr, const int32_t* colidx, const double* vals, int s,
             const double* X, int ldx, double alpha, double beta, const double* Y0, int ldy0,
             double* Y, int ldy, void* st);

int pmp_gcro_step(int n, int s, int nfac, const int32_t* const* fac_rowptr,
                  const int32_t* const* fac_colidx, const double* const* fac_vals,
                  const int32_t* a_rowptr, const int32_t* a_colidx, const double* a_vals,
                  double* V, int cap, int q0, int sb, double* W, double* T0, double* T1,
                  double* T2, const double* C, int kc, int k, int total, double* d_small,
                  double* mirror, int offB, int offH1, int offH2, int offR, int offFlag,
                  void* ws, size_t ws_bytes, void* stream, void* ev_begin, void* ev_end) {
  // W = A F_0 F_1 ... F_{nfac-1} V[:, q0 : q0 + sb], applied right to left
  const double* src = V + q0;
  int lds = cap;
  double* tmp[2] = {T0, T1};
  for (int i = nfac - 1; i >= 0; --i) {
    double* dst = (i == 0) ? T2 : tmp[(nfac - 1 - i) % 2];
    int rc = pmp_spmm(n, fac_rowptr[i], fac_colidx[i], fac_vals[i], sb, src, lds, 1.0, 0.0,
                      nullptr, 0, dst, s, stream);
    if (rc) return rc;
    src = dst;
    lds = s;
  }
  int rc = pmp_spmm(n, a_rowptr, a_colidx, a_vals, sb, src, lds, 1.0, 0.0, nullptr, 0, W, s,
                    stream);
  if (rc) return rc;
  mirror[offFlag] = -1.0;  // sentinel, overwritten by the kernel's last write
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (ev_begin) cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_begin), st);
  rc = pmp::orth_step_mirrored(n, C, kc, k, V, cap, total, 2, W, s, sb, total, d_small + offB,
                               d_small + offH1, d_small + offH2, d_small + offR,
                               d_small + offFlag, ws, ws_bytes, stream, d_small, mirror);
  if (ev_end) cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_end), st);
  return rc;
}

int pmp_tsmm(int n, int kv, const double* V, int ldv, int nc, const double* H, double alpha,
             double beta, double* Out, int ldo, void* st);
int pmp_axpby_cols(int n, int nc, double alpha, const double* src, int lds, const int32_t* sc,
                   double beta, double* dst, int ldd, const int32_t* dc, void* st);
int pmp_copy_cols(int n, int nc, const double* src, int lds, const int32_t* sc, double* dst,
                  int ldd, const int32_t* dc, void* st);
int pmp_gram(int n, int kv, const double* V, int ldv, int nw, const double* W, int ldw,
             double* G, void* ws, size_t bytes, void* st);

// End of a GCRO cycle (krylov.py:221-234), all on the device:
//   dX = V[:, :m] Yv + U[:, :k] Yu ; Xt[:, act] += dX
//   Xa = P Xt[:, act] ; X[:, act] = Xa
//   Rb = B[:, act] - A Xa ; R[:, act] = Rb ; nrm = Rb^T Rb
// Blocks are n x s row-major (ld s); Yv (m x na), Yu (k x na), nrm (na x na)
// are device matrices.
int pmp_gcro_cycle_end(int n, int s, int na, const int32_t* act, const double* V, int cap, int m,
                       const double* Yv, const double* U, int kc, int k, const double* Yu,
                       double* dX, double* Xt, double* Z, double* Xa, double* X, const double* B,
                       double* Rb, double* R, int nfac, const int32_t* const* fac_rowptr,
                       const int32_t* const* fac_colidx, const double* const* fac_vals,
                       const int32_t* a_rowptr, const int32_t* a_colidx, const double* a_vals,
                       double* T0, double* T1, double* nrm, void* gram_ws, size_t gram_ws_bytes,
                       void* stream) {
  int rc;
  if (m > 0) {
    if ((rc = pmp_tsmm(n, m, V, cap, na, Yv, 1.0, 0.0, dX, s, stream))) return rc;
  } else if ((rc = pmp_axpby_cols(n, na, 0.0, dX, s, nullptr, 0.0, dX, s, nullptr, stream))) {
    return rc;
  }
  if (k > 0 && (rc = pmp_tsmm(n, k, U, kc, na, Yu, 1.0, 1.0, dX, s, stream))) return rc;
  if ((rc = pmp_axpby_cols(n, na, 1.0, dX, s, nullptr, 1.0, Xt, s, act, stream))) return rc;
  if ((rc = pmp_copy_cols(n, na, Xt, s, act, Z, s, nullptr, stream))) return rc;
  const double* xa = Z;
  if (nfac > 0) {
    const double* src = Z;
    double* tmp[2] = {T0, T1};
    for (int i = nfac - 1; i >= 0; --i) {
      double* dst = (i == 0) ? Xa : tmp[(nfac - 1 - i) % 2];
      if ((rc = pmp_spmm(n, fac_rowptr[i], fac_colidx[i], fac_vals[i], na, src, s, 1.0, 0.0,
                         nullptr, 0, dst, s, stream)))
        return rc;
      src = dst;
    }
    xa = Xa;
  }
  if ((rc = pmp_copy_cols(n, na, xa, s, nullptr, X, s, act, stream))) return rc;
  if ((rc = pmp_copy_cols(n, na, B, s, act, Rb, s, nullptr, stream))) return rc;
  if ((rc = pmp_spmm(n, a_rowptr, a_colidx, a_vals, na, xa, s, -1.0, 1.0, Rb, s, Rb, s, stream)))
    return rc;
  if ((rc = pmp_copy_cols(n, na, Rb, s, nullptr, R, s, act, stream))) return rc;
  return pmp_gram(n, na, Rb, s, na, Rb, s, nrm, gram_ws, gram_ws_bytes, stream);
}

int pmp_host_hls_append(int ldq, int nrhs, int ncols_old, int nnew, int nrows,
                        const double* newcols, double* QR, double* tau, int* ext, double* C,
                        double* Y, double* resnorm);

// Fold a finished fast-path step (rank == sb) into the projected problem:
// Bmat[:, q0:q1] = B, Hb[:total, q0:q1] += H1, += H2 (krylov.py:190-196),
// Hb[total:total+sb, q0:q1] = R (krylov.py:198-200), then append the new
// block columns of G to its incremental QR (first call also adds the k
// identity columns).  Hb: cap x cap row-major, Bmat: k x cap row-major.
// Returns the pmp_host_hls_append code (1 = G rank deficient).
int pmp_gcro_absorb(const double* small, int offB, int offH1, int offH2, int offR, int cap, int k,
                    int q0, int sb, int total, double* Bmat, double* Hb, int ldq, int nrhs,
                    int ncols_old, double* QR, double* tau, int* ext, double* Cq, double* Y,
                    double* resnorm, double* colsbuf) {
  const double* B = small + offB;
  const double* H1 = small + offH1;
  const double* H2 = small + offH2;
  const double* R = small + offR;
  for (int i = 0; i < k; ++i)
    for (int c = 0; c < sb; ++c) Bmat[(size_t)i * cap + q0 + c] = B[i * sb + c];
  for (int i = 0; i < total; ++i)
    for (int c = 0; c < sb; ++c) {
      double h = Hb[(size_t)i * cap + q0 + c];
      h += H1[i * sb + c];
      h += H2[i * sb + c];
      Hb[(size_t)i * cap + q0 + c] = h;
    }
  for (int i = 0; i < sb; ++i)
    for (int c = 0; c < sb; ++c) Hb[(size_t)(total + i) * cap + q0 + c] = R[i * sb + c];
  const int tot_new = total + sb;
  const int nrows = k + tot_new;
  const bool first = ncols_old == 0;
  const int nnew = first ? k + sb : sb;
  // new columns of G (column-major nrows x nnew)
  for (int q = 0; q < nrows * nnew; ++q) colsbuf[q] = 0.0;
  int o = 0;
  if (first) {
    for (int i = 0; i < k; ++i) colsbuf[i + (size_t)i * nrows] = 1.0;
    o = k;
  }
  for (int c = 0; c < sb; ++c) {
    double* col = colsbuf + (size_t)(o + c) * nrows;
    for (int i = 0; i < k; ++i) col[i] = Bmat[(size_t)i * cap + q0 + c];
    for (int i = 0; i < tot_new; ++i) col[k + i] = Hb[(size_t)i * cap + q0 + c];
  }
  return pmp_host_hls_append(ldq, nrhs, ncols_old, nnew, nrows, colsbuf, QR, tau, ext, Cq, Y,
                             resnorm);
}

// The inner loop of one GCRO cycle (krylov.py:184-216), natively, for the
// fast path (every block step full rank, G full rank).  Mirrors the Python
// loop in krylov._solve exactly: launch (or reuse the speculatively
// launched) step, wait for its flag, speculate the next step, absorb,
// estimate, stop on convergence / restart length / max_iters.  Returns to
// the caller (status 4 / 5) when a step needs the host fallbacks.
int pmp_gcro_inner(PmpGcroInner* g) {
  const int na = g->na;
  g->steps_done = 0;
  while (true) {
    if (g->iterations >= g->max_iters) {
      g->status = 3;
      return PMP_OK;
    }
    if (g->m >= g->inner_restart) {
      g->status = 2;
      return PMP_OK;
    }
    const int q0 = g->m, sb = g->total - g->m;
    double* mirror = g->mirror[g->buf];
    if (!g->launched) {
      int rc = pmp_gcro_step(g->n, g->s, g->nfac, g->fac_rowptr, g->fac_colidx, g->fac_vals,
                             g->a_rowptr, g->a_colidx, g->a_vals, g->V, g->cap, q0, sb, g->W,
                             g->T0, g->T1, g->T2, g->C, g->kc, g->k, g->total, g->d_small, mirror,
                             g->offB, g->offH1, g->offH2, g->offR, g->offFlag, g->orth_ws,
                             g->orth_ws_bytes, g->stream, nullptr, nullptr);
      if (rc) return rc;
      g->launched = 1;
    }
    int rc = pmp_host_wait_flag(mirror + g->offFlag, -1.0, 60000000LL, g->stream);
    if (rc) return rc;
    if (mirror[g->offFlag] != 0.0) {
      g->status = 5;  // deflation fallback: the Python loop takes this step
      return PMP_OK;
    }
    // consume the step
    g->launched = 0;
    g->iterations += 1;
    g->matvecs += sb;
    if (g->nfac) g->precond_applies += sb;
    const int m_new = g->total, total_new = g->total + sb;
    const int cur = g->buf;
    if (g->iterations < g->max_iters && m_new < g->inner_restart &&
        g->prev_max > 20.0 * g->tol) {
      rc = pmp_gcro_step(g->n, g->s, g->nfac, g->fac_rowptr, g->fac_colidx, g->fac_vals,
                         g->a_rowptr, g->a_colidx, g->a_vals, g->V, g->cap, m_new, sb, g->W,
                         g->T0, g->T1, g->T2, g->C, g->kc, g->k, total_new, g->d_small,
                         g->mirror[cur ^ 1], g->offB, g->offH1, g->offH2, g->offR, g->offFlag,
                         g->orth_ws, g->orth_ws_bytes, g->stream, nullptr, nullptr);
      if (rc) return rc;
      g->launched = 1;
      g->buf = cur ^ 1;
    }
    const int nnew = g->ncols == 0 ? g->k + sb : sb;
    rc = pmp_gcro_absorb(g->mirror[cur], g->offB, g->offH1, g->offH2, g->offR, g->cap, g->k, q0,
                         sb, g->total, g->Bmat, g->Hb, g->ldq, na, g->ncols, g->QR, g->tau,
                         g->ext, g->Cq, g->Y, g->res, g->colsbuf);
    g->ncols += nnew;
    g->m = m_new;
    g->total = total_new;
    if (rc == 1) {
      g->status = 4;  // G rank deficient: the caller solves min-norm (gelsd)
      return PMP_OK;
    }
    if (rc) return rc;
    bool conv = true;
    double mx = 0.0;
    double* h = g->hist + (size_t)g->steps_done * na;
    for (int c = 0; c < na; ++c) {
      const double est = g->bn[c] > 0 ? g->res[c] / g->bn[c] : 0.0;
      h[c] = est;
      if (!(est <= g->tol)) conv = false;
      if (est > mx) mx = est;
    }
    g->steps_done += 1;
    g->prev_max = mx;
    if (conv) {
      g->status = 0;
      return PMP_OK;
    }
  }
}

}  // extern "C"
