// Device-resident inner loop of one block-GCRO cycle (krylov.py:184-216).
//
// pmp_gcro_inner drives a cycle from the host: per block step it launches
// the operator chain and the fused orthogonalisation, waits for the small
// results in mapped memory and folds them into the projected least-squares
// problem.  At BASELINE sizes (c2: n = 32768, s = 8) the device work of a
// step is ~50 us while launch gaps + the host round trip add ~100 us, so the
// step is latency bound on the HOST.  k_cycle removes the host from the
// loop: one persistent cooperative launch runs every step of the cycle.
//
//   per step (nfac preconditioner factors):
//     T0 = F_{nfac-1} V[:, q0:q0+sb]  ...  grid barrier per factor
//     W  = A T_last                       rows owned by the block -> smem
//     R1: [C | V]^T W  (reduce, 2 barriers)  W1 = W - C B - V H1
//     R2: [V | W1]^T W1 (reduce, 2 barriers) W2 = W1 - V H2
//     pivoted Cholesky of W2^T W2 (every block, redundantly)
//     [R3: Cholesky-QR2 second pass when kappa > 4 (2 barriers)]
//     Q = W2 P R^-1 -> V[:, total:total+sb] (global + the block's smem copy)
//     control block: Bmat / Hb update, incremental Householder QR of G with
//     Q^T rhs carried along, per-column residual estimates, stop test
//     grid barrier (decision + new V block visible to every block)
//
// Block 0 is the control block: it owns no rows, keeps the projected QR
// (ldq x ldq, column-major), tau / ext and Q^T rhs in its shared memory for
// the whole cycle, and writes them back at exit.  Worker blocks keep their
// rows of [C | V] resident in shared memory across steps when they fit
// (c2: 111 rows x 87 columns), so each step reads only the new block.
#include "orth_dev.cuh"

namespace pmp {

struct CycleArgs {
  int n, s, cap, kc, ldq, k, na, sb, nfac;
  const int32_t* frp[3];
  const int32_t* fci[3];
  const double* fva[3];
  const int32_t* arp;
  const int32_t* aci;
  const double* ava;
  double *V, *W, *T0, *T1;
  const double* C;
  double* small;
  double* mirror;
  int offB, offH1, offH2, offR;
  double *partial, *gout, *Q1g;
  int rows_per_block, ldx, max_iters, inner_restart, hist_cap;
  double tol;
  double* proj;
  int oBmat, oHb, oQR, oTau, oCq, oY, oRes, oBn, oHist;
  int* ist;
};

// Y[r][c] = sum_e vals[e] X[colidx[e]][c] for this block's rows r0 + [0, nr):
// NY lanes per row (lane = column), two rows per thread, the row's entries
// gathered 8 at a time with all index / value loads issued before the X
// gathers (independent L2 round trips).  X may have been written earlier in
// this kernel by other blocks: loads bypass L1 (ld.cg).  Accumulation order
// matches k_spmm (even / odd entries, then summed).
template <int NY>
__device__ void spmm_rows(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ va, const double* X, int ldx, int sb,
                          double* Y, int ldy, int r0, int nr) {
  constexpr int PER = kOrthT / NY;
  const int c = threadIdx.x % NY, slot = threadIdx.x / NY;
  const bool col_ok = c < sb;
  for (int base = 0; base < nr; base += 2 * PER) {
    int lo[2], hi[2];
    double a0[2] = {0.0, 0.0}, a1[2] = {0.0, 0.0};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int r = base + slot + u * PER;
      lo[u] = 0;
      hi[u] = 0;
      if (r < nr) {
        lo[u] = __ldg(rp + r0 + r);
        hi[u] = __ldg(rp + r0 + r + 1);
      }
    }
    const int len = max(hi[0] - lo[0], hi[1] - lo[1]);
    for (int e0 = 0; e0 < len; e0 += 8) {
      int j[2][8];
      double w[2][8], x[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = lo[u] + e0 + q;
          const bool ok = e < hi[u];
          j[u][q] = ok ? __ldg(ci + e) : -1;
          w[u][q] = ok ? __ldg(va + e) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int q = 0; q < 8; ++q)
          x[u][q] = (j[u][q] >= 0 && col_ok) ? __ldcg(X + (size_t)j[u][q] * ldx + c) : 0.0;
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q & 1)
            a1[u] += w[u][q] * x[u][q];
          else
            a0[u] += w[u][q] * x[u][q];
        }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int r = base + slot + u * PER;
      if (r < nr && col_ok) Y[(size_t)r * ldy + c] = a0[u] + a1[u];
    }
  }
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// control-block shared state
struct Ctl {
  double* QR;    // ldq x ldq, column-major
  double* tau;   // ldq
  double* Cq;    // ldq x na, column-major (Q^T rhs)
  double* cols;  // sb x ldq: the step's new columns of G
  double* ybuf;  // 8 x ldq: per-warp back-substitution
  double* Rr;    // sb x sb: R of the step (un-pivoted)
  double* res;   // na
  int* ext;      // ldq
};

// Fold one full-rank step into Bmat / Hb and the incremental QR of G
// (pmp_gcro_absorb + pmp_host_hls_append, csrc/gcro_host.cu, hostls.cpp),
// then the residual estimates and the stop test (krylov.py:204-216).
// Returns 0 continue, 1 converged, 4 G (near) rank deficient.
__device__ int ctl_absorb(const CycleArgs& P, const Ctl& S, int q0, int total, int ncols_old,
                          int hrow) {
  const int k = P.k, sb = P.sb, na = P.na, ldq = P.ldq, cap = P.cap;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned full = 0xffffffffu;
  const int nrows = k + total + sb;
  const bool first = ncols_old == 0;
  const int jb = ncols_old + (first ? k : 0);  // G column of the step's first new column
  const int n1 = jb + sb;
  const double* B = P.small + P.offB;
  const double* H1 = P.small + P.offH1;
  const double* H2 = P.small + P.offH2;
  __shared__ int s_def;
  __shared__ int s_ret;
  if (first) {
    // the k identity columns of G: trivial reflectors (tau = 0)
    for (int q = threadIdx.x; q < k * ldq; q += kOrthT) {
      const int j = q / ldq, i = q % ldq;
      S.QR[(size_t)j * ldq + i] = (i == j) ? 1.0 : 0.0;
    }
    for (int j = threadIdx.x; j < k; j += kOrthT) {
      S.tau[j] = 0.0;
      S.ext[j] = nrows;
    }
  }
  // Bmat[:, q0:q1] = B ; Hb[:total, q0:q1] += H1, += H2 ; Hb[total:, q0:q1] = R
  for (int q = threadIdx.x; q < sb * ldq; q += kOrthT) {
    const int c = q / ldq, i = q % ldq;
    double v = 0.0;
    if (i < k) {
      v = __ldcg(B + i * sb + c);
      P.proj[P.oBmat + (size_t)i * cap + q0 + c] = v;
    } else if (i < k + total) {
      const int t = i - k;
      v = 0.0 + __ldcg(H1 + t * sb + c);
      v += __ldcg(H2 + t * sb + c);
      P.proj[P.oHb + (size_t)t * cap + q0 + c] = v;
    } else if (i < nrows) {
      const int t = i - k - total;
      v = S.Rr[t * sb + c];
      P.proj[P.oHb + (size_t)(total + t) * cap + q0 + c] = v;
    }
    S.cols[(size_t)c * ldq + i] = v;
  }
  __syncthreads();
  // the existing reflectors, in order, on every new column (warp per column)
  if (!first) {
    for (int c = wid; c < sb; c += kOrthT / 32) {
      double* col = S.cols + (size_t)c * ldq;
      for (int j = 0; j < ncols_old; ++j) {
        const double tj = S.tau[j];
        if (tj == 0.0) continue;
        const int e = S.ext[j];
        const double* v = S.QR + (size_t)j * ldq;
        double w = 0.0;
        for (int i = j + 1 + lane; i < e; i += 32) w += v[i] * col[i];
        w = col[j] + warp_sum(w);
        __syncwarp();
        if (lane == 0) col[j] -= tj * w;
        for (int i = j + 1 + lane; i < e; i += 32) col[i] -= tj * w * v[i];
        __syncwarp();
      }
    }
    __syncthreads();
  }
  // factor the new columns; carry Q^T rhs
  for (int c = 0; c < sb; ++c) {
    const int j = jb + c;
    double* col = S.cols + (size_t)c * ldq;
    if (wid == 0) {
      double x2 = 0.0;
      for (int i = j + 1 + lane; i < nrows; i += 32) x2 += col[i] * col[i];
      x2 = warp_sum(x2);
      const double a = col[j];
      double tj = 0.0, beta = a;
      if (x2 != 0.0) {
        beta = -copysign(hypot(a, sqrt(x2)), a);
        tj = (beta - a) / beta;
        const double scal = 1.0 / (a - beta);
        for (int i = j + 1 + lane; i < nrows; i += 32) col[i] *= scal;
      }
      __syncwarp();
      if (lane == 0) {
        col[j] = beta;
        S.tau[j] = tj;
        S.ext[j] = nrows;
      }
      __syncwarp();
      for (int i = lane; i < ldq; i += 32) S.QR[(size_t)j * ldq + i] = i < nrows ? col[i] : 0.0;
    }
    __syncthreads();
    const double tj = S.tau[j];
    if (tj != 0.0) {
      const int rest = sb - c - 1;
      for (int t = wid; t < rest + na; t += kOrthT / 32) {
        double* o = t < rest ? S.cols + (size_t)(c + 1 + t) * ldq : S.Cq + (size_t)(t - rest) * ldq;
        double w = 0.0;
        for (int i = j + 1 + lane; i < nrows; i += 32) w += col[i] * o[i];
        w = o[j] + warp_sum(w);
        __syncwarp();
        if (lane == 0) o[j] -= tj * w;
        for (int i = j + 1 + lane; i < nrows; i += 32) o[i] -= tj * w * col[i];
      }
    }
    __syncthreads();
  }
  // rank check on the R diagonal (warp 0); residual norms from the tail of
  // Q^T rhs (warp per column)
  if (wid == 0) {
    double dmax = 0.0;
    for (int j = lane; j < n1; j += 32) dmax = fmax(dmax, fabs(S.QR[(size_t)j * ldq + j]));
    dmax = warp_max(dmax);
    int def = 0;
    for (int j = lane; j < n1; j += 32)
      if (!(fabs(S.QR[(size_t)j * ldq + j]) > 1e-13 * dmax)) def = 1;
    def = __any_sync(full, def);
    if (lane == 0) s_def = def;
  }
  for (int r = wid; r < na; r += kOrthT / 32) {
    const double* cr = S.Cq + (size_t)r * ldq;
    double s2 = 0.0;
    for (int i = n1 + lane; i < nrows; i += 32) s2 += cr[i] * cr[i];
    s2 = warp_sum(s2);
    if (lane == 0) {
      S.res[r] = sqrt(s2);
      P.proj[P.oRes + r] = S.res[r];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int ret = 0;
    if (s_def) {
      ret = 4;
    } else {
      bool conv = true;
      for (int c = 0; c < na; ++c) {
        const double bn = P.proj[P.oBn + c];
        const double est = bn > 0.0 ? S.res[c] / bn : 0.0;
        if (hrow < P.hist_cap) P.proj[P.oHist + (size_t)hrow * na + c] = est;
        if (!(est <= P.tol)) conv = false;
      }
      ret = conv ? 1 : 0;
    }
    s_ret = ret;
  }
  __syncthreads();
  return s_ret;
}

// Y = R^-1 (Q^T rhs)[:n1], one warp per right-hand side (row-oriented back
// substitution, hostls.cpp:175-182); Y is stored rhs-major (na x n1).
__device__ void ctl_solve_y(const CycleArgs& P, const Ctl& S, int n1) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ldq = P.ldq;
  double* y = S.ybuf + (size_t)wid * ldq;
  for (int r = wid; r < P.na; r += kOrthT / 32) {
    const double* cr = S.Cq + (size_t)r * ldq;
    for (int i = n1 - 1; i >= 0; --i) {
      double s = 0.0;
      for (int t = i + 1 + lane; t < n1; t += 32) s += S.QR[(size_t)t * ldq + i] * y[t];
      s = warp_sum(s);
      if (lane == 0) y[i] = (cr[i] - s) / S.QR[(size_t)i * ldq + i];
      __syncwarp();
    }
    for (int i = lane; i < n1; i += 32) P.proj[P.oY + (size_t)r * n1 + i] = y[i];
    __syncwarp();
  }
}

template <bool CACHED, int NY>
__global__ void __launch_bounds__(kOrthT, 2) k_cycle(CycleArgs P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sh[];
  const bool ctl = blockIdx.x == 0;
  const int r0 = ctl ? 0 : (blockIdx.x - 1) * P.rows_per_block;
  const int r1 = ctl ? 0 : min(P.n, r0 + P.rows_per_block);
  const int nr = max(0, r1 - r0);
  const int sb = P.sb, k = P.k, cap = P.cap, kc = P.kc, ldq = P.ldq;
  const int kmax = (k + cap + sb) * sb;
  double* p = sh;
  double* G = p;
  p += kmax;
  double* R1 = p;
  p += sb * sb;
  double* R2 = p;
  p += sb * sb;
  double* red = p;
  p += 8 * 32 * sb;
  int* piv = reinterpret_cast<int*>(p);
  int* piv2 = piv + 16;
  int* flag = piv + 32;
  p += 20;
  double* region = p;  // worker: cached rows; control: the projected state

  // ---- worker row views ----------------------------------------------------
  const int ldx = P.ldx;
  const int ldw = CACHED ? odd_ld(sb) : P.s;
  double* Xs = region;
  double* Wv = CACHED ? region + (size_t)nr * ldx : P.W + (size_t)r0 * P.s;
  double* Q1 = P.Q1g + (size_t)r0 * sb;

  // ---- control state ---------------------------------------------------------
  Ctl S;
  {
    double* q = region;
    S.QR = q;
    q += (size_t)ldq * ldq;
    S.tau = q;
    q += ldq;
    S.Cq = q;
    q += (size_t)ldq * P.na;
    S.cols = q;
    q += (size_t)sb * ldq;
    S.ybuf = q;
    q += (size_t)8 * ldq;
    S.Rr = q;
    q += sb * sb;
    S.res = q;
    q += 16;
    S.ext = reinterpret_cast<int*>(q);
  }

  int m = P.ist[0], total = P.ist[1], ncols = P.ist[2], it = P.ist[3];
  if (ctl) {
    for (int q = threadIdx.x; q < ncols * ldq; q += kOrthT)
      S.QR[q] = P.proj[P.oQR + q];
    for (int q = threadIdx.x; q < ldq; q += kOrthT) {
      S.tau[q] = P.proj[P.oTau + q];
      S.ext[q] = P.ist[16 + q];
    }
    for (int q = threadIdx.x; q < ldq * P.na; q += kOrthT) S.Cq[q] = P.proj[P.oCq + q];
    if (ncols == 0) {
      for (int q = threadIdx.x; q < k * cap; q += kOrthT) P.proj[P.oBmat + q] = 0.0;
      for (int q = threadIdx.x; q < cap * cap; q += kOrthT) P.proj[P.oHb + q] = 0.0;
    }
  } else if (CACHED) {
    const int kx0 = k + total;
    for (int q = threadIdx.x; q < nr * kx0; q += kOrthT) {
      const int r = q / kx0, t = q % kx0;
      Xs[(size_t)r * ldx + t] = t < k ? P.C[(size_t)(r0 + r) * kc + t]
                                      : P.V[(size_t)(r0 + r) * cap + t - k];
    }
  }
  __syncthreads();

  int status = 0, hrow = 0;
  while (true) {
    if (it >= P.max_iters) {
      status = 3;
      break;
    }
    if (m >= P.inner_restart) {
      status = 2;
      break;
    }
    const int q0 = m;
    // ---- W = A F_0 .. F_{nfac-1} V[:, q0 : q0 + sb] ---------------------------
    const double* src = P.V + q0;
    int lds = cap;
    for (int f = P.nfac - 1; f >= 0; --f) {
      double* dst = ((P.nfac - 1 - f) & 1) ? P.T1 : P.T0;
      spmm_rows<NY>(P.frp[f], P.fci[f], P.fva[f], src, lds, sb, dst + (size_t)r0 * P.s, P.s, r0,
                    nr);
      __threadfence();
      grid.sync();
      src = dst;
      lds = P.s;
    }
    spmm_rows<NY>(P.arp, P.aci, P.ava, src, lds, sb, Wv, ldw, r0, nr);
    __syncthreads();

    // ---- R1: [C | V]^T W --------------------------------------------------------
    const int kx = k + total;
    const Rows CV = CACHED ? Rows{Xs, ldx, kx, Xs, ldx}
                           : Rows{P.C + (size_t)r0 * kc, kc, k, P.V + (size_t)r0 * cap, cap};
    const double* Vrows = CACHED ? Xs + k : P.V + (size_t)r0 * cap;
    const int ldvr = CACHED ? ldx : cap;
    const Rows Vonly{Vrows, ldvr, total, Vrows, ldvr};
    double* outB = P.small + P.offB;
    double* outH1 = P.small + P.offH1;
    double* outH2 = P.small + P.offH2;
    block_gram<NY>(CV, kx, Wv, ldw, sb, nr, red, P.partial);
    grid_reduce(grid, P.partial, P.gout, kx * sb, G, outB, k * sb, outH1);
    block_update<NY>(CV, kx, Wv, ldw, sb, nr, G);
    // ---- R2: [V | W1]^T W1 ------------------------------------------------------
    const int kx2 = total + sb;
    {
      const Rows VW{Vrows, ldvr, total, Wv, ldw};
      block_gram<NY>(VW, kx2, Wv, ldw, sb, nr, red, P.partial);
      grid_reduce(grid, P.partial, P.gout, kx2 * sb, G, outH2, total * sb, nullptr);
    }
    // G_W = W1^T W1 - H2^T H2 (into R2 as scratch), then W2 = W1 - V H2
    const int n4 = 4 * sb * sb, lim4 = (n4 + 31) & ~31;
    for (int q4 = threadIdx.x; q4 < lim4; q4 += kOrthT) {
      const bool act = q4 < n4;
      const int q = q4 >> 2, part = q4 & 3;
      const int i = act ? q / sb : 0, j = act ? q % sb : 0;
      double s = 0.0;
      if (act)
        for (int t = part; t < total; t += 4) s += G[t * sb + i] * G[t * sb + j];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (act && part == 0) R2[q] = G[(size_t)(total + i) * sb + j] - s;
    }
    __syncthreads();
    block_update<NY>(Vonly, total, Wv, ldw, sb, nr, G);
    for (int q = threadIdx.x; q < sb * sb; q += kOrthT) {
      const int i = q / sb, j = q % sb;
      G[q] = 0.5 * (R2[i * sb + j] + R2[j * sb + i]);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      bool ok = warp_cholesky_reg<NY>(G, sb, R1, piv, true, kCholRatio);
      if (threadIdx.x == 0) flag[0] = ok ? 0 : 1;
    }
    __syncthreads();
    bool single = false;
    if (flag[0] == 0) single = fabs(R1[0]) / fabs(R1[(sb - 1) * sb + (sb - 1)]) <= kSkipKappa;
    if (flag[0] == 0 && !single) {
      block_trsm_rows<NY>(Wv, ldw, Q1, sb, nr, sb, R1, piv);
      const Rows Qv{Q1, sb, sb, Q1, sb};
      block_gram<NY>(Qv, sb, Q1, sb, sb, nr, red, P.partial);
      grid_reduce(grid, P.partial, P.gout, sb * sb, G, nullptr, 0, nullptr);
      if (threadIdx.x < 32) {
        bool ok = warp_cholesky_reg<NY>(G, sb, R2, piv2, false, 0.0);
        if (threadIdx.x == 0) flag[0] = ok ? 0 : 1;
      }
      __syncthreads();
    }
    if (flag[0]) {
      // grid-uniform: Cholesky cannot decide the rank -> host Householder
      if (CACHED)
        for (int q = threadIdx.x; q < nr * sb; q += kOrthT)
          P.W[(size_t)(r0 + q / sb) * P.s + q % sb] = Wv[(size_t)(q / sb) * ldw + q % sb];
      status = 5;
      break;
    }
    // ---- Q -> V[:, total : total + sb] -------------------------------------------
    {
      double* qd = CACHED ? Xs + k + total : P.V + (size_t)r0 * cap + total;
      const int ldqd = CACHED ? ldx : cap;
      if (single)
        block_trsm_rows<NY>(Wv, ldw, qd, ldqd, nr, sb, R1, piv);
      else
        block_trsm_rows<NY>(Q1, sb, qd, ldqd, nr, sb, R2, nullptr);
      if (CACHED)
        for (int q = threadIdx.x; q < nr * sb; q += kOrthT)
          P.V[(size_t)(r0 + q / sb) * cap + total + q % sb] = qd[(size_t)(q / sb) * ldx + q % sb];
    }
    // ---- control block: projected problem + stop test ---------------------------
    if (ctl) {
      // R = R2 R1 (pivoted order), un-pivoted: Rr[i, piv[c]] = R[i, c]
      for (int q = threadIdx.x; q < sb * sb; q += kOrthT) {
        const int i = q / sb, c = q % sb;
        double s = 0.0;
        if (single) {
          s = R1[i * sb + c];
        } else {
          for (int a = i; a <= c; ++a) s += R2[i * sb + a] * R1[a * sb + c];
        }
        S.Rr[i * sb + piv[c]] = (c >= i) ? s : 0.0;
      }
      __syncthreads();
      const int dec = ctl_absorb(P, S, q0, total, ncols, hrow);
      if (threadIdx.x == 0) P.ist[6] = dec;
    }
    ncols += (ncols == 0) ? k + sb : sb;
    ++it;
    m = total;
    total += sb;
    __threadfence();
    grid.sync();
    const int dec = __ldcg(P.ist + 6);
    if (dec == 4) {
      status = 4;
      break;
    }
    ++hrow;
    if (dec == 1) {
      status = 0;
      break;
    }
  }

  if (ctl) {
    if (status == 5) {
      // the pending step's B / H1 / H2 for the host fallback (krylov.py
      // _native_cycle status 5)
      const int lens[3] = {k * sb, total * sb, total * sb};
      const int offs[3] = {P.offB, P.offH1, P.offH2};
      for (int a = 0; a < 3; ++a)
        for (int q = threadIdx.x; q < lens[a]; q += kOrthT)
          P.mirror[offs[a] + q] = __ldcg(P.small + offs[a] + q);
    }
    if (status != 5 && status != 4 && ncols > 0) ctl_solve_y(P, S, ncols);
    for (int q = threadIdx.x; q < ncols * ldq; q += kOrthT) P.proj[P.oQR + q] = S.QR[q];
    for (int q = threadIdx.x; q < ldq; q += kOrthT) {
      P.proj[P.oTau + q] = S.tau[q];
      P.ist[16 + q] = S.ext[q];
    }
    for (int q = threadIdx.x; q < ldq * P.na; q += kOrthT) P.proj[P.oCq + q] = S.Cq[q];
    if (threadIdx.x == 0) {
      P.ist[0] = m;
      P.ist[1] = total;
      P.ist[2] = ncols;
      P.ist[3] = it;
      P.ist[4] = status;
      P.ist[5] = hrow;
    }
  }
}

size_t cycle_region_doubles(int rows, int ldx, int sb, int ldq, int na, int cached) {
  size_t ctl = (size_t)ldq * ldq + ldq + (size_t)ldq * na + (size_t)sb * ldq + 8 * (size_t)ldq +
               sb * sb + 16 + (ldq + 1) / 2 + 8;
  size_t work = cached ? (size_t)rows * (ldx + odd_ld(sb)) : 0;
  return ctl > work ? ctl : work;
}

size_t cycle_smem_bytes(int rows, int ldx, int k, int cap, int sb, int ldq, int na, int cached) {
  size_t d = (size_t)(k + cap + sb) * sb + 2 * sb * sb + 8 * 32 * sb + 20;
  d += cycle_region_doubles(rows, ldx, sb, ldq, na, cached);
  return d * sizeof(double);
}

}  // namespace pmp

using namespace pmp;

extern "C" {

size_t pmp_cycle_workspace(int n, int cap, int kc, int s) {
  const int g = orth_max_grid();
  const size_t kmax = (size_t)(kc + cap + s) * s;
  return 256 + sizeof(double) * ((size_t)g * kmax + kmax + (size_t)n * s + 64);
}

int pmp_gcro_cycle_dev(PmpGcroCycle* c) {
  if (!c || c->n < 1 || c->sb < 1 || c->sb > 16 || c->na < 1 || c->na > 16 || c->nfac < 0 ||
      c->nfac > 3 || c->s < c->sb || c->k < 0 || c->k > c->kc || c->ldq < c->kc + c->cap) {
    set_error("pmp_gcro_cycle_dev: bad arguments");
    return PMP_ERR_ARG;
  }
  if (c->ws_bytes < pmp_cycle_workspace(c->n, c->cap, c->kc, c->s)) {
    set_error("pmp_gcro_cycle_dev: workspace too small");
    return PMP_ERR_WORKSPACE;
  }
  const int sms = orth_max_grid() / 2;
  const int ldx = odd_ld(c->kc + c->cap);
  const int NYsel = c->sb <= 8 ? 8 : 16;
  auto pick = [&](int cached) -> void* {
    if (NYsel == 8) return cached ? (void*)k_cycle<true, 8> : (void*)k_cycle<false, 8>;
    return cached ? (void*)k_cycle<true, 16> : (void*)k_cycle<false, 16>;
  };
  // geometry: 1 control block + workers; prefer the cached layout with two
  // blocks per SM, then one, then streaming rows from global memory
  int g = 0, rows = 0, cached = 0;
  size_t smem = 0;
  void* fn = nullptr;
  const int want_bps = c->blocks_per_sm;
  for (int attempt = 0; attempt < 3 && !fn; ++attempt) {
    const int bps = attempt == 0 ? 2 : 1;
    if (want_bps && bps != want_bps && attempt < 2) continue;
    const int cach = attempt < 2 ? 1 : 0;
    const int gb = (attempt == 2 ? (want_bps ? want_bps : 2) : bps) * sms;
    int workers = gb - 1;
    const int need = (c->n + 31) / 32;
    if (need < workers) workers = need;
    const int r = (c->n + workers - 1) / workers;
    const size_t sm = cycle_smem_bytes(r, ldx, c->kc, c->cap, c->sb, c->ldq, c->na, cach);
    if (sm > (size_t)(gb > sms ? 110 : 220) * 1024) continue;
    void* f = pick(cach);
    const int occ = prepare_smem(f, sm, kOrthT);
    if (occ * sms < workers + 1) continue;
    fn = f;
    g = workers + 1;
    rows = r;
    cached = cach;
    smem = sm;
  }
  if (!fn) {
    set_error("pmp_gcro_cycle_dev: no co-resident geometry (n=%d ldq=%d)", c->n, c->ldq);
    return PMP_ERR_ARG;
  }
  (void)cached;
  CycleArgs P;
  P.n = c->n;
  P.s = c->s;
  P.cap = c->cap;
  P.kc = c->kc;
  P.ldq = c->ldq;
  P.k = c->k;
  P.na = c->na;
  P.sb = c->sb;
  P.nfac = c->nfac;
  for (int i = 0; i < 3; ++i) {
    P.frp[i] = i < c->nfac ? c->fac_rowptr[i] : nullptr;
    P.fci[i] = i < c->nfac ? c->fac_colidx[i] : nullptr;
    P.fva[i] = i < c->nfac ? c->fac_vals[i] : nullptr;
  }
  P.arp = c->a_rowptr;
  P.aci = c->a_colidx;
  P.ava = c->a_vals;
  P.V = c->V;
  P.W = c->W;
  P.T0 = c->T0;
  P.T1 = c->T1;
  P.C = c->C;
  P.small = c->d_small;
  P.mirror = c->mirror;
  P.offB = c->offB;
  P.offH1 = c->offH1;
  P.offH2 = c->offH2;
  P.offR = c->offR;
  const size_t kmax = (size_t)(c->kc + c->cap + c->s) * c->s;
  double* w = (double*)((char*)c->ws + 256);
  P.partial = w;
  P.gout = w + (size_t)orth_max_grid() * kmax;
  P.Q1g = P.gout + kmax;
  P.rows_per_block = rows;
  P.ldx = ldx;
  P.max_iters = c->max_iters;
  P.inner_restart = c->inner_restart;
  P.hist_cap = c->hist_cap;
  P.tol = c->tol;
  P.proj = c->d_proj;
  P.oBmat = c->oBmat;
  P.oHb = c->oHb;
  P.oQR = c->oQR;
  P.oTau = c->oTau;
  P.oCq = c->oCq;
  P.oY = c->oY;
  P.oRes = c->oRes;
  P.oBn = c->oBn;
  P.oHist = c->oHist;
  P.ist = c->d_istate;
  void* args[] = {&P};
  cudaError_t e = coop_launch(fn, g, args, smem, reinterpret_cast<cudaStream_t>(c->stream));
  if (e != cudaSuccess) {
    set_error("pmp_gcro_cycle_dev: %s", cudaGetErrorString(e));
    return PMP_ERR_CUDA;
  }
  return cuda_status("pmp_gcro_cycle_dev");
}

}  // extern "C"
