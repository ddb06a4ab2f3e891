// Host-side small dense algebra of block GCRO (plain C++, no device).
//
// The reference does the s x s rank-revealing QR with LAPACK geqp3
// (krylov.py:88, via scipy) and the projected least-squares problem
// min ||rhs - G Y|| with LAPACK gelsd from scratch at every block step
// (krylov.py:204-212).  Both are tiny, but through numpy/scipy they cost
// 0.05-1 ms of host time per step -- more than the device work of a step.
// These routines compute the same quantities natively:
//   pmp_host_deflate : column-pivoted Householder QR of the s x s TSQR factor,
//                      rank by |R_kk| > tol |R_00| (krylov.py:89-95), the
//                      un-pivoted R rows and T = Pi R11^-1 that maps the
//                      block to its orthonormal basis on the device;
//   pmp_host_hls_append : incremental Householder QR of G as block columns
//                      (and rows) are appended, with Q^T rhs carried along,
//                      returning Y and the per-column residual norms
//                      ||rhs - G Y|| (krylov.py:211-212).  For full column
//                      rank G this is the same minimiser gelsd returns; a
//                      (near-)rank-deficient G is reported so the caller can
//                      fall back to the minimum-norm gelsd solve.
#include <math.h>
#include <string.h>

#include "../../include/pmorb200.h"

namespace {

inline double sq(double x) { return x * x; }

// LAPACK dlarfg on (alpha, x[0..len)) with stride: returns tau, overwrites
// alpha with beta and x with v(1:)
double larfg(double* alpha, double* x, int len, int stride) {
  double xn2 = 0.0;
  for (int i = 0; i < len; ++i) xn2 += sq(x[i * stride]);
  if (xn2 == 0.0) return 0.0;
  double a = *alpha;
  double beta = -copysign(hypot(a, sqrt(xn2)), a);
  double tau = (beta - a) / beta;
  double scal = 1.0 / (a - beta);
  for (int i = 0; i < len; ++i) x[i * stride] *= scal;
  *alpha = beta;
  return tau;
}

}  // namespace

extern "C" {

int pmp_host_deflate(int mz, const double* rt, double tol, int* rank_out, double* T,
                     double* Rout, double* cond_out) {
  if (mz < 0 || mz > 64) return PMP_ERR_ARG;
  double A[64 * 64];   // column-major work copy
  int piv[64];
  double nrm[64];
  for (int i = 0; i < mz; ++i)
    for (int j = 0; j < mz; ++j) A[i + j * mz] = rt[i * mz + j];
  for (int j = 0; j < mz; ++j) piv[j] = j;
  for (int k = 0; k < mz; ++k) {
    // exact norms of the trailing columns (rows k..mz-1), first max wins
    int p = k;
    double best = -1.0;
    for (int j = k; j < mz; ++j) {
      double s = 0.0;
      for (int i = k; i < mz; ++i) s += sq(A[i + j * mz]);
      nrm[j] = s;
      if (s > best) {
        best = s;
        p = j;
      }
    }
    if (p != k) {
      for (int i = 0; i < mz; ++i) {
        double t = A[i + k * mz];
        A[i + k * mz] = A[i + p * mz];
        A[i + p * mz] = t;
      }
      int t = piv[k];
      piv[k] = piv[p];
      piv[p] = t;
    }
    double tau = larfg(&A[k + k * mz], &A[k + 1 + k * mz], mz - k - 1, 1);
    if (tau != 0.0) {
      for (int j = k + 1; j < mz; ++j) {
        double w = A[k + j * mz];
        for (int i = k + 1; i < mz; ++i) w += A[i + k * mz] * A[i + j * mz];
        A[k + j * mz] -= tau * w;
        for (int i = k + 1; i < mz; ++i) A[i + j * mz] -= tau * w * A[i + k * mz];
      }
    }
  }
  double d0 = mz ? fabs(A[0]) : 0.0;
  int r = 0;
  if (d0 > 0.0)
    for (int k = 0; k < mz; ++k) r += fabs(A[k + k * mz]) > tol * d0;
  *rank_out = r;
  for (int q = 0; q < mz * mz; ++q) {
    T[q] = 0.0;
    Rout[q] = 0.0;
  }
  if (r == 0) {
    *cond_out = 0.0;
    return PMP_OK;
  }
  // R rows < r un-pivoted: Rout[i, piv[c]] = R[i, c]
  for (int i = 0; i < r; ++i)
    for (int c = 0; c < mz; ++c) Rout[i * mz + piv[c]] = (c >= i) ? A[i + c * mz] : 0.0;
  // inverse of the leading r x r triangle, column by column
  double Rinv[64 * 64];
  for (int c = 0; c < r; ++c) {
    for (int i = r - 1; i >= 0; --i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int t = i + 1; t < r; ++t) s -= A[i + t * mz] * Rinv[t + c * 64];
      Rinv[i + c * 64] = s / A[i + i * mz];
    }
  }
  for (int a = 0; a < r; ++a)
    for (int c = 0; c < r; ++c) T[piv[a] * r + c] = Rinv[a + c * 64];
  *cond_out = d0 / fabs(A[(r - 1) + (r - 1) * mz]);
  return PMP_OK;
}

int pmp_host_hls_append(int ldq, int nrhs, int ncols_old, int nnew, int nrows,
                        const double* newcols, double* QR, double* tau, int* ext, double* C,
                        double* Y, double* resnorm) {
  if (ldq < nrows || ncols_old + nnew > nrows || nrhs < 0) return PMP_ERR_ARG;
  const int n1 = ncols_old + nnew;
  // place the new columns (rows 0..nrows-1, zero below)
  for (int c = 0; c < nnew; ++c) {
    double* col = QR + (size_t)(ncols_old + c) * ldq;
    for (int i = 0; i < ldq; ++i) col[i] = (i < nrows) ? newcols[i + (size_t)c * nrows] : 0.0;
  }
  // apply the existing reflectors, in order
  for (int j = 0; j < ncols_old; ++j) {
    const double tj = tau[j];
    if (tj == 0.0) continue;
    const double* v = QR + (size_t)j * ldq;
    const int e = ext[j];
    for (int c = 0; c < nnew; ++c) {
      double* col = QR + (size_t)(ncols_old + c) * ldq;
      double w = col[j];
      for (int i = j + 1; i < e; ++i) w += v[i] * col[i];
      col[j] -= tj * w;
      for (int i = j + 1; i < e; ++i) col[i] -= tj * w * v[i];
    }
  }
  // factor the new columns; carry Q^T rhs
  for (int c = 0; c < nnew; ++c) {
    const int j = ncols_old + c;
    double* col = QR + (size_t)j * ldq;
    double tj = larfg(&col[j], &col[j + 1], nrows - j - 1, 1);
    tau[j] = tj;
    ext[j] = nrows;
    if (tj == 0.0) continue;
    for (int c2 = c + 1; c2 < nnew; ++c2) {
      double* o = QR + (size_t)(ncols_old + c2) * ldq;
      double w = o[j];
      for (int i = j + 1; i < nrows; ++i) w += col[i] * o[i];
      o[j] -= tj * w;
      for (int i = j + 1; i < nrows; ++i) o[i] -= tj * w * col[i];
    }
    for (int r = 0; r < nrhs; ++r) {
      double* o = C + (size_t)r * ldq;
      double w = o[j];
      for (int i = j + 1; i < nrows; ++i) w += col[i] * o[i];
      o[j] -= tj * w;
      for (int i = j + 1; i < nrows; ++i) o[i] -= tj * w * col[i];
    }
  }
  // rank check on the R diagonal
  double dmax = 0.0;
  for (int j = 0; j < n1; ++j) dmax = fmax(dmax, fabs(QR[j + (size_t)j * ldq]));
  int deficient = 0;
  for (int j = 0; j < n1; ++j)
    if (!(fabs(QR[j + (size_t)j * ldq]) > 1e-13 * dmax)) deficient = 1;
  // Y = R^-1 C[:n1], residual norms from the tail of C
  for (int r = 0; r < nrhs; ++r) {
    const double* cr = C + (size_t)r * ldq;
    double* y = Y + (size_t)r * n1;
    for (int i = n1 - 1; i >= 0; --i) {
      double s = cr[i];
      for (int t = i + 1; t < n1; ++t) s -= QR[i + (size_t)t * ldq] * y[t];
      y[i] = s / QR[i + (size_t)i * ldq];
    }
    double s2 = 0.0;
    for (int i = n1; i < nrows; ++i) s2 += sq(cr[i]);
    resnorm[r] = sqrt(s2);
  }
  return deficient ? 1 : PMP_OK;
}

}  // extern "C"
