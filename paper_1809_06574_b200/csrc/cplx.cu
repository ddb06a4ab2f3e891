// Complex128 (the reference's native scalar type, sparsecore.py:8-10) on the
// real FP64 kernels, through the real form of a complex matrix:
//
//   A = Ar + i Ai  ->  R(A), 2n x 2n, entry (r, c) -> block [[Ar, -Ai], [Ai, Ar]]
//   x = xr + i xi  ->  R(x) = (xr_0, xi_0, xr_1, xi_1, ...)      (interleaved)
//
// R(A) R(x) = R(A x) and R(A B) = R(A) R(B), so:
//  * a complex least-squares column min ||A(J, I) m - t||_2 (spai.py:229-253)
//    is EXACTLY the real least-squares problem over the columns
//    {2k, 2k + 1 : k in I} of R(A) with target R(t) (same minimiser, same
//    residual norm; complex rank r <-> real rank 2 r);
//  * a complex block Krylov space span_C{B, A B, ...} is the real space
//    spanned by R(b), R(i b), R(A b), ... (krylov.py:105-275 on the block
//    [R(b_0), R(i b_0), R(b_1), R(i b_1), ...]).
// Every structural entry of A becomes a FULL 2 x 2 block (zeros kept) and
// every row holds its diagonal block, so the level-0 support of column 2j of
// R(A) is {2k, 2k + 1 : k in rows(A(:, j)) U {j}} -- the real form of the
// complex level-0 pattern (spai.py:201-204).
#include "common.cuh"

namespace pmp {

// realified CSR: rows 2r and 2r + 1 both hold columns (2c, 2c + 1) for every
// c of row r (sorted), values [re, -im] / [im, re]
__global__ void k_realify(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                          const double* __restrict__ re, const double* __restrict__ im,
                          int* __restrict__ rp2, int* __restrict__ ci2, double* __restrict__ v2) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > n) return;
  if (r == n) {
    rp2[2 * n] = 4 * rp[n];
    return;
  }
  const int lo = rp[r], len = rp[r + 1] - lo;
  const int b0 = 4 * lo, b1 = 4 * lo + 2 * len;
  rp2[2 * r] = b0;
  rp2[2 * r + 1] = b1;
  for (int p = 0; p < len; ++p) {
    const int c = ci[lo + p];
    const double a = re ? re[lo + p] : 0.0, b = im ? im[lo + p] : 0.0;
    if (ci2) {
      ci2[b0 + 2 * p] = 2 * c;
      ci2[b0 + 2 * p + 1] = 2 * c + 1;
      ci2[b1 + 2 * p] = 2 * c;
      ci2[b1 + 2 * p + 1] = 2 * c + 1;
    }
    v2[b0 + 2 * p] = a;
    v2[b0 + 2 * p + 1] = -b;
    v2[b1 + 2 * p] = b;
    v2[b1 + 2 * p + 1] = a;
  }
}

// complex n x s block (re / im row-major, ld ldx) -> real 2n x 2s block,
// column 2c = R(x_c), column 2c + 1 = R(i x_c)
__global__ void k_realify_block(int n, int s, const double* __restrict__ xr,
                                const double* __restrict__ xi, int ldx, double* __restrict__ Y,
                                int ldy) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)n * s) return;
  const int r = (int)(q / s), c = (int)(q % s);
  const double a = xr[(size_t)r * ldx + c], b = xi ? xi[(size_t)r * ldx + c] : 0.0;
  double* y0 = Y + (size_t)(2 * r) * ldy + 2 * c;
  double* y1 = y0 + ldy;
  y0[0] = a;
  y1[0] = b;
  y0[1] = -b;
  y1[1] = a;
}

// real 2n x (2s or s) block -> complex n x s (re, im): x_c = column `stride c`
__global__ void k_derealify_block(int n, int s, const double* __restrict__ Y, int ldy,
                                  int stride, double* __restrict__ xr, double* __restrict__ xi,
                                  int ldx) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)n * s) return;
  const int r = (int)(q / s), c = (int)(q % s);
  xr[(size_t)r * ldx + c] = Y[(size_t)(2 * r) * ldy + stride * c];
  xi[(size_t)r * ldx + c] = Y[(size_t)(2 * r + 1) * ldy + stride * c];
}

// |a| of complex entries (the level-1 weights |A| |A|[:, j], spai.py:212)
__global__ void k_modulus(int nnz, const double* __restrict__ re, const double* __restrict__ im,
                          double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) out[e] = hypot(re[e], im[e]);
}

// complex supports I_j (CSC-like iptr / iidx) -> real-form supports of
// columns 2j and 2j + 1: {2k, 2k + 1 : k in I_j}
__global__ void k_pattern_realify(int n, const int* __restrict__ iptr, const int* __restrict__ iidx,
                                  int* __restrict__ optr, int* __restrict__ oidx) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > n) return;
  if (j == n) {
    optr[2 * n] = 4 * iptr[n];
    return;
  }
  const int lo = iptr[j], len = iptr[j + 1] - lo;
  const int b0 = 4 * lo, b1 = 4 * lo + 2 * len;
  optr[2 * j] = b0;
  optr[2 * j + 1] = b1;
  for (int p = 0; p < len; ++p) {
    const int k = iidx[lo + p];
    oidx[b0 + 2 * p] = 2 * k;
    oidx[b0 + 2 * p + 1] = 2 * k + 1;
    oidx[b1 + 2 * p] = 2 * k;
    oidx[b1 + 2 * p + 1] = 2 * k + 1;
  }
}

// ---------------------------------------------------------------------------
// complex assembly: A = (s^2 M(p) + s D(p)) + K(p) (rpmor.py:92-107, complex
// s / p / terms) or A0 + sum c_j A_j (affine.py:118-134), per union entry in
// the reference's operation order and rounding (numpy's complex128 multiply
// contracts one product of each part into an FMA, see cmul; sums are rounded
// separately -- __dadd_rn).  With real term values and real coefficients
// every product is a real x real product and the contraction is invisible.
// ---------------------------------------------------------------------------

struct CAsm {
  int nterms, mode, any_diag;
  double sr, si, s2r, s2i;
  const double* re[PMP_MAX_TERMS];
  const double* im[PMP_MAX_TERMS];  // null: real term
  int kind[PMP_MAX_TERMS];          // 0 union-expanded, 1 diagonal n-vector
  int group[PMP_MAX_TERMS];
  int first[PMP_MAX_TERMS];
  double cr[PMP_MAX_TERMS], ci[PMP_MAX_TERMS];
};

// numpy's complex128 product a * b (the reference's arithmetic: its SIMD loop
// is mul + fused muladdsub, tests/golden/make_complex_golden.py pins it):
// re = fma(a_re, b_re, -(a_im b_im)), im = fma(a_re, b_im, a_im b_re) -- NOT
// symmetric in (a, b).  scipy's scalar * matrix is data * scalar (a = data,
// rpmor.py:47, :104); affine.py:129 is scalar * data (a = scalar).
__device__ __forceinline__ void cmul(double ar, double ai, double br, double bi, double& r,
                                     double& i) {
  r = __fma_rn(ar, br, -__dmul_rn(ai, bi));
  i = __fma_rn(ar, bi, __dmul_rn(ai, br));
}

__global__ void __launch_bounds__(256) k_assemble_cplx(CAsm R, int nnz, const int* __restrict__ rowid,
                                                       const int* __restrict__ colidx,
                                                       double* __restrict__ ore,
                                                       double* __restrict__ oim,
                                                       int* zero_count) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  bool zero = false;
  if (e < nnz) {
    bool diag = false;
    int row = 0;
    if (R.any_diag) {
      row = __ldg(rowid + e);
      diag = (__ldg(colidx + e) == row);
    }
    // (group accumulators as register selects: a dynamically indexed array
    // lives in local memory, assemble.cu Groups)
    double gr0 = 0.0, gr1 = 0.0, gr2 = 0.0, gi0 = 0.0, gi1 = 0.0, gi2 = 0.0;
    bool gp0 = false, gp1 = false, gp2 = false;
#pragma unroll 1
    for (int t = 0; t < R.nterms; ++t) {
      const int g = R.group[t];
      double vr, vi;
      if (R.kind[t] == 0) {
        vr = __ldg(R.re[t] + e);
        vi = R.im[t] ? __ldg(R.im[t] + e) : 0.0;
      } else {
        vr = diag ? __ldg(R.re[t] + row) : 0.0;
        vi = (diag && R.im[t]) ? __ldg(R.im[t] + row) : 0.0;
      }
      if (R.first[t]) {
        if (g == 0) { gr0 = vr; gi0 = vi; gp0 = true; }
        else if (g == 1) { gr1 = vr; gi1 = vi; gp1 = true; }
        else { gr2 = vr; gi2 = vi; gp2 = true; }
      } else {
        double pr, pi;
        if (R.mode == 0)
          cmul(vr, vi, R.cr[t], R.ci[t], pr, pi);  // data * scalar
        else
          cmul(R.cr[t], R.ci[t], vr, vi, pr, pi);  // scalar * data
        if (g == 0) { gr0 = __dadd_rn(gr0, pr); gi0 = __dadd_rn(gi0, pi); }
        else if (g == 1) { gr1 = __dadd_rn(gr1, pr); gi1 = __dadd_rn(gi1, pi); }
        else { gr2 = __dadd_rn(gr2, pr); gi2 = __dadd_rn(gi2, pi); }
      }
    }
    const double gr[3] = {gr0, gr1, gr2}, gi[3] = {gi0, gi1, gi2};
    const bool gp[3] = {gp0, gp1, gp2};
    double vr = 0.0, vi = 0.0;
    if (R.mode == 0) {
      bool have = false;
      const double cr[3] = {R.s2r, R.sr, 1.0}, ci[3] = {R.s2i, R.si, 0.0};
#pragma unroll
      for (int g = 0; g < 3; ++g) {
        if (!gp[g]) continue;
        double pr, pi;
        if (g == 2) {
          pr = gr[g];  // 1.0 * part: exact
          pi = gi[g];
        } else {
          cmul(gr[g], gi[g], cr[g], ci[g], pr, pi);  // part data * coef
        }
        if (have) {
          vr = __dadd_rn(vr, pr);
          vi = __dadd_rn(vi, pi);
        } else {
          vr = pr;
          vi = pi;
        }
        have = true;
      }
    } else {
      vr = gr[0];
      vi = gi[0];
      if (hypot(vr, vi) < 1e-300) vr = vi = 0.0;  // affine.py:36, :132-133
    }
    if (vr == 0.0) vr = 0.0;
    if (vi == 0.0) vi = 0.0;
    zero = (vr == 0.0 && vi == 0.0);
    ore[e] = vr;
    oim[e] = vi;
  }
  const unsigned b = __ballot_sync(0xffffffffu, zero);
  if ((threadIdx.x & 31) == 0 && b && zero_count) atomicAdd(zero_count, __popc(b));
}

}  // namespace pmp

using namespace pmp;

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int pmp_realify(int n, const int32_t* d_rowptr, const int32_t* d_colidx, const double* d_re,
                const double* d_im, int32_t* d_rowptr2, int32_t* d_colidx2, double* d_vals2,
                void* stream) {
  if (n < 0 || !d_rowptr || !d_rowptr2 || !d_vals2) {
    set_error("pmp_realify: bad arguments");
    return PMP_ERR_ARG;
  }
  k_realify<<<(n + 1 + 255) / 256, 256, 0, S(stream)>>>(n, d_rowptr, d_colidx, d_re, d_im,
                                                        d_rowptr2, d_colidx2, d_vals2);
  return cuda_status("pmp_realify");
}

int pmp_realify_block(int n, int s, const double* d_re, const double* d_im, int ldx, double* d_y,
                      int ldy, void* stream) {
  if (n < 0 || s < 1 || ldx < s || ldy < 2 * s || !d_re || !d_y) {
    set_error("pmp_realify_block: bad arguments");
    return PMP_ERR_ARG;
  }
  const long long tot = (long long)n * s;
  if (tot == 0) return PMP_OK;
  k_realify_block<<<(unsigned)((tot + 255) / 256), 256, 0, S(stream)>>>(n, s, d_re, d_im, ldx,
                                                                         d_y, ldy);
  return cuda_status("pmp_realify_block");
}

int pmp_derealify_block(int n, int s, const double* d_y, int ldy, int stride, double* d_re,
                        double* d_im, int ldx, void* stream) {
  if (n < 0 || s < 1 || stride < 1 || ldy < stride * (s - 1) + 1 || ldx < s || !d_y || !d_re ||
      !d_im) {
    set_error("pmp_derealify_block: bad arguments");
    return PMP_ERR_ARG;
  }
  const long long tot = (long long)n * s;
  if (tot == 0) return PMP_OK;
  k_derealify_block<<<(unsigned)((tot + 255) / 256), 256, 0, S(stream)>>>(n, s, d_y, ldy, stride,
                                                                           d_re, d_im, ldx);
  return cuda_status("pmp_derealify_block");
}

int pmp_modulus(int nnz, const double* d_re, const double* d_im, double* d_out, void* stream) {
  if (nnz < 0 || (nnz && (!d_re || !d_im || !d_out))) {
    set_error("pmp_modulus: bad arguments");
    return PMP_ERR_ARG;
  }
  if (!nnz) return PMP_OK;
  k_modulus<<<(nnz + 255) / 256, 256, 0, S(stream)>>>(nnz, d_re, d_im, d_out);
  return cuda_status("pmp_modulus");
}

int pmp_pattern_realify(int n, const int32_t* d_iptr, const int32_t* d_iidx, int32_t* d_optr,
                        int32_t* d_oidx, void* stream) {
  if (n < 0 || !d_iptr || !d_optr) {
    set_error("pmp_pattern_realify: bad arguments");
    return PMP_ERR_ARG;
  }
  k_pattern_realify<<<(n + 1 + 255) / 256, 256, 0, S(stream)>>>(n, d_iptr, d_iidx, d_optr,
                                                                d_oidx);
  return cuda_status("pmp_pattern_realify");
}

int pmp_assemble_cplx(int nnz, int nterms, const double* const* h_re, const double* const* h_im,
                      const int32_t* h_kind, const int32_t* h_group, const int32_t* h_first,
                      const double* h_cr, const double* h_ci, int mode, double sr, double si,
                      double s2r, double s2i, const int32_t* d_rowid, const int32_t* d_colidx,
                      double* d_re, double* d_im, int32_t* d_zero_count, void* stream) {
  if (nnz < 0 || nterms < 1 || nterms > PMP_MAX_TERMS || !h_re || !d_re || !d_im) {
    set_error("pmp_assemble_cplx: bad arguments");
    return PMP_ERR_ARG;
  }
  CAsm R;
  R.nterms = nterms;
  R.mode = mode;
  R.any_diag = 0;
  R.sr = sr;
  R.si = si;
  R.s2r = s2r;
  R.s2i = s2i;
  for (int t = 0; t < nterms; ++t) {
    R.re[t] = h_re[t];
    R.im[t] = h_im ? h_im[t] : nullptr;
    R.kind[t] = h_kind[t];
    R.group[t] = h_group[t];
    R.first[t] = h_first[t];
    R.cr[t] = h_cr[t];
    R.ci[t] = h_ci[t];
    if (h_kind[t] == 1) R.any_diag = 1;
  }
  if (R.any_diag && (!d_rowid || !d_colidx)) {
    set_error("pmp_assemble_cplx: diagonal terms need row ids");
    return PMP_ERR_ARG;
  }
  if (!nnz) return PMP_OK;
  k_assemble_cplx<<<(nnz + 255) / 256, 256, 0, S(stream)>>>(R, nnz, d_rowid, d_colidx, d_re, d_im,
                                                           d_zero_count);
  return cuda_status("pmp_assemble_cplx");
}

}  // extern "C"
