// Kernel 5: the n-sized work of block GCRO (krylov.py:105-275):
//   5a  CSR SpMM            Y = alpha A X + beta Y0   (op, P.apply, B - A X)
//   5b  tall-skinny Gram    G = V^T W                 (block CGS, C projection)
//       tall-skinny update  Out = beta Out + alpha V H
//   5c  TSQR, R only        Householder QR of row chunks + in-order tree
// Dense blocks are row-major n x k (leading dimension ld): one row of an
// n x s block is s contiguous doubles, so the SpMM gathers X[col, 0:s] as
// one 32..128-byte segment.  All reductions are fixed-order (no floating-
// point atomics): results are bitwise reproducible.
#include "common.cuh"

namespace pmp {

// ---------------------------------------------------------------------------
// 5a SpMM: G lanes per row (G = next pow2 >= s), lane c owns column c
// ---------------------------------------------------------------------------

template <int G>
__global__ void __launch_bounds__(256) k_spmm(int n, const int* __restrict__ rowptr,
                                              const int* __restrict__ colidx,
                                              const double* __restrict__ vals, int s,
                                              const double* __restrict__ X, int ldx, double alpha,
                                              double beta, const double* Y0, int ldy0, double* Y,
                                              int ldy) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(g / G);
  const int c = (int)(g % G);
  if (row >= n || c >= s) return;
  const int lo = __ldg(rowptr + row), hi = __ldg(rowptr + row + 1);
  double a0 = 0.0, a1 = 0.0;
  int e = lo;
  for (; e + 1 < hi; e += 2) {
    const int k0 = __ldg(colidx + e), k1 = __ldg(colidx + e + 1);
    const double v0 = __ldg(vals + e), v1 = __ldg(vals + e + 1);
    a0 += v0 * __ldg(X + (size_t)k0 * ldx + c);
    a1 += v1 * __ldg(X + (size_t)k1 * ldx + c);
  }
  if (e < hi) a0 += __ldg(vals + e) * __ldg(X + (size_t)__ldg(colidx + e) * ldx + c);
  double r = alpha * (a0 + a1);
  if (beta != 0.0) r += beta * Y0[(size_t)row * ldy0 + c];
  Y[(size_t)row * ldy + c] = r;
}

// ---------------------------------------------------------------------------
// 5b Gram G = V^T W: each block reduces a row range into a kv x nw partial
// (rows staged through shared memory), the last block to finish sums the
// partials in block order.
// ---------------------------------------------------------------------------

constexpr int kGramRows = 32;

template <int MAXO>
__global__ void __launch_bounds__(256) k_gram(int n, int kv, const double* __restrict__ V, int ldv,
                                              int nw, const double* __restrict__ W, int ldw,
                                              int chunk, double* partial, unsigned* ticket,
                                              double* Gout) {
  extern __shared__ __align__(16) double sh[];
  double* Vs = sh;                        // kGramRows x kv
  double* Ws = sh + kGramRows * kv;       // kGramRows x nw
  const int tid = threadIdx.x;
  const int K = kv * nw;
  double acc[MAXO];
  int ot[MAXO], oc[MAXO];
#pragma unroll
  for (int q = 0; q < MAXO; ++q) {
    acc[q] = 0.0;
    int o = tid + q * 256;
    ot[q] = o < K ? o / nw : 0;
    oc[q] = o < K ? o % nw : 0;
  }
  const int r0 = blockIdx.x * chunk;
  const int r1 = min(n, r0 + chunk);
  for (int base = r0; base < r1; base += kGramRows) {
    const int rows = min(kGramRows, r1 - base);
    for (int q = tid; q < rows * kv; q += 256) {
      int r = q / kv, t = q % kv;
      Vs[r * kv + t] = V[(size_t)(base + r) * ldv + t];
    }
    for (int q = tid; q < rows * nw; q += 256) {
      int r = q / nw, t = q % nw;
      Ws[r * nw + t] = W[(size_t)(base + r) * ldw + t];
    }
    __syncthreads();
    for (int r = 0; r < rows; ++r) {
#pragma unroll
      for (int q = 0; q < MAXO; ++q) acc[q] += Vs[r * kv + ot[q]] * Ws[r * nw + oc[q]];
    }
    __syncthreads();
  }
  double* mine = partial + (size_t)blockIdx.x * K;
#pragma unroll
  for (int q = 0; q < MAXO; ++q) {
    int o = tid + q * 256;
    if (o < K) mine[o] = acc[q];
  }
  __threadfence();
  __shared__ int last;
  if (tid == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // fixed-order sum over the block partials with 8 independent chains
  // (b mod 8) so the L2 loads overlap; combined in a fixed tree
  const int nb = gridDim.x;
  // `per` threads share one output (all 256 threads busy even for small K);
  // each sums a fixed strided subset of the partials, then the subsets are
  // combined in order through shared memory
  int per = 256 / K;
  if (per < 1) per = 1;
  if (per > 32) per = 32;
  __shared__ double red[256];
  for (int o0 = 0; o0 < K; o0 += 256 / per) {
    const int o = o0 + tid / per, sub = tid % per;
    double s = 0.0;
    if (o < K && tid / per < 256 / per) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      const double* pp = partial + o;
      int b = sub;
      for (; b + 3 * per < nb; b += 4 * per) {
        a0 += __ldcg(pp + (size_t)b * K);
        a1 += __ldcg(pp + (size_t)(b + per) * K);
        a2 += __ldcg(pp + (size_t)(b + 2 * per) * K);
        a3 += __ldcg(pp + (size_t)(b + 3 * per) * K);
      }
      for (; b < nb; b += per) a0 += __ldcg(pp + (size_t)b * K);
      s = (a0 + a1) + (a2 + a3);
    }
    red[tid] = s;
    __syncthreads();
    if (sub == 0 && o < K && tid / per < 256 / per) {
      double t = 0.0;
      for (int q = 0; q < per; ++q) t += red[tid + q];
      Gout[o] = t;
    }
    __syncthreads();
  }
  if (tid == 0) *ticket = 0u;
}

// enough blocks to cover the SMs with >= 64 rows each, but few enough that
// the last block's fixed-order pass over the partials stays ~<= 128 KB
static int gram_blocks(int n, int K) {
  int nb = ceil_div(n, 64);
  if (nb > 296) nb = 296;
  int cap = 16384 / (K > 0 ? K : 1);
  if (cap < 16) cap = 16;
  if (nb > cap) nb = cap;
  if (nb < 1) nb = 1;
  return nb;
}

// ---------------------------------------------------------------------------
// tall-skinny update Out = beta Out + alpha V H
// ---------------------------------------------------------------------------

template <int G>
__global__ void __launch_bounds__(256) k_tsmm(int n, int kv, const double* __restrict__ V, int ldv,
                                              int nc, const double* __restrict__ H, double alpha,
                                              double beta, double* Out, int ldo) {
  extern __shared__ __align__(16) double Hs[];
  for (int q = threadIdx.x; q < kv * nc; q += blockDim.x) Hs[q] = H[q];
  __syncthreads();
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(g / G);
  const int c = (int)(g % G);
  if (row >= n || c >= nc) return;
  const double* v = V + (size_t)row * ldv;
  double a0 = 0.0, a1 = 0.0;
  int t = 0;
  for (; t + 1 < kv; t += 2) {
    a0 += v[t] * Hs[t * nc + c];
    a1 += v[t + 1] * Hs[(t + 1) * nc + c];
  }
  if (t < kv) a0 += v[t] * Hs[t * nc + c];
  double r = alpha * (a0 + a1);
  double* o = Out + (size_t)row * ldo + c;
  if (beta != 0.0) r += beta * (*o);
  *o = r;
}

// ---------------------------------------------------------------------------
// 5c TSQR (R only).  Team = the CTA (256 threads).  The running R (nz x nz)
// sits on top of the next chunk of rows; an unpivoted Householder QR of the
// stack leaves the updated R in its top rows.  Blocks write their R; the
// last block to finish reduces the block R's in block order the same way.
// ---------------------------------------------------------------------------

constexpr int kTsqrT = 256;

__device__ void house_qr_R(double* M, int mm, int nz, const Team<kTsqrT>& tm, double* w) {
  // unpivoted Householder QR of the mm x nz column-major block M (ld = mm);
  // only R (rows 0..nz-1, upper triangle) is kept meaningful.
  const int K = mm < nz ? mm : nz;
  for (int k = 0; k < K; ++k) {
    double part = 0.0;
    for (int i = k + 1 + tm.tid; i < mm; i += kTsqrT) {
      double v = M[i + (size_t)k * mm];
      part += v * v;
    }
    const double xn2 = tm.sum(part);
    const double alpha = M[k + (size_t)k * mm];
    double tau = 0.0, scal = 0.0, beta = alpha;
    if (xn2 > 0.0) {
      beta = -copysign(hypot(alpha, sqrt(xn2)), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (tau == 0.0) continue;
    for (int i = k + 1 + tm.tid; i < mm; i += kTsqrT) M[i + (size_t)k * mm] *= scal;
    tm.sync();
    tm.colsum(
        nz - k - 1, k + 1, mm,
        [&](int c, int i) { return M[i + (size_t)k * mm] * M[i + (size_t)(k + 1 + c) * mm]; },
        w + k + 1);
    tm.sync();
    for (int c = tm.tid; c < nz - k - 1; c += kTsqrT) w[k + 1 + c] += M[k + (size_t)(k + 1 + c) * mm];
    tm.sync();
    const int rows = mm - k, ncol = nz - k - 1;
    for (int q = tm.tid; q < rows * ncol; q += kTsqrT) {
      int i = k + q % rows;
      int jj = k + 1 + q / rows;
      double wj = w[jj];
      if (i == k)
        M[k + (size_t)jj * mm] -= tau * wj;
      else
        M[i + (size_t)jj * mm] -= tau * wj * M[i + (size_t)k * mm];
    }
    if (tm.tid == 0) M[k + (size_t)k * mm] = beta;
    tm.sync();
  }
}

// load R (nz x nz upper, row-major at src) into the top of M (ld mm)
__device__ inline void load_R_top(double* M, int mm, int nz, const double* src, int tid) {
  for (int q = tid; q < nz * nz; q += kTsqrT) {
    int i = q / nz, c = q % nz;
    M[i + (size_t)c * mm] = (c >= i) ? src[q] : 0.0;
  }
}

__device__ inline void store_R(const double* M, int mm, int nz, double* dst, int tid) {
  for (int q = tid; q < nz * nz; q += kTsqrT) {
    int i = q / nz, c = q % nz;
    dst[q] = (c >= i) ? M[i + (size_t)c * mm] : 0.0;
  }
}

__global__ void __launch_bounds__(kTsqrT) k_tsqr(int n, int nz, const double* __restrict__ Z, int ldz,
                                                 int chunk, int sub, double* partial,
                                                 unsigned* ticket, double* Rout) {
  extern __shared__ __align__(16) double sh[];
  double* w = sh;              // nz + 1
  double* red = sh + 40;       // 16
  double* M = sh + 64;         // (nz + sub) x nz
  Team<kTsqrT> tm{(int)threadIdx.x, red};
  const int tid = threadIdx.x;
  const int r0 = blockIdx.x * chunk;
  const int r1 = min(n, r0 + chunk);
  bool have = false;
  double* mine = partial + (size_t)blockIdx.x * nz * nz;
  for (int base = r0; base < r1; base += sub) {
    const int rows = min(sub, r1 - base);
    const int top = have ? nz : 0;
    const int mm = top + rows;
    if (have) load_R_top(M, mm, nz, mine, tid);
    for (int q = tid; q < rows * nz; q += kTsqrT) {
      int r = q / nz, c = q % nz;
      M[top + r + (size_t)c * mm] = Z[(size_t)(base + r) * ldz + c];
    }
    tm.sync();
    house_qr_R(M, mm, nz, tm, w);
    // rows < nz of the result may be fewer than nz when mm < nz: pad zeros
    for (int q = tid; q < nz * nz; q += kTsqrT) {
      int i = q / nz, c = q % nz;
      mine[q] = (c >= i && i < mm) ? M[i + (size_t)c * mm] : 0.0;
    }
    tm.sync();
    have = true;
  }
  if (!have)
    for (int q = tid; q < nz * nz; q += kTsqrT) mine[q] = 0.0;
  __threadfence();
  __shared__ int last;
  if (tid == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // reduce the block R factors in block order
  const int per = sub / nz > 1 ? sub / nz : 1;
  bool have_run = false;
  double* run = Rout;  // running R lives in the output buffer
  for (int b0 = 0; b0 < (int)gridDim.x; b0 += per) {
    const int nb = min(per, (int)gridDim.x - b0);
    const int top = have_run ? nz : 0;
    const int mm = top + nb * nz;
    if (have_run) load_R_top(M, mm, nz, run, tid);
    for (int q = tid; q < nb * nz * nz; q += kTsqrT) {
      int b = q / (nz * nz), rem = q % (nz * nz);
      int i = rem / nz, c = rem % nz;
      M[top + b * nz + i + (size_t)c * mm] = __ldcg(partial + (size_t)(b0 + b) * nz * nz + rem);
    }
    tm.sync();
    house_qr_R(M, mm, nz, tm, w);
    store_R(M, mm, nz, run, tid);
    tm.sync();
    have_run = true;
  }
  if (tid == 0) *ticket = 0u;
}

static void tsqr_geometry(int n, int nz, int* nb, int* chunk, int* sub) {
  int s = nz <= 8 ? 1024 : (nz <= 16 ? 512 : 256);
  *sub = s;
  int blocks = ceil_div(n, s);
  if (blocks > 148) blocks = 148;
  if (blocks < 1) blocks = 1;
  *nb = blocks;
  *chunk = ceil_div(n, blocks);
}

static size_t tsqr_smem(int nz, int sub) { return sizeof(double) * (64 + (size_t)(nz + sub) * nz); }

// ---------------------------------------------------------------------------
// 5c' TSQR for nz <= 16 in registers: lane = row of a 32-row tile.  A warp
// keeps its running R in lanes 0..nz-1 and streams (32 - nz) new rows into
// lanes nz..31 per tile; one Householder QR of the tile (shfl reductions)
// leaves the new R on top.  Warp R's are combined pairwise (2 nz <= 32 rows
// per QR) in a fixed tree inside the block, and the last block combines the
// block R's the same way, so the result is deterministic.
// ---------------------------------------------------------------------------

template <int NZ>
__device__ __forceinline__ void warp_house_qr(double (&a)[NZ], int nz, int lane) {
#pragma unroll
  for (int k = 0; k < NZ; ++k) {
    if (k >= nz) break;
    const double x = (lane > k) ? a[k] : 0.0;
    const double xn2 = warp_sum(x * x);
    const double alpha = __shfl_sync(0xffffffffu, a[k], k);
    if (xn2 == 0.0) continue;
    const double beta = -copysign(hypot(alpha, sqrt(xn2)), alpha);
    const double tau = (beta - alpha) / beta;
    const double scal = 1.0 / (alpha - beta);
    const double v = (lane > k) ? a[k] * scal : (lane == k ? 1.0 : 0.0);
#pragma unroll
    for (int j = k + 1; j < NZ; ++j) {
      if (j >= nz) break;
      const double w = warp_sum(v * a[j]);
      if (lane >= k) a[j] -= tau * w * v;
    }
    if (lane == k)
      a[k] = beta;
    else if (lane > k)
      a[k] = 0.0;
  }
}

// stack R (lanes 0..nz-1, in registers) on top of the R stored row-major at
// src (loaded into lanes nz..2nz-1) and re-triangularise
template <int NZ>
__device__ __forceinline__ void warp_combine(double (&a)[NZ], int nz, int lane, const double* src) {
  if (lane >= nz && lane < 2 * nz) {
#pragma unroll
    for (int c = 0; c < NZ; ++c)
      if (c < nz) a[c] = src[(lane - nz) * nz + c];
  } else if (lane >= 2 * nz) {
#pragma unroll
    for (int c = 0; c < NZ; ++c) a[c] = 0.0;
  }
  warp_house_qr<NZ>(a, nz, lane);
}

template <int NZ>
__device__ __forceinline__ void warp_store_R(const double (&a)[NZ], int nz, int lane, double* dst) {
  if (lane < nz) {
#pragma unroll
    for (int c = 0; c < NZ; ++c)
      if (c < nz) dst[lane * nz + c] = (c >= lane) ? a[c] : 0.0;
  }
}

template <int NZ>
__global__ void __launch_bounds__(256) k_tsqr_warp(int n, int nz, const double* __restrict__ Z,
                                                   int ldz, int chunk, double* partial,
                                                   unsigned* ticket, double* Rout) {
  __shared__ double sR[8][NZ * NZ];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double a[NZ];
#pragma unroll
  for (int c = 0; c < NZ; ++c) a[c] = 0.0;
  // rows of this block, split evenly over its 8 warps
  const int b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  const int per = (b1 - b0 + 7) / 8;
  const int r0 = min(b1, b0 + wid * per), r1 = min(b1, r0 + per);
  const int fresh = 32 - nz;
  for (int base = r0; base < r1; base += fresh) {
    if (lane >= nz) {
      const int row = base + lane - nz;
      if (row < r1) {
        const double* zr = Z + (size_t)row * ldz;
#pragma unroll
        for (int c = 0; c < NZ; ++c) a[c] = (c < nz) ? zr[c] : 0.0;
      } else {
#pragma unroll
        for (int c = 0; c < NZ; ++c) a[c] = 0.0;
      }
    }
    warp_house_qr<NZ>(a, nz, lane);
  }
  warp_store_R<NZ>(a, nz, lane, sR[wid]);
  __syncthreads();
  // tree over the 8 warps: 0+1, 2+3, ... then 0+2, 4+6, then 0+4
  for (int step = 1; step < 8; step <<= 1) {
    if ((wid % (2 * step)) == 0) {
      warp_combine<NZ>(a, nz, lane, sR[wid + step]);
      warp_store_R<NZ>(a, nz, lane, sR[wid]);
    }
    __syncthreads();
  }
  double* mine = partial + (size_t)blockIdx.x * nz * nz;
  for (int q = threadIdx.x; q < nz * nz; q += blockDim.x) mine[q] = sR[0][q];
  __threadfence();
  __shared__ int last;
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // last block: warp w folds block partials w, w+8, w+16, ... in order,
  // then the same fixed tree over the 8 warps
  const int nb = gridDim.x;
#pragma unroll
  for (int c = 0; c < NZ; ++c) a[c] = 0.0;
  for (int b = wid; b < nb; b += 8) {
    // stage partial b in the warp's smem slot, then combine
    for (int q = lane; q < nz * nz; q += 32) sR[wid][q] = __ldcg(partial + (size_t)b * nz * nz + q);
    __syncwarp();
    warp_combine<NZ>(a, nz, lane, sR[wid]);
    __syncwarp();
  }
  warp_store_R<NZ>(a, nz, lane, sR[wid]);
  __syncthreads();
  for (int step = 1; step < 8; step <<= 1) {
    if ((wid % (2 * step)) == 0) {
      warp_combine<NZ>(a, nz, lane, sR[wid + step]);
      warp_store_R<NZ>(a, nz, lane, sR[wid]);
    }
    __syncthreads();
  }
  for (int q = threadIdx.x; q < nz * nz; q += blockDim.x) Rout[q] = sR[0][q];
  if (threadIdx.x == 0) *ticket = 0u;
}

static int tsqr_warp_blocks(int n) {
  int nb = ceil_div(n, 8 * 32 * 4);
  if (nb > 148) nb = 148;
  if (nb < 1) nb = 1;
  return nb;
}

}  // namespace pmp

using namespace pmp;

extern "C" {

int pmp_spmm(int n, const int32_t* rowptr, const int32_t* colidx, const double* vals, int s,
             const double* X, int ldx, double alpha, double beta, const double* Y0, int ldy0,
             double* Y, int ldy, void* st) {
  if (n < 0 || s < 0 || s > 32 || ldx < s || ldy < s || (beta != 0.0 && (!Y0 || ldy0 < s))) {
    set_error("pmp_spmm: bad arguments (n=%d s=%d)", n, s);
    return PMP_ERR_ARG;
  }
  if (n == 0 || s == 0) return PMP_OK;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(st);
  int G = 1;
  while (G < s) G <<= 1;
  long long threads = (long long)n * G;
  int grid = ceil_div(threads, 256);
  switch (G) {
    case 1: k_spmm<1><<<grid, 256, 0, stream>>>(n, rowptr, colidx, vals, s, X, ldx, alpha, beta, Y0, ldy0, Y, ldy); break;
    case 2: k_spmm<2><<<grid, 256, 0, stream>>>(n, rowptr, colidx, vals, s, X, ldx, alpha, beta, Y0, ldy0, Y, ldy); break;
    case 4: k_spmm<4><<<grid, 256, 0, stream>>>(n, rowptr, colidx, vals, s, X, ldx, alpha, beta, Y0, ldy0, Y, ldy); break;
    case 8: k_spmm<8><<<grid, 256, 0, stream>>>(n, rowptr, colidx, vals, s, X, ldx, alpha, beta, Y0, ldy0, Y, ldy); break;
    case 16: k_spmm<16><<<grid, 256, 0, stream>>>(n, rowptr, colidx, vals, s, X, ldx, alpha, beta, Y0, ldy0, Y, ldy); break;
    default: k_spmm<32><<<grid, 256, 0, stream>>>(n, rowptr, colidx, vals, s, X, ldx, alpha, beta, Y0, ldy0, Y, ldy); break;
  }
  return cuda_status("pmp_spmm");
}

size_t pmp_gram_workspace(int n, int kv, int nw) {
  // any K' <= kv * nw needs gram_blocks(n, K') * K' <= max(16384, 296 * 55) doubles
  size_t need = (size_t)gram_blocks(n, kv * nw) * kv * nw;
  if (need < 16384 + 296) need = 16384 + 296;
  return 256 + sizeof(double) * need;
}

int pmp_gram(int n, int kv, const double* V, int ldv, int nw, const double* W, int ldw,
             double* G, void* ws, size_t bytes, void* st) {
  if (n < 0 || kv < 0 || nw < 0 || kv * nw > 8 * 256 || ldv < kv || ldw < nw) {
    set_error("pmp_gram: bad arguments (n=%d kv=%d nw=%d)", n, kv, nw);
    return PMP_ERR_ARG;
  }
  if (kv == 0 || nw == 0) return PMP_OK;
  if (bytes < pmp_gram_workspace(n, kv, nw)) {
    set_error("pmp_gram: workspace too small");
    return PMP_ERR_WORKSPACE;
  }
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(st);
  unsigned* ticket = (unsigned*)ws;
  double* partial = (double*)((char*)ws + 256);
  int nb = gram_blocks(n, kv * nw);
  int chunk = ceil_div(n > 0 ? n : 1, nb);
  size_t sm = sizeof(double) * kGramRows * (kv + nw);
  int K = kv * nw;
  int maxo = ceil_div(K, 256);
  if (maxo <= 1)
    k_gram<1><<<nb, 256, sm, stream>>>(n, kv, V, ldv, nw, W, ldw, chunk, partial, ticket, G);
  else if (maxo <= 2)
    k_gram<2><<<nb, 256, sm, stream>>>(n, kv, V, ldv, nw, W, ldw, chunk, partial, ticket, G);
  else if (maxo <= 4)
    k_gram<4><<<nb, 256, sm, stream>>>(n, kv, V, ldv, nw, W, ldw, chunk, partial, ticket, G);
  else
    k_gram<8><<<nb, 256, sm, stream>>>(n, kv, V, ldv, nw, W, ldw, chunk, partial, ticket, G);
  return cuda_status("pmp_gram");
}

int pmp_tsmm(int n, int kv, const double* V, int ldv, int nc, const double* H, double alpha,
             double beta, double* Out, int ldo, void* st) {
  if (n < 0 || kv < 0 || nc < 0 || nc > 32 || kv * nc > 4096 || ldo < nc || (kv > 0 && ldv < kv)) {
    set_error("pmp_tsmm: bad arguments (n=%d kv=%d nc=%d)", n, kv, nc);
    return PMP_ERR_ARG;
  }
  if (n == 0 || nc == 0) return PMP_OK;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(st);
  int G = 1;
  while (G < nc) G <<= 1;
  int grid = ceil_div((long long)n * G, 256);
  size_t sm = sizeof(double) * (size_t)(kv * nc > 0 ? kv * nc : 1);
  switch (G) {
    case 1: k_tsmm<1><<<grid, 256, sm, stream>>>(n, kv, V, ldv, nc, H, alpha, beta, Out, ldo); break;
    case 2: k_tsmm<2><<<grid, 256, sm, stream>>>(n, kv, V, ldv, nc, H, alpha, beta, Out, ldo); break;
    case 4: k_tsmm<4><<<grid, 256, sm, stream>>>(n, kv, V, ldv, nc, H, alpha, beta, Out, ldo); break;
    case 8: k_tsmm<8><<<grid, 256, sm, stream>>>(n, kv, V, ldv, nc, H, alpha, beta, Out, ldo); break;
    case 16: k_tsmm<16><<<grid, 256, sm, stream>>>(n, kv, V, ldv, nc, H, alpha, beta, Out, ldo); break;
    default: k_tsmm<32><<<grid, 256, sm, stream>>>(n, kv, V, ldv, nc, H, alpha, beta, Out, ldo); break;
  }
  return cuda_status("pmp_tsmm");
}

size_t pmp_tsqr_workspace(int n, int nz) {
  int nb, chunk, sub;
  tsqr_geometry(n, nz, &nb, &chunk, &sub);
  int nbw = tsqr_warp_blocks(n);
  if (nbw > nb) nb = nbw;
  return 256 + sizeof(double) * (size_t)nb * nz * nz;
}

int pmp_tsqr_r(int n, int nz, const double* Z, int ldz, double* R, void* ws, size_t bytes,
               void* st) {
  if (n < 0 || nz < 1 || nz > 32 || ldz < nz) {
    set_error("pmp_tsqr_r: bad arguments (n=%d nz=%d)", n, nz);
    return PMP_ERR_ARG;
  }
  if (bytes < pmp_tsqr_workspace(n, nz)) {
    set_error("pmp_tsqr_r: workspace too small");
    return PMP_ERR_WORKSPACE;
  }
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(st);
  if (nz <= 16) {
    int nb = tsqr_warp_blocks(n);
    int chunk = ceil_div(n > 0 ? n : 1, nb);
    double* partial = (double*)((char*)ws + 256);
    if (nz <= 8)
      k_tsqr_warp<8><<<nb, 256, 0, stream>>>(n, nz, Z, ldz, chunk, partial, (unsigned*)ws, R);
    else
      k_tsqr_warp<16><<<nb, 256, 0, stream>>>(n, nz, Z, ldz, chunk, partial, (unsigned*)ws, R);
    return cuda_status("pmp_tsqr_r");
  }
  int nb, chunk, sub;
  tsqr_geometry(n, nz, &nb, &chunk, &sub);
  size_t sm = tsqr_smem(nz, sub);
  prepare_smem((const void*)k_tsqr, sm, kTsqrT);
  k_tsqr<<<nb, kTsqrT, sm, reinterpret_cast<cudaStream_t>(st)>>>(
      n, nz, Z, ldz, chunk, sub, (double*)((char*)ws + 256), (unsigned*)ws, R);
  return cuda_status("pmp_tsqr_r");
}

}  // extern "C"
