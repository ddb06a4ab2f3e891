// Device building blocks of the tall-skinny orthogonalisation kernels
// (k_orth / k_fold in orth.cu, the persistent cycle kernel in cycle.cu).
// The heavier ones are __noinline__ (operands by value): the persistent
// kernels call them several times per step, and inlined copies made the
// step loop (~25k instructions, 400 KB) overflow the SM's instruction cache
// -- every step then re-fetched its code from L2, ~700 cycles per 128-byte
// line (measured: the 8 x 8 Cholesky took 37k cycles in situ vs 9k alone).
// Every block owns a contiguous row range; reductions are two-stage
// (fixed-order per-block partials, then a distributed fixed-order sum)
// separated by grid barriers, so results are bitwise reproducible.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

#ifndef PMP_UPD_UNROLL
#define PMP_UPD_UNROLL 8
#endif
#ifndef PMP_GRAM_BATCH
#define PMP_GRAM_BATCH 8
#endif
#ifndef PMP_GRAM_INLINE
#define PMP_GRAM_INLINE __forceinline__
#endif

namespace pmp {

namespace cg = cooperative_groups;

constexpr int kOrthT = 256;
constexpr int kUpdUnroll = PMP_UPD_UNROLL;
constexpr double kCholRatio = 1e-5;
constexpr double kSkipKappa = 4.0;

// operand view of this block's rows: columns [0, ka) from a, then from b
struct Rows {
  const double* a;
  int lda, ka;
  const double* b;
  int ldb;
  __device__ __forceinline__ double at(int r, int t) const {
    return t < ka ? a[(size_t)r * lda + t] : b[(size_t)r * ldb + (t - ka)];
  }
};

__host__ __device__ __forceinline__ int odd_ld(int w) { return w | 1; }

// partial[b][t * ny + c] = sum over this block's rows of X(r, t) Y[r][c].
// Lanes own columns t (coalesced / conflict-free with odd leading
// dimensions), warps split the rows; the per-warp sums are combined in a
// fixed order through smem.
template <int NY>
__device__ PMP_GRAM_INLINE void block_gram(const Rows X, int kx, const double* Y, int ldy, int ny, int nrows,
                           double* red, double* partial, int slot = -1) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int K = kx * ny;
  double* part = partial + (size_t)(slot < 0 ? (int)blockIdx.x : slot) * K;
  const int rounds = (kx + 31) / 32;
  int splits = 8 / rounds;
  if (splits < 1) splits = 1;
  for (int job0 = 0; job0 < rounds * splits; job0 += 8) {
    const int job = job0 + wid;
    const int rd = job / splits, sp = job % splits;
    double acc[NY];
#pragma unroll
    for (int c = 0; c < NY; ++c) acc[c] = 0.0;
    const int t = rd * 32 + lane;
    if (job < rounds * splits && t < kx) {
      const int per = (nrows + splits - 1) / splits;
      const int ra = sp * per, rb = min(nrows, ra + per);
      // rows in batches of GB: the X loads of a batch are all in flight
      // before its FMAs (row order, hence the sums, unchanged)
      const double* xa = t < X.ka ? X.a + t : X.b + (t - X.ka);
      const int ldxr = t < X.ka ? X.lda : X.ldb;
      int r = ra;
      constexpr int GB = PMP_GRAM_BATCH;
      for (; r + GB <= rb; r += GB) {
        double x[GB];
#pragma unroll
        for (int u = 0; u < GB; ++u) x[u] = xa[(size_t)(r + u) * ldxr];
#pragma unroll
        for (int u = 0; u < GB; ++u) {
          const double* y = Y + (size_t)(r + u) * ldy;
#pragma unroll
          for (int c = 0; c < NY; ++c)
            if (c < ny) acc[c] += x[u] * y[c];
        }
      }
      for (; r < rb; ++r) {
        const double x = xa[(size_t)r * ldxr];
        const double* y = Y + (size_t)r * ldy;
#pragma unroll
        for (int c = 0; c < NY; ++c)
          if (c < ny) acc[c] += x * y[c];
      }
    }
    if (job < rounds * splits) {
#pragma unroll
      for (int c = 0; c < NY; ++c)
        if (c < ny) red[((size_t)(job - job0) * 32 + lane) * ny + c] = acc[c];
    }
    __syncthreads();
    // fixed-order sum over the splits of every round covered by this batch
    for (int o = threadIdx.x; o < K; o += kOrthT) {
      const int tt = o / ny, c = o % ny, r2 = tt / 32, ln = tt % 32;
      const int j0 = r2 * splits;
      if (j0 >= job0 && j0 < job0 + 8) {
        double s = 0.0;
        for (int q = 0; q < splits; ++q) s += red[((size_t)(j0 + q - job0) * 32 + ln) * ny + c];
        part[o] = s;
      }
    }
    __syncthreads();
  }
}

// The same product with the block's threads laid out flat over (row split,
// column): thread id -> column t = id % kx of split id / kx, 256 / kx splits
// of the rows.  block_gram gives each warp 32 columns of one round, so a
// last round of kx % 32 columns leaves most of its lanes idle (kx = 42: a
// third of the block's lanes); here every lane carries a column's row chain
// and 256 / kx > 8 / rounds splits keep more loads in flight.  Used by the
// global-row geometry (rows stream from HBM: the loads in flight bound the
// phase).  Fixed summation order (rows in order within a split, splits in
// order): deterministic, not bitwise equal to block_gram.  kx <= 128.
template <int NY>
__device__ __forceinline__ void block_gram_flat(const Rows X, int kx, const double* Y, int ldy,
                                                int ny, int nrows, double* red, double* partial,
                                                int slot) {
  const int K = kx * ny;
  double* part = partial + (size_t)slot * K;
  const int nsplit = kOrthT / kx;
  const int sp = threadIdx.x / kx, t = threadIdx.x - sp * kx;
  double acc[NY];
#pragma unroll
  for (int c = 0; c < NY; ++c) acc[c] = 0.0;
  if (sp < nsplit) {
    const int per = (nrows + nsplit - 1) / nsplit;
    const int ra = sp * per, rb = min(nrows, ra + per);
    const double* xa = t < X.ka ? X.a + t : X.b + (t - X.ka);
    const int ldxr = t < X.ka ? X.lda : X.ldb;
    int r = ra;
    constexpr int GB = PMP_GRAM_BATCH;
    for (; r + GB <= rb; r += GB) {
      double x[GB];
#pragma unroll
      for (int u = 0; u < GB; ++u) x[u] = xa[(size_t)(r + u) * ldxr];
#pragma unroll
      for (int u = 0; u < GB; ++u) {
        const double* y = Y + (size_t)(r + u) * ldy;
#pragma unroll
        for (int c = 0; c < NY; ++c)
          if (c < ny) acc[c] += x[u] * y[c];
      }
    }
    for (; r < rb; ++r) {
      const double x = xa[(size_t)r * ldxr];
      const double* y = Y + (size_t)r * ldy;
#pragma unroll
      for (int c = 0; c < NY; ++c)
        if (c < ny) acc[c] += x * y[c];
    }
#pragma unroll
    for (int c = 0; c < NY; ++c)
      if (c < ny) red[(size_t)threadIdx.x * ny + c] = acc[c];
  }
  __syncthreads();
  for (int o = threadIdx.x; o < K; o += kOrthT) {
    double s = 0.0;
    for (int q = 0; q < nsplit; ++q) s += red[(size_t)q * K + o];
    part[o] = s;
  }
  __syncthreads();
}

// distributed fixed-order reduction of the block partials; every block ends
// with the full K-vector in smem G.  Entries [0, split) are also copied to
// out, entries [split, K) to out2 (either may be null).
static __device__ __noinline__ void grid_reduce(cg::grid_group& grid, double* partial, double* gout, int K,
                            double* G,
                            double* out, int split, double* out2) {
  __threadfence();
  grid.sync();
  const int nb = gridDim.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = blockIdx.x + nb * wid; o < K; o += nb * (kOrthT / 32)) {
    double s = 0.0;
    if (nb <= 512) {
      // every load in flight at once (one L2 round trip), then the same
      // fixed-order sum as below: t0 over even, t1 over odd strides of 32
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int b = lane + 32 * u;
        v[u] = b < nb ? __ldcg(partial + (size_t)b * K + o) : 0.0;
      }
      double t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int u = 0; u < 16; u += 2) {
        t0 += v[u];
        t1 += v[u + 1];
      }
      s = t0 + t1;
    } else {
      double t0 = 0.0, t1 = 0.0;
      int b = lane;
      for (; b + 32 < nb; b += 64) {
        t0 += __ldcg(partial + (size_t)b * K + o);
        t1 += __ldcg(partial + (size_t)(b + 32) * K + o);
      }
      if (b < nb) t0 += __ldcg(partial + (size_t)b * K + o);
      s = t0 + t1;
    }
    s = warp_sum(s);
    if (lane == 0) {
      gout[o] = s;
      if (o < split) {
        if (out) out[o] = s;
      } else if (out2) {
        out2[o - split] = s;
      }
    }
  }
  __threadfence();
  grid.sync();
  for (int o = threadIdx.x; o < K; o += kOrthT) G[o] = __ldcg(gout + o);
  __syncthreads();
}

// Y[r][c] -= sum_t X(r, t) G[t][c] ; thread per row, all ny outputs
template <int NY>
__device__ PMP_GRAM_INLINE void block_update(const Rows X, int kx, double* Y, int ldy, int ny, int nrows,
                             const double* G) {
  const int ka = min(kx, X.ka);
  for (int r = threadIdx.x; r < nrows; r += kOrthT) {
    double acc[NY];
#pragma unroll
    for (int c = 0; c < NY; ++c) acc[c] = 0.0;
    // the two column segments separately (no per-element branch), unrolled
    // so several row loads are in flight
    const double* xa = X.a + (size_t)r * X.lda;
#pragma unroll kUpdUnroll
    for (int t = 0; t < ka; ++t) {
      const double x = xa[t];
      const double* g = G + t * ny;
#pragma unroll
      for (int c = 0; c < NY; ++c)
        if (c < ny) acc[c] += x * g[c];
    }
    const double* xb = X.b + (size_t)r * X.ldb - X.ka;
#pragma unroll kUpdUnroll
    for (int t = ka; t < kx; ++t) {
      const double x = xb[t];
      const double* g = G + t * ny;
#pragma unroll
      for (int c = 0; c < NY; ++c)
        if (c < ny) acc[c] += x * g[c];
    }
    double* y = Y + (size_t)r * ldy;
#pragma unroll
    for (int c = 0; c < NY; ++c)
      if (c < ny) y[c] -= acc[c];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// FP64 tensor-core (DMMA m8n8k4) forms of the two tall-skinny products of the
// block step.  The point is the memory access, not the flops: a fragment load
// of the A operand touches 8 rows x 32 B (update) or 4 rows x 64 B (Gram) --
// whole sectors, every byte used -- where the thread-per-row update had each
// warp-wide load hit 32 different rows, 8 of 32 bytes used per sector and
// the rest left to an L1 that the kernel's shared memory squeezes to a few
// tens of KB (ncu: 35 % excess sectors).  Fragment layout (PTX ISA, .f64
// m8n8k4): g = lane >> 2, t = lane & 3; A[g][t], B[t][g], C/D[g][2t + i].
// Fixed summation order (4-term chunks in row / column order): bitwise
// reproducible run to run.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Y[r][c] -= sum_t X(r, t) G[t][c] (G row-major ld ny, shared memory): one
// warp per 8-row block, ALL kx columns of the block's rows streamed as
// 8 x 4 A fragments (four in flight), G as B fragments.
template <int NY>
__device__ __noinline__ void block_update_mma(const Rows X, int kx, double* Y, int ldy, int ny,
                                              int nrows, const double* G) {
  constexpr int NH = (NY + 7) / 8;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int nch = (kx + 3) >> 2;
  for (int rb = wid * 8; rb < nrows; rb += (kOrthT / 32) * 8) {
    const int r = rb + g;
    const bool rok = r < nrows;
    const double* xa = X.a + (size_t)(rok ? r : 0) * X.lda;
    const double* xb = X.b + (size_t)(rok ? r : 0) * X.ldb - X.ka;
    double acc[NH][2];
#pragma unroll
    for (int h = 0; h < NH; ++h) acc[h][0] = acc[h][1] = 0.0;
    for (int ch = 0; ch < nch; ch += 4) {
      double a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = (ch + u) * 4 + t4;
        a[u] = (rok && t < kx) ? (t < X.ka ? xa[t] : xb[t]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (ch + u >= nch) break;  // warp-uniform
        const int t = (ch + u) * 4 + t4;
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int c = h * 8 + g;
          const double b = (t < kx && c < ny) ? G[t * ny + c] : 0.0;
          dmma884(acc[h], a[u], b);
        }
      }
    }
    if (rok) {
      double* y = Y + (size_t)r * ldy;
#pragma unroll
      for (int h = 0; h < NH; ++h)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int c = h * 8 + 2 * t4 + i;
          if (c < ny) y[c] -= acc[h][i];
        }
    }
  }
  __syncthreads();
}

// partial[slot][t * ny + c] = sum over this block's rows of X(r, t) Y[r][c]:
// jobs = (8-column tile of X, row split); one warp per job, 4 x 4 rows per
// round of fragments; splits summed in a fixed order through `red`
// (>= 512 * NH doubles).
template <int NY>
__device__ __noinline__ void block_gram_mma(const Rows X, int kx, const double* Y, int ldy, int ny,
                                            int nrows, double* red, double* partial, int slot) {
  constexpr int NH = (NY + 7) / 8;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int K = kx * ny;
  double* part = partial + (size_t)slot * K;
  const int ntile = (kx + 7) >> 3;
  int splits = (kOrthT / 32) / ntile;
  if (splits < 1) splits = 1;
  const int njobs = ntile * splits;
  const int per = ((nrows + splits - 1) / splits + 3) & ~3;
  for (int j0 = 0; j0 < njobs; j0 += kOrthT / 32) {
    const int job = j0 + wid;
    double acc[NH][2];
#pragma unroll
    for (int h = 0; h < NH; ++h) acc[h][0] = acc[h][1] = 0.0;
    if (job < njobs) {  // warp-uniform
      const int tile = job / splits, sp = job % splits;
      const int ra = sp * per, rb = min(nrows, ra + per);
      const int t = tile * 8 + g;
      const bool tok = t < kx;
      const double* xcol = tok ? (t < X.ka ? X.a + t : X.b + (t - X.ka)) : X.a;
      const int ldxc = (tok && t >= X.ka) ? X.ldb : X.lda;
      for (int r0 = ra; r0 < rb; r0 += 16) {
        double a[4], b[NH][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = r0 + 4 * u + t4;
          const bool ok = r < rb;
          a[u] = (ok && tok) ? xcol[(size_t)r * ldxc] : 0.0;
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const int c = h * 8 + g;
            b[h][u] = (ok && c < ny) ? Y[(size_t)r * ldy + c] : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int h = 0; h < NH; ++h) dmma884(acc[h], a[u], b[h][u]);
      }
    }
    if (job < njobs) {
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        red[((size_t)(job - j0) * NH + h) * 64 + g * 8 + 2 * t4] = acc[h][0];
        red[((size_t)(job - j0) * NH + h) * 64 + g * 8 + 2 * t4 + 1] = acc[h][1];
      }
    }
    __syncthreads();
    // fixed-order sum over the splits of the tiles finished in this round
    const int tile_lo = j0 / splits, tile_hi = min(ntile, (j0 + kOrthT / 32) / splits);
    const int nout = (tile_hi - tile_lo) * 8 * ny;
    for (int o = threadIdx.x; o < nout; o += kOrthT) {
      const int tl = o / (8 * ny), rem = o % (8 * ny);
      const int tt = rem / ny, c = rem % ny;
      const int tile = tile_lo + tl, t = tile * 8 + tt;
      if (t < kx) {
        double s = 0.0;
        for (int q = 0; q < splits; ++q) {
          const int jj = tile * splits + q - j0;
          s += red[((size_t)jj * NH + c / 8) * 64 + tt * 8 + (c % 8)];
        }
        part[t * ny + c] = s;
      }
    }
    __syncthreads();
  }
}

// Pivoted Cholesky of the m x m SPD matrix A (row-major, shared memory,
// destroyed) by one warp with rolled loops: lane i owns row i.  R (row-major,
// upper) is the factor of P^T A P, piv the permutation.  Small code on
// purpose: the persistent cycle kernel runs it once per block step, and
// the fully unrolled register version is large enough to miss in the
// instruction cache every time.  Returns ok (all pivots positive and the
// last >= ratio x the first).
static __device__ __noinline__ bool warp_cholesky_smem(double* A, int m, double* R, int* piv, bool pivot,
                                                double ratio) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  if (lane < m) piv[lane] = lane;
  for (int q = lane; q < m * m; q += 32) R[q] = 0.0;
  __syncwarp();
  bool ok = true;
  double r00 = 0.0;
  for (int k = 0; k < m; ++k) {
    int p = k;
    if (pivot) {
      // packed (diagonal bits, 31 - lane) key: ties within 32 ulp go to the
      // lowest row; a negative diagonal counts as 0 (a failing pivot)
      long long key = (lane >= k && lane < m)
                          ? ((__double_as_longlong(fmax(A[lane * m + lane], 0.0)) & ~31LL) |
                             (31 - lane))
                          : -1LL;
      for (int o = 16; o > 0; o >>= 1) {
        const long long other = __shfl_xor_sync(full, key, o);
        key = other > key ? other : key;
      }
      p = 31 - (int)(key & 31);
    }
    if (p != k) {
      if (lane < m) {
        const double t = A[k * m + lane];
        A[k * m + lane] = A[p * m + lane];
        A[p * m + lane] = t;
      }
      __syncwarp();
      if (lane < m) {
        const double t = A[lane * m + k];
        A[lane * m + k] = A[lane * m + p];
        A[lane * m + p] = t;
      }
      if (lane < k) {
        const double t = R[lane * m + k];
        R[lane * m + k] = R[lane * m + p];
        R[lane * m + p] = t;
      }
      if (lane == 0) {
        const int t = piv[k];
        piv[k] = piv[p];
        piv[p] = t;
      }
      __syncwarp();
    }
    const double dkk = A[k * m + k];
    if (!(dkk > 0.0)) {
      ok = false;
      break;
    }
    const double inv = rsqrt(dkk);
    const double rkk = dkk * inv;
    if (k == 0) r00 = rkk;
    if (lane >= k && lane < m) R[k * m + lane] = lane == k ? rkk : A[k * m + lane] * inv;
    __syncwarp();
    if (lane > k && lane < m) {
      const double ri = R[k * m + lane];
      for (int c = k + 1; c < m; ++c) A[lane * m + c] -= ri * R[k * m + c];
    }
    __syncwarp();
  }
  if (ok && m > 0) ok = fabs(R[(m - 1) * m + (m - 1)]) > ratio * r00;
  __syncwarp();
  return ok;
}

// Same factorisation held in registers: lane i owns row i (m <= NY <= 32),
// pivot search by a warp arg-max, row swaps by shuffles, column swaps by
// register selects -- no shared-memory round trips or __syncwarp chains.
template <int NY>
__device__ __noinline__ bool warp_cholesky_reg(const double* G, int m, double* R, int* piv, bool pivot,
                                  double ratio) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double a[NY];
#pragma unroll
  for (int c = 0; c < NY; ++c) a[c] = (lane < m && c < m) ? G[lane * m + c] : 0.0;
  int pv = lane;
  bool ok = true;
  double r00 = 0.0;
#pragma unroll
  for (int k = 0; k < NY; ++k) {
    if (k >= m) break;
    int p = k;
    if (pivot) {
      double dii = 0.0;
#pragma unroll
      for (int c = 0; c < NY; ++c)
        if (c == lane) dii = a[c];
      // arg-max as one 64-bit key: the diagonal's bits (order-preserving for
      // non-negative doubles) with the low 5 mantissa bits replaced by
      // 31 - lane, so (near-)ties within 32 ulp go to the lowest lane
      // (a negative diagonal counts as 0: still a valid, failing pivot;
      // lanes outside [k, m) get key -1, below every valid key)
      long long key = (lane >= k && lane < m)
                          ? ((__double_as_longlong(fmax(dii, 0.0)) & ~31LL) | (31 - lane))
                          : -1LL;
#pragma unroll
      for (int o = NY / 2; o > 0; o >>= 1) {
        const long long ok = __shfl_xor_sync(full, key, o);
        key = ok > key ? ok : key;
      }
      // lanes >= NY reduced their own group: take lane 0's (warp-uniform)
      p = 31 - (int)(__shfl_sync(full, key, 0) & 31);
    }
    if (p != k) {
      const int src = lane == k ? p : (lane == p ? k : lane);
#pragma unroll
      for (int c = 0; c < NY; ++c) a[c] = __shfl_sync(full, a[c], src);
      pv = __shfl_sync(full, pv, src);
      double ap = 0.0;
#pragma unroll
      for (int c = 0; c < NY; ++c)
        if (c == p) ap = a[c];
      const double ak = a[k];
#pragma unroll
      for (int c = 0; c < NY; ++c)
        if (c == p) a[c] = ak;
      a[k] = ap;
    }
    const double dkk = __shfl_sync(full, a[k], k);
    if (!(dkk > 0.0)) {
      ok = false;
      break;
    }
    const double inv = rsqrt(dkk);
    const double rkk = dkk * inv;
    if (k == 0) r00 = rkk;
    if (lane == k) {
#pragma unroll
      for (int c = 0; c < NY; ++c)
        if (c > k) a[c] *= inv;
      a[k] = rkk;
    }
    double rk[NY];
#pragma unroll
    for (int c = 0; c < NY; ++c) rk[c] = __shfl_sync(full, a[c], k);
    double mine = 0.0;
#pragma unroll
    for (int c = 0; c < NY; ++c)
      if (c == lane) mine = rk[c];
    if (lane > k && lane < m) {
#pragma unroll
      for (int c = 0; c < NY; ++c)
        if (c > k) a[c] -= mine * rk[c];
    }
  }
  if (ok && m > 0) {
    double dl = 0.0;
#pragma unroll
    for (int c = 0; c < NY; ++c)
      if (c == lane) dl = a[c];
    dl = __shfl_sync(full, dl, m - 1);
    ok = fabs(dl) > ratio * r00;
  }
  if (lane < m) {
#pragma unroll
    for (int c = 0; c < NY; ++c)
      if (c < m) R[lane * m + c] = (c >= lane) ? a[c] : 0.0;
    piv[lane] = pv;
  }
  __syncwarp();
  return ok;
}

// Y[r][:] = X[r][piv] R^-1 (row-vector triangular solve); thread per row
template <int NY>
__device__ __noinline__ void block_trsm_rows(const double* X, int ldx, double* Y, int ldy, int nrows, int m,
                                const double* R, const int* piv) {
  __shared__ double rinv[16];
  if (threadIdx.x < m) rinv[threadIdx.x] = 1.0 / R[threadIdx.x * m + threadIdx.x];
  __syncthreads();
  for (int r = threadIdx.x; r < nrows; r += kOrthT) {
    double x[NY], y[NY];
#pragma unroll
    for (int c = 0; c < NY; ++c) x[c] = (c < m) ? X[(size_t)r * ldx + (piv ? piv[c] : c)] : 0.0;
#pragma unroll
    for (int c = 0; c < NY; ++c) {
      if (c < m) {
        double s = x[c];
#pragma unroll
        for (int a = 0; a < NY; ++a)
          if (a < c) s -= y[a] * R[a * m + c];
        y[c] = s * rinv[c];
      } else {
        y[c] = 0.0;
      }
    }
#pragma unroll
    for (int c = 0; c < NY; ++c)
      if (c < m) Y[(size_t)r * ldy + c] = y[c];
  }
  __syncthreads();
}

// block_update and block_trsm_rows in one pass over the rows (thread per
// row): y = Y[r] - X(r, :) G, then Q[r] = y[piv] R^-1 written to Qd; Y is not
// written back.  For the block step whose Cholesky-QR needs a single pass:
// W2 = W1 - V H2 is consumed where it is produced, so W2 is neither stored
// nor read again (one pass over the block's W rows and one barrier-free
// sweep less per step).  Same arithmetic as the two functions in sequence.
template <int NY>
__device__ __forceinline__ void block_update_trsm(const Rows X, int kx, const double* Y, int ldy,
                                                  int ny, int nrows, const double* G,
                                                  const double* R, const int* piv, double* Qd,
                                                  int ldq) {
  __shared__ double rinv_f[16];
  __shared__ int piv_f[16];
  if (threadIdx.x < ny) {
    rinv_f[threadIdx.x] = 1.0 / R[threadIdx.x * ny + threadIdx.x];
    piv_f[threadIdx.x] = piv[threadIdx.x];
  }
  __syncthreads();
  const int ka = min(kx, X.ka);
  for (int r = threadIdx.x; r < nrows; r += kOrthT) {
    double acc[NY];
#pragma unroll
    for (int c = 0; c < NY; ++c) acc[c] = 0.0;
    const double* xa = X.a + (size_t)r * X.lda;
#pragma unroll kUpdUnroll
    for (int t = 0; t < ka; ++t) {
      const double x = xa[t];
      const double* g = G + t * ny;
#pragma unroll
      for (int c = 0; c < NY; ++c)
        if (c < ny) acc[c] += x * g[c];
    }
    const double* xb = X.b + (size_t)r * X.ldb - X.ka;
#pragma unroll kUpdUnroll
    for (int t = ka; t < kx; ++t) {
      const double x = xb[t];
      const double* g = G + t * ny;
#pragma unroll
      for (int c = 0; c < NY; ++c)
        if (c < ny) acc[c] += x * g[c];
    }
    const double* y = Y + (size_t)r * ldy;
    double w2[NY];
#pragma unroll
    for (int c = 0; c < NY; ++c) w2[c] = (c < ny) ? y[c] - acc[c] : 0.0;
    // q = w2[piv] R^-1 (row-vector triangular solve, as block_trsm_rows)
    double xq[NY], q[NY];
#pragma unroll
    for (int c = 0; c < NY; ++c) {
      double v = 0.0;
      if (c < ny) {
        const int pc = piv_f[c];
#pragma unroll
        for (int a = 0; a < NY; ++a)
          if (a == pc) v = w2[a];
      }
      xq[c] = v;
    }
#pragma unroll
    for (int c = 0; c < NY; ++c) {
      if (c < ny) {
        double sv = xq[c];
#pragma unroll
        for (int a = 0; a < NY; ++a)
          if (a < c) sv -= q[a] * R[a * ny + c];
        q[c] = sv * rinv_f[c];
      } else {
        q[c] = 0.0;
      }
    }
    double* qo = Qd + (size_t)r * ldq;
#pragma unroll
    for (int c = 0; c < NY; ++c)
      if (c < ny) qo[c] = q[c];
  }
  __syncthreads();
}

// cooperative launch of kOrthT-thread blocks, routed through the shared
// cooperative stream when one is set (orth.cu, pmp_set_coop_stream)
cudaError_t coop_launch(const void* fn, int g, void** args, size_t smem, cudaStream_t user);
// 2 x #SMs (the largest co-resident grid the kernels here use)
int orth_max_grid();

}  // namespace pmp
