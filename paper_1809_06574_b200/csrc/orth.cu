// Kernel 5b+5c fused: one block-Arnoldi orthogonalisation step of block GCRO
// (krylov.py:189-202) in ONE cooperative launch.
//
//   W  -= C (C^T W)                         outer-space projection  :189-192
//   2x { H = V^T W ; W -= V H }             block CGS2              :193-196
//   W = Q R                                 _qr_deflate             :197-202
//
// The reference runs these as separate BLAS/LAPACK calls; on the device
// each is a tall-skinny reduction whose cost at BASELINE sizes is latency,
// not bandwidth.  Here every block owns a contiguous row range, keeps its
// rows of V, C and W in shared memory when they fit (c2: 222 rows x 86
// columns = 153 KB), and the reductions are two-stage (per-block partials,
// then a distributed fixed-order reduction) separated by grid-wide
// barriers, so HBM/L2 is touched once per operand and no host round trip
// is needed between the passes.
//
// The QR is Cholesky-QR2 with symmetric pivoting: G = W^T W, R1 = chol(G),
// Q1 = W P R1^-1, R2 = chol(Q1^T Q1), Q = Q1 R2^-1, R = R2 R1 (un-pivoted).
// When the pivoted Cholesky shows min |R_kk| / |R_00| <= 1e-5 the block is
// too close to rank deficiency for Cholesky to decide the 1e-12 deflation
// rank of the reference (krylov.py:92); the kernel then leaves the
// projected W in global memory and raises a flag, and the host falls back
// to Householder TSQR + pivoted QR (pmp_tsqr_r + pmp_host_deflate), which
// reproduce geqp3's rank decision.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace pmp {

constexpr int kOrthT = 256;
constexpr double kCholRatio = 1e-5;

struct OrthParams {
  int n;
  const double* C;
  int ldc, k;
  double* V;
  int ldv, total, npass;
  double* W;
  int ldw, sb;
  int qout;            // V column receiving the new orthonormal block
  int rows_per_block;
  int cached;
  double* partial;     // gridDim.x * kmax doubles
  double* Q1;          // n x sb scratch (streaming mode)
  double* gout;        // reduction results (global): kmax doubles
  double* outB;        // k x sb      (C^T W)
  double* outH1;       // total x sb  (first CGS pass)
  double* outH2;       // total x sb  (second CGS pass)
  double* outR;        // sb x sb     (R, un-pivoted, row-major)
  double* outFlag;     // 1 double: 0 ok, 1 fallback needed
};

struct OrthSmem {
  double* Vs;  // rows x total   (cached mode)
  double* Cs;  // rows x k
  double* Ws;  // rows x sb
  double* Qs;  // rows x sb
  double* G;   // kmax  (reduced matrix)
  double* A;   // 16 x 16 Cholesky work
  double* R1;  // 16 x 16
  double* R2;  // 16 x 16
  int* piv;    // 16
  int* piv2;   // 16
  int* flag;   // 2
};

// partial[b][o] = sum over this block's rows of X[r][t] Y[r][c], o = t*ny + c
__device__ inline void block_gram(const double* X, int ldx, int kx, const double* Y, int ldy, int ny,
                                  int nrows, double* partial) {
  const int K = kx * ny;
  double* part = partial + (size_t)blockIdx.x * K;
  for (int o = threadIdx.x; o < K; o += kOrthT) {
    const int t = o / ny, c = o % ny;
    double a0 = 0.0, a1 = 0.0;
    int r = 0;
    for (; r + 1 < nrows; r += 2) {
      a0 += X[(size_t)r * ldx + t] * Y[(size_t)r * ldy + c];
      a1 += X[(size_t)(r + 1) * ldx + t] * Y[(size_t)(r + 1) * ldy + c];
    }
    if (r < nrows) a0 += X[(size_t)r * ldx + t] * Y[(size_t)r * ldy + c];
    part[o] = a0 + a1;
  }
}

// fixed-order distributed reduction of the block partials; every block
// ends with the full result in smem G (and block 0's slice writes `out`)
__device__ inline void grid_reduce(cg::grid_group& grid, const OrthParams& P, int K, double* G,
                                   double* out) {
  __threadfence();
  grid.sync();
  const int nb = gridDim.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = blockIdx.x + nb * wid; o < K; o += nb * (kOrthT / 32)) {
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += __ldcg(P.partial + (size_t)b * K + o);
    s = warp_sum(s);
    if (lane == 0) {
      P.gout[o] = s;
      if (out) out[o] = s;
    }
  }
  __threadfence();
  grid.sync();
  for (int o = threadIdx.x; o < K; o += kOrthT) G[o] = __ldcg(P.gout + o);
  __syncthreads();
}

// Y[r][c] -= sum_t X[r][t] G[t][c]
__device__ inline void block_update(const double* X, int ldx, int kx, double* Y, int ldy, int ny,
                                    int nrows, const double* G) {
  for (int q = threadIdx.x; q < nrows * ny; q += kOrthT) {
    const int r = q / ny, c = q % ny;
    const double* x = X + (size_t)r * ldx;
    double a0 = 0.0, a1 = 0.0;
    int t = 0;
    for (; t + 1 < kx; t += 2) {
      a0 += x[t] * G[t * ny + c];
      a1 += x[t + 1] * G[(t + 1) * ny + c];
    }
    if (t < kx) a0 += x[t] * G[t * ny + c];
    Y[(size_t)r * ldy + c] -= a0 + a1;
  }
  __syncthreads();
}

// Cholesky of the m x m SPD matrix in G (row-major), by warp 0.  With
// pivot != 0, symmetric pivoting on the largest remaining diagonal.
// R (m x m, row-major, upper) gets the factor of P^T G P; returns ok.
__device__ inline bool warp_cholesky(const double* G, int m, double* A, double* R, int* piv,
                                     bool pivot, double ratio) {
  const int lane = threadIdx.x & 31;
  for (int q = lane; q < m * m; q += 32) {
    A[q] = G[q];
    R[q] = 0.0;
  }
  if (lane < m) piv[lane] = lane;
  __syncwarp();
  bool ok = true;
  for (int k = 0; k < m; ++k) {
    int p = k;
    if (pivot) {
      double best = A[k * m + k];
      for (int j = k + 1; j < m; ++j)
        if (A[j * m + j] > best) {
          best = A[j * m + j];
          p = j;
        }
    }
    if (p != k) {
      // symmetric swap of rows/columns k and p of the trailing matrix, and
      // of the already computed R columns
      for (int q = lane; q < m; q += 32) {
        double t = A[k * m + q];
        A[k * m + q] = A[p * m + q];
        A[p * m + q] = t;
      }
      __syncwarp();
      for (int q = lane; q < m; q += 32) {
        double t = A[q * m + k];
        A[q * m + k] = A[q * m + p];
        A[q * m + p] = t;
      }
      for (int q = lane; q < k; q += 32) {
        double t = R[q * m + k];
        R[q * m + k] = R[q * m + p];
        R[q * m + p] = t;
      }
      if (lane == 0) {
        int t = piv[k];
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
    const double d = sqrt(dkk);
    for (int j = k + lane; j < m; j += 32) R[k * m + j] = (j == k) ? d : A[k * m + j] / d;
    __syncwarp();
    for (int q = lane; q < (m - k - 1) * (m - k - 1); q += 32) {
      int i = k + 1 + q / (m - k - 1), j = k + 1 + q % (m - k - 1);
      A[i * m + j] -= R[k * m + i] * R[k * m + j];
    }
    __syncwarp();
  }
  if (ok && m > 0) ok = fabs(R[(m - 1) * m + (m - 1)]) > ratio * fabs(R[0]);
  return ok;
}

// Y[r][:] = X[r][piv] R^-1 (row-vector triangular solve), in place allowed
__device__ inline void block_trsm_rows(const double* X, int ldx, double* Y, int ldy, int nrows,
                                       int m, const double* R, const int* piv) {
  for (int r = threadIdx.x; r < nrows; r += kOrthT) {
    double x[16], y[16];
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c < m) x[c] = X[(size_t)r * ldx + (piv ? piv[c] : c)];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      if (c >= m) break;
      double s = x[c];
#pragma unroll
      for (int a = 0; a < 16; ++a)
        if (a < c) s -= y[a] * R[a * m + c];
      y[c] = s / R[c * m + c];
    }
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c < m) Y[(size_t)r * ldy + c] = y[c];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kOrthT, 1) k_orth(OrthParams P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sh[];
  const int r0 = blockIdx.x * P.rows_per_block;
  const int r1 = min(P.n, r0 + P.rows_per_block);
  const int nr = max(0, r1 - r0);
  const int sb = P.sb, k = P.k, tot = P.total;
  const int kmax = max(max(k, tot), sb) * sb;
  OrthSmem S;
  double* p = sh;
  S.G = p;
  p += kmax;
  S.A = p;
  p += 256;
  S.R1 = p;
  p += 256;
  S.R2 = p;
  p += 256;
  S.piv = reinterpret_cast<int*>(p);
  S.piv2 = S.piv + 16;
  p += 16;
  S.flag = reinterpret_cast<int*>(p);
  p += 4;
  // operand views: shared-memory copies of this block's rows, or global
  const double *Cv = P.C + (size_t)r0 * P.ldc, *Vv = P.V + (size_t)r0 * P.ldv;
  double* Wv = P.W + (size_t)r0 * P.ldw;
  int ldc = P.ldc, ldv = P.ldv, ldw = P.ldw;
  if (P.cached) {
    S.Vs = p;
    p += (size_t)nr * tot;
    S.Cs = p;
    p += (size_t)nr * k;
    S.Ws = p;
    p += (size_t)nr * sb;
    S.Qs = p;
    for (int q = threadIdx.x; q < nr * tot; q += kOrthT)
      S.Vs[q] = Vv[(size_t)(q / tot) * P.ldv + q % tot];
    for (int q = threadIdx.x; q < nr * k; q += kOrthT)
      S.Cs[q] = Cv[(size_t)(q / k) * P.ldc + q % k];
    for (int q = threadIdx.x; q < nr * sb; q += kOrthT)
      S.Ws[q] = Wv[(size_t)(q / sb) * P.ldw + q % sb];
    __syncthreads();
    Vv = S.Vs;
    Cv = S.Cs;
    Wv = S.Ws;
    ldv = tot;
    ldc = k;
    ldw = sb;
  }
  double* part = P.partial;

  // ---- W -= C (C^T W) --------------------------------------------------------
  if (k > 0) {
    block_gram(Cv, ldc, k, Wv, ldw, sb, nr, part);
    grid_reduce(grid, P, k * sb, S.G, P.outB);
    block_update(Cv, ldc, k, Wv, ldw, sb, nr, S.G);
  }
  // ---- block CGS2 against V[:, :total] -----------------------------------------
  for (int pass = 0; pass < P.npass && tot > 0; ++pass) {
    // same fixed-order reduction structure for both passes
    block_gram(Vv, ldv, tot, Wv, ldw, sb, nr, part);
    grid_reduce(grid, P, tot * sb, S.G, pass == 0 ? P.outH1 : P.outH2);
    block_update(Vv, ldv, tot, Wv, ldw, sb, nr, S.G);
  }
  // ---- Cholesky-QR2 -------------------------------------------------------------
  block_gram(Wv, ldw, sb, Wv, ldw, sb, nr, part);
  grid_reduce(grid, P, sb * sb, S.G, nullptr);
  if (threadIdx.x < 32) {
    bool ok = warp_cholesky(S.G, sb, S.A, S.R1, S.piv, true, kCholRatio);
    if (threadIdx.x == 0) S.flag[0] = ok ? 0 : 1;
  }
  __syncthreads();
  // Q1 = W P R1^-1 into a separate view, so W stays intact for a fallback
  double* Q1 = P.cached ? S.Qs : (P.Q1 + (size_t)r0 * sb);
  if (!S.flag[0]) {
    block_trsm_rows(Wv, ldw, Q1, sb, nr, sb, S.R1, S.piv);
    block_gram(Q1, sb, sb, Q1, sb, sb, nr, part);
  }
  // the flag is grid-uniform (every block factors the same reduced G), so
  // this reduction is reached by all blocks or by none
  if (!S.flag[0]) {
    grid_reduce(grid, P, sb * sb, S.G, nullptr);
    if (threadIdx.x < 32) {
      bool ok = warp_cholesky(S.G, sb, S.A, S.R2, S.piv2, false, 0.0);
      if (threadIdx.x == 0) S.flag[0] = ok ? 0 : 1;
    }
    __syncthreads();
  }
  if (S.flag[0]) {
    // fallback: leave the projected block in global W for the host path
    if (P.cached)
      for (int q = threadIdx.x; q < nr * sb; q += kOrthT)
        P.W[(size_t)(r0 + q / sb) * P.ldw + q % sb] = Wv[q];
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.outFlag = 1.0;
    return;
  }
  // Q = Q1 R2^-1 -> V[:, qout : qout + sb]
  block_trsm_rows(Q1, sb, P.V + (size_t)r0 * P.ldv + P.qout, P.ldv, nr, sb, S.R2, nullptr);
  if (blockIdx.x == 0) {
    // R = R2 R1 (pivoted column order), un-pivoted: Rout[i, piv[c]] = R[i, c]
    for (int q = threadIdx.x; q < sb * sb; q += kOrthT) {
      const int i = q / sb, c = q % sb;
      double s = 0.0;
      for (int a = i; a <= c; ++a) s += S.R2[i * sb + a] * S.R1[a * sb + c];
      P.outR[i * sb + S.piv[c]] = (c >= i) ? s : 0.0;
    }
    if (threadIdx.x == 0) *P.outFlag = 0.0;
  }
}

size_t orth_smem_bytes(int rows, int total, int k, int sb, int cached) {
  const int kmax = (k > total ? (k > sb ? k : sb) : (total > sb ? total : sb)) * sb;
  size_t d = (size_t)kmax + 3 * 256 + 16 + 16 + 4;
  if (cached) d += (size_t)rows * (total + k + 2 * sb);
  return d * sizeof(double);
}

}  // namespace pmp

using namespace pmp;

static int orth_geometry(int n, int total, int k, int sb, int* grid, int* rows, int* cached,
                         size_t* smem) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  int g = sms;
  int want = (n + 31) / 32;
  if (want < g) g = want > 0 ? want : 1;
  int r = (n + g - 1) / g;
  size_t full = orth_smem_bytes(r, total, k, sb, 1);
  *cached = full <= (size_t)200 * 1024;
  *smem = *cached ? full : orth_smem_bytes(r, total, k, sb, 0);
  *grid = g;
  *rows = r;
  return 0;
}

extern "C" {

size_t pmp_orth_workspace(int n, int total_max, int k_max, int sb) {
  int g, r, c;
  size_t sm;
  orth_geometry(n, total_max, k_max, sb, &g, &r, &c, &sm);
  const int kmax = (k_max > total_max ? (k_max > sb ? k_max : sb)
                                      : (total_max > sb ? total_max : sb)) * sb;
  return 256 + sizeof(double) * ((size_t)g * kmax + kmax + (size_t)n * sb + 64);
}

int pmp_orth_step(int n, const double* C, int ldc, int k, double* V, int ldv, int total, int npass,
                  double* W, int ldw, int sb, int qout, double* outB, double* outH1,
                  double* outH2, double* outR, double* outFlag, void* ws, size_t ws_bytes,
                  void* stream) {
  if (n < 1 || sb < 1 || sb > 16 || k < 0 || total < 0 || (k && ldc < k) || ldw < sb ||
      ldv < qout + sb || (npass && total && ldv < total)) {
    set_error("pmp_orth_step: bad arguments (n=%d k=%d total=%d sb=%d)", n, k, total, sb);
    return PMP_ERR_ARG;
  }
  if (ws_bytes < pmp_orth_workspace(n, total, k, sb)) {
    set_error("pmp_orth_step: workspace too small");
    return PMP_ERR_WORKSPACE;
  }
  int g, rows, cached;
  size_t smem;
  orth_geometry(n, total, k, sb, &g, &rows, &cached, &smem);
  cudaFuncSetAttribute(k_orth, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bps = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_orth, kOrthT, smem);
  if (bps < 1) {
    set_error("pmp_orth_step: kernel does not fit on an SM (smem %zu)", smem);
    return PMP_ERR_ARG;
  }
  const int kmax = (k > total ? (k > sb ? k : sb) : (total > sb ? total : sb)) * sb;
  OrthParams P;
  P.n = n;
  P.C = C;
  P.ldc = ldc;
  P.k = k;
  P.V = V;
  P.ldv = ldv;
  P.total = total;
  P.npass = npass;
  P.W = W;
  P.ldw = ldw;
  P.sb = sb;
  P.qout = qout;
  P.rows_per_block = rows;
  P.cached = cached;
  double* w = (double*)((char*)ws + 256);
  P.partial = w;
  P.gout = w + (size_t)g * kmax;
  P.Q1 = P.gout + kmax;
  P.outB = outB;
  P.outH1 = outH1;
  P.outH2 = outH2;
  P.outR = outR;
  P.outFlag = outFlag;
  void* args[] = {&P};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)k_orth, dim3(g), dim3(kOrthT), args, smem,
                                              reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    set_error("pmp_orth_step: %s", cudaGetErrorString(e));
    return PMP_ERR_CUDA;
  }
  return cuda_status("pmp_orth_step");
}

}  // extern "C"
