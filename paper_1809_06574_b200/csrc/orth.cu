// Kernel 5b+5c fused: one block-Arnoldi orthogonalisation step of block GCRO
// (krylov.py:189-202) in ONE cooperative launch.
//
//   W  -= C (C^T W)                         outer-space projection  :189-192
//   2x { H = V^T W ; W -= V H }             block CGS2              :193-196
//   W = Q R                                 _qr_deflate             :197-202
//
// The reference runs these as separate BLAS/LAPACK calls; on the device
// each is a tall-skinny reduction whose cost at BASELINE sizes is latency,
// not bandwidth.  Here every block owns a contiguous row range and keeps
// its rows of [C | V], W and Q in shared memory when they fit (c2: 222 rows
// x 87 columns), so HBM/L2 is read once; the reductions are two-stage
// (per-block partials, then a distributed fixed-order reduction) separated
// by grid-wide barriers, so no host round trip happens inside the step.
//
// Reduction schedule (3 reductions, 6 grid barriers):
//   R1: [C | V]^T W           -> B = C^T W, H1 = V^T W
//       W1 = W - C B - V H1          (C and V are mutually orthogonal, so
//                                     projecting on [C | V] at once equals
//                                     the reference's C-then-V order up to
//                                     rounding, which the second pass cleans)
//   R2: [V | W1]^T W1         -> H2 = V^T W1, W1^T W1
//       W2 = W1 - V H2,  G = W1^T W1 - H2^T H2   (= W2^T W2; H2 ~ eps)
//       R1f = chol(P^T G P) (symmetric pivoting), Q1 = W2 P R1f^-1
//   R3: Q1^T Q1 -> R2f = chol(.), Q = Q1 R2f^-1, R = R2f R1f (un-pivoted)
// When the pivoted Cholesky shows min |R_kk| / |R_00| <= 1e-5, Cholesky
// cannot decide the reference's 1e-12 deflation rank (krylov.py:92): the
// kernel leaves W2 in global memory, raises a flag, and the host falls back
// to Householder TSQR + pivoted QR (pmp_tsqr_r + pmp_host_deflate), which
// reproduce geqp3's rank decision.
#include "orth_dev.cuh"

namespace pmp {


struct OrthParams {
  int n;
  const double* C;
  int ldc, k;
  double* V;
  int ldv, total, npass;
  double* W;
  int ldw, sb;
  int qout;  // V column receiving the new orthonormal block
  int rows_per_block;
  double* partial;  // gridDim.x * kmax doubles
  double* Q1g;      // n x sb scratch (streaming mode)
  double* gout;     // reduction results (global): kmax doubles
  double* outB;     // k x sb      (C^T W)
  double* outH1;    // total x sb  (first CGS pass)
  double* outH2;    // total x sb  (second CGS pass)
  double* outR;     // sb x sb     (R, un-pivoted, row-major)
  double* outFlag;  // 1 double: 0 ok, 1 fallback needed
  // optional zero-copy mirror: the small outputs above live at offsets of
  // one device buffer `dbase`; block 0 copies them to the same offsets of
  // mapped host memory `mbase` and writes the flag there last
  const double* dbase;
  double* mbase;
  unsigned long long* dbg;  // optional phase timestamps (block 0), diagnostics
};

__device__ __forceinline__ void stamp(const OrthParams& P, int i) {
#ifdef PMP_STAMPS
  if (P.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.dbg[i] = t;
  }
#else
  (void)P;
  (void)i;
#endif
}

// block 0, all threads: flag (and, with a mirror, the small results) out
__device__ void publish(const OrthParams& P, double flag) {
  if (threadIdx.x == 0) *P.outFlag = flag;
  if (P.mbase) {
    const int sb = P.sb;
    const double* src[4] = {P.outB, P.outH1, P.outH2, P.outR};
    const int len[4] = {P.k * sb, P.npass ? P.total * sb : 0, P.npass ? P.total * sb : 0,
                        flag == 0.0 ? sb * sb : 0};
    for (int a = 0; a < 4; ++a) {
      if (!src[a] || len[a] == 0) continue;
      double* dst = P.mbase + (src[a] - P.dbase);
      for (int q = threadIdx.x; q < len[a]; q += kOrthT) dst[q] = __ldcg(src[a] + q);
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      *(volatile double*)(P.mbase + (P.outFlag - P.dbase)) = flag;
    }
  }
}







template <bool CACHED, int NY>
__global__ void __launch_bounds__(kOrthT, 2) k_orth(OrthParams P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sh[];
  stamp(P, 0);
  const int r0 = blockIdx.x * P.rows_per_block;
  const int r1 = min(P.n, r0 + P.rows_per_block);
  const int nr = max(0, r1 - r0);
  const int sb = P.sb, k = P.k, tot = P.total;
  const int kx = k + tot;
  const int kmax = (kx + sb) * sb;
  double* p = sh;
  double* G = p;
  p += kmax;
  p += sb * sb;  // (unused slot kept: the smem size formula counts it)
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
  Rows CV;
  double* Wv;
  int ldw;
  double* Q1;
  int ldq;
  if (CACHED) {
    const int ldx = odd_ld(kx);
    double* Xs = p;
    p += (size_t)nr * ldx;
    ldw = odd_ld(sb);
    Wv = p;
    p += (size_t)nr * ldw;
    ldq = ldw;
    Q1 = p;
    const double* Cg = P.C + (size_t)r0 * P.ldc;
    const double* Vg = P.V + (size_t)r0 * P.ldv;
    const double* Wg = P.W + (size_t)r0 * P.ldw;
    // 4 independent loads in flight per thread before the stores
    const int tot4 = nr * kx;
    for (int q0 = threadIdx.x; q0 < tot4; q0 += 4 * kOrthT) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * kOrthT;
        if (q < tot4) {
          const int r = q / kx, t = q % kx;
          v[u] = t < k ? __ldcg(Cg + (size_t)r * P.ldc + t) : __ldcg(Vg + (size_t)r * P.ldv + t - k);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * kOrthT;
        if (q < tot4) Xs[(size_t)(q / kx) * ldx + q % kx] = v[u];
      }
    }
    for (int q = threadIdx.x; q < nr * sb; q += kOrthT)
      Wv[(size_t)(q / sb) * ldw + q % sb] = Wg[(size_t)(q / sb) * P.ldw + q % sb];
    CV = Rows{Xs, ldx, kx, Xs, ldx};
    __syncthreads();
  } else {
    CV = Rows{P.C + (size_t)r0 * P.ldc, P.ldc, k, P.V + (size_t)r0 * P.ldv, P.ldv};
    Wv = P.W + (size_t)r0 * P.ldw;
    ldw = P.ldw;
    Q1 = P.Q1g + (size_t)r0 * sb;
    ldq = sb;
  }
  const double* Vrows = CACHED ? CV.a + k : P.V + (size_t)r0 * P.ldv;
  const int ldvr = CACHED ? CV.lda : P.ldv;
  const Rows Vonly{Vrows, ldvr, tot, Vrows, ldvr};
  stamp(P, 1);

  // ---- R1: [C | V]^T W -------------------------------------------------------
  if (kx > 0) {
    block_gram<NY>(CV, kx, Wv, ldw, sb, nr, red, P.partial);
    stamp(P, 2);
    grid_reduce(grid, P.partial, P.gout, kx * sb, G, P.outB, k * sb, P.npass ? P.outH1 : nullptr);
    stamp(P, 3);
    block_update<NY>(CV, kx, Wv, ldw, sb, nr, G);
    stamp(P, 4);
  }
  // ---- R2: [V | W1]^T W1 -----------------------------------------------------
  const bool second = P.npass >= 2 && tot > 0;
  const int kv2 = second ? tot : 0;
  const int kx2 = kv2 + sb;
  {
    const Rows VW{Vrows, ldvr, kv2, Wv, ldw};
    block_gram<NY>(VW, kx2, Wv, ldw, sb, nr, red, P.partial);
    stamp(P, 5);
    grid_reduce(grid, P.partial, P.gout, kx2 * sb, G, second ? P.outH2 : nullptr, kv2 * sb, nullptr);
    stamp(P, 6);
  }
  // G_W = W1^T W1 - H2^T H2 (into R2 as scratch), then W2 = W1 - V H2
  // (4 threads per entry over strided t, combined in a fixed order)
  const int n4 = 4 * sb * sb, lim4 = (n4 + 31) & ~31;   // warp-uniform trip count
  for (int q4 = threadIdx.x; q4 < lim4; q4 += kOrthT) {
    const bool act = q4 < n4;
    const int q = q4 >> 2, part = q4 & 3;
    const int i = act ? q / sb : 0, j = act ? q % sb : 0;
    double s = 0.0;
    if (act)
      for (int t = part; t < kv2; t += 4) s += G[t * sb + i] * G[t * sb + j];
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (act && part == 0) R2[q] = G[(size_t)(kv2 + i) * sb + j] - s;
  }
  __syncthreads();
  if (second) block_update<NY>(Vonly, tot, Wv, ldw, sb, nr, G);
  stamp(P, 7);
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
  stamp(P, 8);
  // a well-conditioned block (|R_00| / |R_mm| <= 4) is orthonormal to
  // ~16 eps after one Cholesky-QR pass: skip the second reduction
  bool single = false;
  if (flag[0] == 0) {
    const double kap = fabs(R1[0]) / fabs(R1[(sb - 1) * sb + (sb - 1)]);
    single = kap <= kSkipKappa;
  }
  if (flag[0] == 0 && !single) {
    block_trsm_rows<NY>(Wv, ldw, Q1, ldq, nr, sb, R1, piv);
    // ---- R3: Q1^T Q1 ---------------------------------------------------------
    const Rows Qv{Q1, ldq, sb, Q1, ldq};
    block_gram<NY>(Qv, sb, Q1, ldq, sb, nr, red, P.partial);
    grid_reduce(grid, P.partial, P.gout, sb * sb, G, nullptr, 0, nullptr);
    if (threadIdx.x < 32) {
      bool ok = warp_cholesky_reg<NY>(G, sb, R2, piv2, false, 0.0);
      if (threadIdx.x == 0) flag[0] = ok ? 0 : 1;
    }
    __syncthreads();
  }
  stamp(P, 9);
  // flag is grid-uniform: every block factored the same reduced matrices
  if (flag[0]) {
    if (CACHED)
      for (int q = threadIdx.x; q < nr * sb; q += kOrthT)
        P.W[(size_t)(r0 + q / sb) * P.ldw + q % sb] = Wv[(size_t)(q / sb) * ldw + q % sb];
    __threadfence();
    grid.sync();   // every block's W rows are written back before the flag
    if (blockIdx.x == 0) publish(P, 1.0);
    return;
  }
  if (single) {
    // Q = W P R1^-1 -> V[:, qout : qout + sb], R2 = I
    block_trsm_rows<NY>(Wv, ldw, P.V + (size_t)r0 * P.ldv + P.qout, P.ldv, nr, sb, R1, piv);
    for (int q = threadIdx.x; q < sb * sb; q += kOrthT) R2[q] = (q / sb == q % sb) ? 1.0 : 0.0;
    __syncthreads();
  } else {
    block_trsm_rows<NY>(Q1, ldq, P.V + (size_t)r0 * P.ldv + P.qout, P.ldv, nr, sb, R2, nullptr);
  }
  if (blockIdx.x == 0) {
    // R = R2 R1 (pivoted column order), un-pivoted: Rout[i, piv[c]] = R[i, c]
    for (int q = threadIdx.x; q < sb * sb; q += kOrthT) {
      const int i = q / sb, c = q % sb;
      double s = 0.0;
      for (int a = i; a <= c; ++a) s += R2[i * sb + a] * R1[a * sb + c];
      P.outR[i * sb + piv[c]] = (c >= i) ? s : 0.0;
    }
    __syncthreads();
    stamp(P, 10);
    publish(P, 0.0);
  }
}

// ---------------------------------------------------------------------------
// Outer-space fold (krylov.py:244-269) in one cooperative launch: for each
// image column, CGS2 against the current C (with the matching U update),
// the 1e-10 drop test, and the append -- all decisions are grid-uniform, so
// no host round trip per column.  Norms: ||w||^2 comes with the first
// projection's reduction, ||w2||^2 = ||w1||^2 - ||h2||^2 with the second
// (recomputed exactly when that difference cancels).
// ---------------------------------------------------------------------------

struct FoldParams {
  int n, na;
  const double* img;
  int ldi;
  const double* dz;
  int ldz;
  double* C;
  double* U;
  int ldc, kc, k0;
  int rows_per_block;
  double* partial;
  double* gout;
  double* wz;   // n x 2 scratch (streaming mode)
  double* out;  // out[0] = final outer dimension, out[1 + col] = kept flag
};

template <bool CACHED>
__global__ void __launch_bounds__(kOrthT, 2) k_fold(FoldParams F) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sh[];
  const int r0 = blockIdx.x * F.rows_per_block;
  const int r1 = min(F.n, r0 + F.rows_per_block);
  const int nr = max(0, r1 - r0);
  const int kc = F.kc;
  double* p = sh;
  double* G = p;
  p += kc + 8;
  double* red = p;
  p += 8 * 32 * 16;
  OrthParams P;  // only the reduction scratch is used by grid_reduce
  P.partial = F.partial;
  P.gout = F.gout;
  double *Cs, *Us, *w, *z;
  int ldcs;
  if (CACHED) {
    ldcs = odd_ld(kc);
    Cs = p;
    p += (size_t)nr * ldcs;
    Us = p;
    p += (size_t)nr * ldcs;
    w = p;
    p += nr;
    z = p;
    for (int q = threadIdx.x; q < nr * kc; q += kOrthT) {
      const int r = q / kc, t = q % kc;
      if (t < F.k0) {
        Cs[(size_t)r * ldcs + t] = F.C[(size_t)(r0 + r) * F.ldc + t];
        Us[(size_t)r * ldcs + t] = F.U[(size_t)(r0 + r) * F.ldc + t];
      }
    }
  } else {
    ldcs = F.ldc;
    Cs = F.C + (size_t)r0 * F.ldc;
    Us = F.U + (size_t)r0 * F.ldc;
    w = F.wz + (size_t)r0 * 2;
    z = w + 1;
  }
  const int ldwz = CACHED ? 1 : 2;
  int kk = F.k0;
  for (int col = 0; col < F.na; ++col) {
    for (int r = threadIdx.x; r < nr; r += kOrthT) {
      w[(size_t)r * ldwz] = F.img[(size_t)(r0 + r) * F.ldi + col];
      z[(size_t)r * ldwz] = F.dz[(size_t)(r0 + r) * F.ldz + col];
    }
    __syncthreads();
    // [C | w]^T w  ->  h1, ||w||^2
    Rows Cw{Cs, ldcs, kk, w, ldwz};
    block_gram<1>(Cw, kk + 1, w, ldwz, 1, nr, red, P.partial);
    grid_reduce(grid, P.partial, P.gout, kk + 1, G, nullptr, 0, nullptr);
    const double w0 = sqrt(G[kk]);
    if (w0 == 0.0) {
      if (blockIdx.x == 0 && threadIdx.x == 0) F.out[1 + col] = 0.0;
      continue;
    }
    double nw;
    if (kk > 0) {
      Rows Conly{Cs, ldcs, kk, Cs, ldcs}, Uonly{Us, ldcs, kk, Us, ldcs};
      block_update<1>(Conly, kk, w, ldwz, 1, nr, G);
      block_update<1>(Uonly, kk, z, ldwz, 1, nr, G);
      block_gram<1>(Cw, kk + 1, w, ldwz, 1, nr, red, P.partial);
      grid_reduce(grid, P.partial, P.gout, kk + 1, G, nullptr, 0, nullptr);
      double h2 = 0.0;
      for (int t = 0; t < kk; ++t) h2 += G[t] * G[t];
      const double w1n2 = G[kk];
      block_update<1>(Conly, kk, w, ldwz, 1, nr, G);
      block_update<1>(Uonly, kk, z, ldwz, 1, nr, G);
      double nw2 = w1n2 - h2;
      if (!(nw2 > 1e-4 * w1n2)) {
        // cancellation: recompute ||w2||^2 exactly
        Rows Wo{w, ldwz, 1, w, ldwz};
        block_gram<1>(Wo, 1, w, ldwz, 1, nr, red, P.partial);
        grid_reduce(grid, P.partial, P.gout, 1, G, nullptr, 0, nullptr);
        nw2 = G[0];
      }
      nw = sqrt(fmax(nw2, 0.0));
    } else {
      nw = w0;
    }
    const bool keep = !(nw <= 1e-10 * w0);
    if (blockIdx.x == 0 && threadIdx.x == 0) F.out[1 + col] = keep ? 1.0 : 0.0;
    if (!keep) continue;
    const double inv = 1.0 / nw;
    for (int r = threadIdx.x; r < nr; r += kOrthT) {
      const double cv = w[(size_t)r * ldwz] * inv, uv = z[(size_t)r * ldwz] * inv;
      F.C[(size_t)(r0 + r) * F.ldc + kk] = cv;
      F.U[(size_t)(r0 + r) * F.ldc + kk] = uv;
      if (CACHED) {
        Cs[(size_t)r * ldcs + kk] = cv;
        Us[(size_t)r * ldcs + kk] = uv;
      }
    }
    __syncthreads();
    ++kk;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) F.out[0] = (double)kk;
}

// micro-benchmark of the grid barrier the cooperative kernels rely on
__global__ void __launch_bounds__(kOrthT, 2) k_grid_sync_bench(int iters, double* sink) {
  cg::grid_group grid = cg::this_grid();
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    acc += 1.0;
    __threadfence();
    grid.sync();
  }
  if (acc < 0) *sink = acc;
}

size_t fold_smem_bytes(int rows, int kc, int cached) {
  size_t d = (size_t)kc + 8 + 8 * 32 * 16;
  if (cached) d += (size_t)rows * (2 * odd_ld(kc) + 2);
  return d * sizeof(double);
}

size_t orth_smem_bytes(int rows, int total, int k, int sb, int cached) {
  const int kx = k + total;
  size_t d = (size_t)(kx + sb) * sb + 3 * sb * sb + 8 * 32 * sb + 20;
  if (cached) d += (size_t)rows * (odd_ld(kx) + 2 * odd_ld(sb));
  return d * sizeof(double);
}

}  // namespace pmp

using namespace pmp;

static void orth_geometry(int n, int total, int k, int sb, int* grid, int* rows, int* cached,
                          size_t* smem) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  // two co-resident blocks per SM when the cached rows fit in half the
  // shared memory (more warps to hide the latency of the row loops, half
  // the rows per block), otherwise one
  for (int bps = 2; bps >= 1; --bps) {
    int g = sms * bps;
    int want = (n + 31) / 32;
    if (want < g) g = want > 0 ? want : 1;
    int r = (n + g - 1) / g;
    size_t full = orth_smem_bytes(r, total, k, sb, 1);
    const size_t budget = bps == 2 ? (size_t)110 * 1024 : (size_t)220 * 1024;
    if (bps == 2 && full > budget) continue;
    *cached = full <= budget;
    *smem = *cached ? full : orth_smem_bytes(r, total, k, sb, 0);
    *grid = g;
    *rows = r;
    return;
  }
}

// Cooperative (grid-barrier) kernels must never be partially resident at the
// same time: when several host threads drive independent systems on their
// own streams, every cooperative launch is routed through one shared
// stream (event handoff both ways), which serialises them while all other
// kernels of the workers still overlap.
static cudaStream_t g_coop_stream = nullptr;
static unsigned long long* g_dbg = nullptr;   // pmp_orth_debug_stamps
static int g_dbg_left = 0;

cudaError_t pmp::coop_launch(const void* fn, int g, void** args, size_t smem,
                             cudaStream_t user) {
  if (!g_coop_stream || g_coop_stream == user)
    return cudaLaunchCooperativeKernel(fn, dim3(g), dim3(kOrthT), args, smem, user);
  thread_local cudaEvent_t in = nullptr, out = nullptr;
  if (!in) {
    cudaEventCreateWithFlags(&in, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&out, cudaEventDisableTiming);
  }
  cudaEventRecord(in, user);
  cudaStreamWaitEvent(g_coop_stream, in, 0);
  cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(g), dim3(kOrthT), args, smem, g_coop_stream);
  cudaEventRecord(out, g_coop_stream);
  cudaStreamWaitEvent(user, out, 0);
  return e;
}

int pmp::orth_max_grid() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return 2 * (sms > 0 ? sms : 148);
}

extern "C" {

size_t pmp_orth_workspace(int n, int total_max, int k_max, int sb) {
  int g, r, c;
  size_t sm;
  orth_geometry(n, total_max, k_max, sb, &g, &r, &c, &sm);
  g = orth_max_grid();   // any (total, k) may pick the two-blocks-per-SM grid
  const int kmax = (k_max + total_max + sb) * sb;
  return 256 + sizeof(double) * ((size_t)g * kmax + kmax + (size_t)n * sb + 64);
}

int pmp_orth_step(int n, const double* C, int ldc, int k, double* V, int ldv, int total, int npass,
                  double* W, int ldw, int sb, int qout, double* outB, double* outH1,
                  double* outH2, double* outR, double* outFlag, void* ws, size_t ws_bytes,
                  void* stream) {
  return pmp::orth_step_mirrored(n, C, ldc, k, V, ldv, total, npass, W, ldw, sb, qout, outB, outH1,
                                 outH2, outR, outFlag, ws, ws_bytes, stream, nullptr, nullptr);
}

}  // extern "C"

int pmp::orth_step_mirrored(int n, const double* C, int ldc, int k, double* V, int ldv, int total,
                            int npass, double* W, int ldw, int sb, int qout, double* outB,
                            double* outH1, double* outH2, double* outR, double* outFlag, void* ws,
                            size_t ws_bytes, void* stream, const double* dbase, double* mbase) {
  if (n < 1 || sb < 1 || sb > 16 || k < 0 || total < 0 || (k && ldc < k) || ldw < sb ||
      ldv < qout + sb || (total && ldv < total) || (npass != 0 && npass != 2)) {
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
  auto pick = [&](int c) -> void* {
    if (sb <= 8) return c ? (void*)k_orth<true, 8> : (void*)k_orth<false, 8>;
    return c ? (void*)k_orth<true, 16> : (void*)k_orth<false, 16>;
  };
  void* fn = pick(cached);
  int bps = prepare_smem(fn, smem, kOrthT);
  if (bps * (orth_max_grid() / 2) < g) {
    // the two-blocks-per-SM grid is not co-resident: one block per SM
    g = orth_max_grid() / 2;
    if ((n + 31) / 32 < g) g = (n + 31) / 32 > 0 ? (n + 31) / 32 : 1;
    rows = (n + g - 1) / g;
    size_t full = orth_smem_bytes(rows, total, k, sb, 1);
    cached = full <= (size_t)220 * 1024;
    smem = cached ? full : orth_smem_bytes(rows, total, k, sb, 0);
    fn = pick(cached);
    bps = prepare_smem(fn, smem, kOrthT);
  }
  if (bps < 1) {
    set_error("pmp_orth_step: kernel does not fit on an SM (smem %zu)", smem);
    return PMP_ERR_ARG;
  }
  const int kmax = (k + total + sb) * sb;
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
  double* w = (double*)((char*)ws + 256);
  P.partial = w;
  P.gout = w + (size_t)g * kmax;
  P.Q1g = P.gout + kmax;
  P.outB = outB;
  P.outH1 = outH1;
  P.outH2 = outH2;
  P.outR = outR;
  P.outFlag = outFlag;
  P.dbase = dbase;
  P.mbase = mbase;
  P.dbg = nullptr;
  if (g_dbg && g_dbg_left > 0) {   // one 16-slot record per launch
    P.dbg = g_dbg;
    g_dbg += 16;
    --g_dbg_left;
  }
  void* args[] = {&P};
  cudaError_t e = coop_launch(fn, g, args, smem, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    set_error("pmp_orth_step: %s", cudaGetErrorString(e));
    return PMP_ERR_CUDA;
  }
  return cuda_status("pmp_orth_step");
}

extern "C" {

// Diagnostics: block 0 of the next `records` k_orth launches writes
// %globaltimer at 11 phase boundaries into d_stamps[16 * launch + 0..10]
// (NULL disables; the default).
int pmp_orth_debug_stamps(unsigned long long* d_stamps, int records) {
  g_dbg = d_stamps;
  g_dbg_left = d_stamps ? records : 0;
  return PMP_OK;
}

// Route every cooperative launch through `stream` (NULL: launch on the
// caller's stream, the single-worker default).
int pmp_set_coop_stream(void* stream) {
  g_coop_stream = reinterpret_cast<cudaStream_t>(stream);
  return PMP_OK;
}

// Enqueue `iters` grid barriers over blocks_per_sm x #SMs CTAs of 256
// threads (time it with events around the call).
int pmp_bench_grid_sync(int blocks_per_sm, int iters, void* stream) {
  int g = orth_max_grid() / 2 * blocks_per_sm;
  double* sink = nullptr;
  void* args[] = {&iters, &sink};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)k_grid_sync_bench, dim3(g), dim3(kOrthT),
                                              args, 0, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    set_error("pmp_bench_grid_sync: %s", cudaGetErrorString(e));
    return PMP_ERR_CUDA;
  }
  return PMP_OK;
}

size_t pmp_fold_workspace(int n, int kc) {
  const int g = orth_max_grid();
  return 256 + sizeof(double) * ((size_t)g * (kc + 1) + (kc + 1) + 2 * (size_t)n + 64);
}

int pmp_fold(int n, int na, const double* img, int ldi, const double* dz, int ldz, double* C,
             double* U, int ldc, int kc, int k0, double* out, void* ws, size_t ws_bytes,
             void* stream) {
  if (n < 1 || na < 0 || k0 < 0 || k0 + na > kc || ldc < kc || ldi < na || ldz < na) {
    set_error("pmp_fold: bad arguments (n=%d na=%d k0=%d kc=%d)", n, na, k0, kc);
    return PMP_ERR_ARG;
  }
  if (ws_bytes < pmp_fold_workspace(n, kc)) {
    set_error("pmp_fold: workspace too small");
    return PMP_ERR_WORKSPACE;
  }
  // one block per SM: the fold is grid-barrier bound (4 barriers per
  // column), and barrier cost grows with the block count
  int g = orth_max_grid() / 2;
  if ((n + 31) / 32 < g) g = (n + 31) / 32 > 0 ? (n + 31) / 32 : 1;
  const int rows = (n + g - 1) / g;
  const int cached = fold_smem_bytes(rows, kc, 1) <= (size_t)220 * 1024;
  const size_t smem = fold_smem_bytes(rows, kc, cached);
  void* fn = cached ? (void*)k_fold<true> : (void*)k_fold<false>;
  if (prepare_smem(fn, smem, kOrthT) * (orth_max_grid() / 2) < g) {
    set_error("pmp_fold: grid of %d blocks is not co-resident", g);
    return PMP_ERR_ARG;
  }
  FoldParams F;
  F.n = n;
  F.na = na;
  F.img = img;
  F.ldi = ldi;
  F.dz = dz;
  F.ldz = ldz;
  F.C = C;
  F.U = U;
  F.ldc = ldc;
  F.kc = kc;
  F.k0 = k0;
  F.rows_per_block = rows;
  double* w = (double*)((char*)ws + 256);
  F.partial = w;
  F.gout = w + (size_t)g * (kc + 1);
  F.wz = F.gout + (kc + 1);
  F.out = out;
  void* args[] = {&F};
  cudaError_t e = coop_launch(fn, g, args, smem, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    set_error("pmp_fold: %s", cudaGetErrorString(e));
    return PMP_ERR_CUDA;
  }
  return cuda_status("pmp_fold");
}

}  // extern "C"
