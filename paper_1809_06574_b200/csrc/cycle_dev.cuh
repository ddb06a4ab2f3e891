// Device pieces shared by the persistent block-GCRO kernels: k_cycle (one
// cycle's inner loop, cycle.cu) and k_solve (whole solves, several systems
// per launch, solve.cu).  See cycle.cu for the design.
#pragma once

#include "orth_dev.cuh"


namespace pmp {

unsigned long long* cycle_dbg_take();  // cycle.cu (diagnostics)

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
  double *partial, *gout, *Q1g, *sbuf;
  int rows_per_block, ldx, max_iters, inner_restart, hist_cap, nblk;
  int wglob;  // W rows in global memory (P.W) instead of shared memory
  double tol;
  double* proj;
  int oBmat, oHb, oQR, oTau, oCq, oY, oRes, oBn, oHist;
  int* ist;
  unsigned long long* dbg;  // optional phase stamps (pmp_cycle_debug_stamps)
};

// diagnostics: %globaltimer of phase i of step `step`, blocks 0 and 1
// (pmp_cycle_debug_stamps; P.dbg is null unless a diagnostics run set it)
static __device__ __forceinline__ void cstamp_on(const CycleArgs& P, int step, int i) {
  if (P.dbg && blockIdx.x < 2 && threadIdx.x == 0 && step < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.dbg[((size_t)step * 32 + i) * 2 + blockIdx.x] = t;
  }
}
static __device__ __forceinline__ void cstamp(const CycleArgs& P, int step, int i) {
#ifdef PMP_STAMPS
  // diagnostics builds (tools/build_variant.sh stamps -DPMP_STAMPS): the
  // stamps perturb code generation, so production builds compile them out
  // of the shared-memory geometries
  cstamp_on(P, step, i);
#else
  (void)P;
  (void)step;
  (void)i;
#endif
}
// The worker step loop's stamps stay compiled in where STAMP is set: the
// global-row instance of k_solve runs 7 % FASTER with them (c4 6-system
// batch 448 -> 416 ms, profiles/r02_codegen_ab.txt; same spills -- the
// volatile timer reads pin the phase order the scheduler otherwise
// interleaves), the shared-memory instances 2 % slower.
template <bool STAMP>
static __device__ __forceinline__ void wstamp(const CycleArgs& P, int step, int i) {
  if (STAMP)
    cstamp_on(P, step, i);
  else
    cstamp(P, step, i);
}

static __device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

#ifndef PMP_SPMM_RPT
#define PMP_SPMM_RPT 2
#endif
#ifndef PMP_SPMM_CH
#define PMP_SPMM_CH 8
#endif
#ifndef PMP_BAR_ACQREL
#define PMP_BAR_ACQREL 1
#endif

// Y[r][c] = sum_e vals[e] X[colidx[e]][c] for this block's rows r0 + [0, nr):
// NY lanes per row (lane = column), RPT rows per thread, entries gathered CH
// at a time with every index / value load issued before the X gathers.  X
// may have been written earlier in this kernel by other blocks: loads
// bypass L1 (ld.cg).  Accumulation order matches k_spmm (even / odd
// entries, then summed).
#ifndef PMP_SPMM_CA
#define PMP_SPMM_CA 1
#endif
#ifndef PMP_SPMM_RP_AHEAD
#define PMP_SPMM_RP_AHEAD 1
#endif

template <int NY, bool CA = false>
__device__ __noinline__ void spmm_rows(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ va, const double* X, int ldx, int sb,
                          double* Y, int ldy, int r0, int nr) {
  constexpr int PER = kOrthT / NY, RPT = PMP_SPMM_RPT, CH = PMP_SPMM_CH;
  const int c = threadIdx.x % NY, slot = threadIdx.x / NY;
  const bool col_ok = c < sb;
#if PMP_SPMM_RP_AHEAD
  // the next pass's row extents are loaded one pass ahead: the row-pointer
  // load leaves the dependent chain (pointer -> index -> gather) of a pass
  int nlo[RPT], nhi[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int r = slot + u * PER;
    nlo[u] = nhi[u] = 0;
    if (r < nr) {
      nlo[u] = __ldg(rp + r0 + r);
      nhi[u] = __ldg(rp + r0 + r + 1);
    }
  }
#endif
  for (int base = 0; base < nr; base += RPT * PER) {
    int lo[RPT], hi[RPT];
    double a0[RPT], a1[RPT];
    int len = 0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int r = base + slot + u * PER;
      a0[u] = 0.0;
      a1[u] = 0.0;
#if PMP_SPMM_RP_AHEAD
      lo[u] = nlo[u];
      hi[u] = nhi[u];
      const int rn = r + RPT * PER;
      nlo[u] = nhi[u] = 0;
      if (rn < nr) {
        nlo[u] = __ldg(rp + r0 + rn);
        nhi[u] = __ldg(rp + r0 + rn + 1);
      }
#else
      lo[u] = 0;
      hi[u] = 0;
      if (r < nr) {
        lo[u] = __ldg(rp + r0 + r);
        hi[u] = __ldg(rp + r0 + r + 1);
      }
#endif
      len = max(len, hi[u] - lo[u]);
    }
    for (int e0 = 0; e0 < len; e0 += CH) {
      int j[RPT][CH];
      double w[RPT][CH], x[RPT][CH];
#pragma unroll
      for (int u = 0; u < RPT; ++u)
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          const int e = lo[u] + e0 + q;
          const bool ok = e < hi[u];
          j[u][q] = ok ? __ldg(ci + e) : -1;
          w[u][q] = ok ? __ldg(va + e) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < RPT; ++u)
#pragma unroll
        for (int q = 0; q < CH; ++q)
          x[u][q] = (j[u][q] >= 0 && col_ok)
                        ? (CA ? __ldca(X + (size_t)j[u][q] * ldx + c)
                              : __ldcg(X + (size_t)j[u][q] * ldx + c))
                        : 0.0;
#pragma unroll
      for (int u = 0; u < RPT; ++u)
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          if (q & 1)
            a1[u] += w[u][q] * x[u][q];
          else
            a0[u] += w[u][q] * x[u][q];
        }
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int r = base + slot + u * PER;
      if (r < nr && col_ok) Y[(size_t)r * ldy + c] = a0[u] + a1[u];
    }
  }
}

// spmm_rows over TILES DEALT CYCLICALLY to the group's workers (worker wi of
// nw takes tiles wi, wi + nw, ... of kCycTile rows of the whole matrix)
// instead of one contiguous row range per block.  With contiguous ranges
// the blocks of a group sweep 48 distant fronts at once, so a far neighbour
// of a grid stencil (row r +- 128^2 at c4) is re-read from HBM every time:
// ncu put k_solve's DRAM traffic at 2.0x the algorithmic bytes, the SpMM's X
// read ~3x.  Dealt cyclically the group works on one window of nw tiles that
// moves through the matrix, and a row gathered as somebody's far neighbour
// is still in L2 when its own tile comes up.  Inside a tile the near
// neighbours (+-1, +-128) still hit L1.  The output rows belong to other
// blocks afterwards: the caller places a group barrier before reading them.
// Same per-row arithmetic as spmm_rows (bitwise equal).
constexpr int kCycTile = 512;
template <int NY, bool CA>
__device__ __noinline__ void spmm_rows_cyc(const int32_t* __restrict__ rp,
                                           const int32_t* __restrict__ ci,
                                           const double* __restrict__ va, const double* X, int ldx,
                                           int sb, double* Y, int ldy, int n, int wi, int nw) {
  constexpr int PER = kOrthT / NY, RPT = PMP_SPMM_RPT, CH = PMP_SPMM_CH, STEP = RPT * PER;
  constexpr int PPT = kCycTile / STEP;  // passes per tile
  static_assert(kCycTile % STEP == 0, "tile must be whole passes");
  const int c = threadIdx.x % NY, slot = threadIdx.x / NY;
  const bool col_ok = c < sb;
  const int ntile = (n + kCycTile - 1) / kCycTile;
  const int mine = wi < ntile ? (ntile - wi + nw - 1) / nw : 0;  // this worker's tiles
  const int npass = mine * PPT;
  // global row of (pass p, sub-row u) of this thread
  auto rowof = [&](int p, int u) {
    return (wi + (p / PPT) * nw) * kCycTile + (p % PPT) * STEP + slot + u * PER;
  };
  int nlo[RPT], nhi[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int r = rowof(0, u);
    nlo[u] = nhi[u] = 0;
    if (npass > 0 && r < n) {
      nlo[u] = __ldg(rp + r);
      nhi[u] = __ldg(rp + r + 1);
    }
  }
  for (int p = 0; p < npass; ++p) {
    int lo[RPT], hi[RPT];
    double a0[RPT], a1[RPT];
    int len = 0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      a0[u] = 0.0;
      a1[u] = 0.0;
      lo[u] = nlo[u];
      hi[u] = nhi[u];
      const int rn = rowof(p + 1, u);
      nlo[u] = nhi[u] = 0;
      if (p + 1 < npass && rn < n) {
        nlo[u] = __ldg(rp + rn);
        nhi[u] = __ldg(rp + rn + 1);
      }
      len = max(len, hi[u] - lo[u]);
    }
    for (int e0 = 0; e0 < len; e0 += CH) {
      int j[RPT][CH];
      double w[RPT][CH], x[RPT][CH];
#pragma unroll
      for (int u = 0; u < RPT; ++u)
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          const int e = lo[u] + e0 + q;
          const bool ok = e < hi[u];
          j[u][q] = ok ? __ldg(ci + e) : -1;
          w[u][q] = ok ? __ldg(va + e) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < RPT; ++u)
#pragma unroll
        for (int q = 0; q < CH; ++q)
          x[u][q] = (j[u][q] >= 0 && col_ok)
                        ? (CA ? __ldca(X + (size_t)j[u][q] * ldx + c)
                              : __ldcg(X + (size_t)j[u][q] * ldx + c))
                        : 0.0;
#pragma unroll
      for (int u = 0; u < RPT; ++u)
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          if (q & 1)
            a1[u] += w[u][q] * x[u][q];
          else
            a0[u] += w[u][q] * x[u][q];
        }
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int r = rowof(p, u);
      if (r < n && col_ok) Y[(size_t)r * ldy + c] = a0[u] + a1[u];
    }
  }
}

// spmm_rows for the step loop and the cycle boundaries; `ring` is unused
// since the asynchronous-ring variant was measured and dropped: cp.async
// index / value segments two tiles ahead, gathered X rows one tile ahead,
// products from shared memory -- 1.09 vs 1.41 ms alone
// (tools/micro/spmm_bench.cu keeps it), but its 74 KB of shared memory per
// block shrink L1 to 28 KB and every other gather phase of k_solve slows
// (c4 batch 634 vs 491 ms, profiles/r02_codegen_ab.txt).
template <int NY, bool CA = false>
__device__ __forceinline__ void spmm_auto(const int32_t* __restrict__ rp,
                                          const int32_t* __restrict__ ci,
                                          const double* __restrict__ va, const double* X, int ldx,
                                          int sb, double* Y, int ldy, int r0, int nr, double* ring,
                                          int ring_doubles) {
  (void)ring;
  (void)ring_doubles;
  spmm_rows<NY, CA>(rp, ci, va, X, ldx, sb, Y, ldy, r0, nr);
}

// control-block shared state
struct Ctl {
  double* Mq;    // nblk x (2b x 2b), row-major: M_q = Q_q^T of step q's window
  double* Rp;    // packed R of the Hb part: block column q is (q+1) b x b, column-major
  double* Cq;    // ldq x na, column-major (Q^T rhs)
  double* cols;  // b x ldq: the step's new columns of G
  double* Rr;    // b x b: R of the step's orthonormalisation (un-pivoted)
  double* ybuf;  // 16 x 96: back substitution (one row per right-hand side)
  double* v;     // 32: current reflector
  double* misc;  // [0] max |R_jj| [1] min |R_jj| [2] tau [3] NaN seen
  double* bn;    // 16: column norms of the right-hand sides
  double* res;   // 16
  double* xw;    // (2b + 1) x (3b + na): window factorisation
  double* bh1;   // (k + total) x b: [B; H1] of the step (R1 reduction)
  double* h2;    // total x b: H2 of the step (R2 reduction)
};

// control-block shared-memory layout (size: cycle_region_doubles)
static __device__ __forceinline__ Ctl ctl_layout(double* region, int sb, int nblk, int ldq, int na) {
  Ctl S;
  const int b2 = 2 * sb;
  double* q = region;
  S.Mq = q;
  q += (size_t)nblk * b2 * b2;
  S.Rp = q;
  q += (size_t)sb * sb * nblk * (nblk + 1) / 2;
  S.Cq = q;
  q += (size_t)ldq * na;
  S.cols = q;
  q += (size_t)sb * ldq;
  S.Rr = q;
  q += sb * sb;
  S.ybuf = q;
  q += 16 * 96;
  S.v = q;
  q += 32;
  S.misc = q;
  q += 8;
  S.bn = q;
  q += 16;
  S.res = q;
  q += 16;
  S.xw = q;
  q += (2 * sb + 1) * (3 * sb + na);
  S.bh1 = q;
  q += (size_t)ldq * sb;
  S.h2 = q;
  return S;
}

static __device__ __forceinline__ size_t rp_off(int q, int b) { return (size_t)b * b * q * (q + 1) / 2; }

// Absorb step q (its B / H1 / H2 in the small buffer, its R in S.Rr) into
// Bmat / Hb and the block QR of G; residual estimates and stop test
// (krylov.py:204-216).  Returns 0 continue, 1 converged, 4 G (near) rank
// deficient.  All threads of the control block.
template <int NY>
__device__ int ctl_absorb(const CycleArgs& P, const Ctl& S, int q, int total, int hrow) {
  const int k = P.k, b = P.sb, na = P.na, ldq = P.ldq, cap = P.cap, b2 = 2 * b;
  const int q0 = q * b;             // first Hb column of the step
  const int nrows = k + total + b;  // total == (q + 1) b
  const int tid = threadIdx.x;
  __shared__ int s_ret;
  // Bmat[:, q0:q1] = B ; Hb[:total, q0:q1] += H1, += H2 ; Hb[total:, q0:q1] = R
  // (B, H1, H2 were copied from the reductions into S.bh1 / S.h2)
  for (int c = 0; c < b; ++c) {
    for (int i = tid; i < ldq; i += kOrthT) {
      double v = 0.0;
      if (i < k) {
        v = S.bh1[i * b + c];
        P.proj[P.oBmat + (size_t)i * cap + q0 + c] = v;
      } else if (i < k + total) {
        const int t = i - k;
        v = 0.0 + S.bh1[(k + t) * b + c];
        v += S.h2[t * b + c];
        P.proj[P.oHb + (size_t)t * cap + q0 + c] = v;
      } else if (i < nrows) {
        const int t = i - k - total;
        v = S.Rr[t * b + c];
        P.proj[P.oHb + (size_t)(total + t) * cap + q0 + c] = v;
      }
      S.cols[(size_t)c * ldq + i] = v;
    }
  }
  __syncthreads();
  cstamp(P, q, 16);
  // earlier steps' window transforms, in order (M_p stored column-major)
  {
    const int nout = b * b2;
    const int x0 = tid, x1 = tid + kOrthT;
    const int c0 = x0 / b2, i0 = x0 % b2, c1 = x1 / b2, i1 = x1 % b2;
#pragma unroll 1
    for (int p = 0; p < q; ++p) {
      const double* M = S.Mq + (size_t)p * b2 * b2;
      const int w0 = k + p * b;
      double o0 = 0.0, o1 = 0.0;
      if (x0 < nout) {
        const double* col = S.cols + (size_t)c0 * ldq + w0;
#pragma unroll 4
        for (int j = 0; j < b2; ++j) o0 += M[j * b2 + i0] * col[j];
      }
      if (x1 < nout) {
        const double* col = S.cols + (size_t)c1 * ldq + w0;
#pragma unroll 4
        for (int j = 0; j < b2; ++j) o1 += M[j * b2 + i1] * col[j];
      }
      __syncthreads();
      if (x0 < nout) S.cols[(size_t)c0 * ldq + w0 + i0] = o0;
      if (x1 < nout) S.cols[(size_t)c1 * ldq + w0 + i1] = o1;
      __syncthreads();
    }
  }
  cstamp(P, q, 17);
  // factor the window [w0, w0 + 2b) of [block | I_2b | rhs]: one thread per
  // column, columns in shared memory (ld 2b + 1), rolled loops
  const int w0 = k + q0;
  const int ncx = 3 * b + na, ldX = b2 + 1;
  double* X = S.xw;
  cstamp(P, q, 28);
  for (int x = tid; x < ncx * b2; x += kOrthT) {
    const int c = x / b2, i = x % b2;
    double v;
    if (c < b)
      v = S.cols[(size_t)c * ldq + w0 + i];
    else if (c < 3 * b)
      v = (i == c - b) ? 1.0 : 0.0;
    else
      v = S.Cq[(size_t)(c - 3 * b) * ldq + w0 + i];
    X[c * ldX + i] = v;
  }
  __syncthreads();
#pragma unroll 1
  for (int j = 0; j < b; ++j) {
    if (tid == j) {
      // LAPACK dlarfg on (x[j], x[j+1 .. 2b)) (hostls.cpp larfg); v is
      // left below the diagonal
      double* xj = X + j * ldX;
      double x2 = 0.0;
      for (int i = j + 1; i < b2; ++i) x2 += xj[i] * xj[i];
      const double a = xj[j];
      double tj = 0.0, beta = a;
      if (x2 != 0.0) {
        beta = -copysign(hypot(a, sqrt(x2)), a);
        tj = (beta - a) / beta;
        const double scal = 1.0 / (a - beta);
        for (int i = j + 1; i < b2; ++i) xj[i] *= scal;
      }
      xj[j] = beta;
      S.misc[2] = tj;
    }
    __syncthreads();
    const double tj = S.misc[2];
    if (tid > j && tid < ncx && tj != 0.0) {
      const double* v = X + j * ldX;
      double* o = X + tid * ldX;
      double w = o[j];
      for (int i = j + 1; i < b2; ++i) w += v[i] * o[i];
      o[j] -= tj * w;
      for (int i = j + 1; i < b2; ++i) o[i] -= tj * w * v[i];
    }
    __syncthreads();
    if (j < 8) cstamp(P, q, 20 + j);
  }
  for (int x = tid; x < ncx * b2; x += kOrthT) {
    const int c = x / b2, i = x % b2;
    const double v = X[c * ldX + i];
    if (c < b)
      S.cols[(size_t)c * ldq + w0 + i] = i <= c ? v : 0.0;  // R (reflectors below)
    else if (c < 3 * b)
      S.Mq[(size_t)q * b2 * b2 + (c - b) * b2 + i] = v;     // column c-b of Q_q^T
    else
      S.Cq[(size_t)(c - 3 * b) * ldq + w0 + i] = v;
  }
  __syncthreads();
  if (tid < na) {
    const double* xr = X + (3 * b + tid) * ldX;
    double s2 = 0.0;
    for (int i = b; i < b2; ++i) s2 += xr[i] * xr[i];
    S.res[tid] = sqrt(s2);
    P.proj[P.oRes + tid] = S.res[tid];
  }
  __syncthreads();
  cstamp(P, q, 18);
  // packed R of this block column: rows [0, q0 + b) of the Hb part
  {
    const int h = q0 + b;
    double* Rq = S.Rp + rp_off(q, b);
    for (int x = tid; x < b * h; x += kOrthT) {
      const int c = x / h, t = x % h;
      Rq[(size_t)c * h + t] = S.cols[(size_t)c * ldq + k + t];
    }
  }
  if (tid == 0) {
    // rank test over every R diagonal so far (hostls.cpp:168-173):
    // deficient when some |R_jj| <= 1e-13 max |R_jj|
    double dmax = S.misc[0], dmin = S.misc[1], nan = S.misc[3];
    for (int c = 0; c < b; ++c) {
      const double d = fabs(S.cols[(size_t)c * ldq + w0 + c]);
      if (!(d == d)) nan = 1.0;
      dmax = fmax(dmax, d);
      dmin = fmin(dmin, d);
    }
    S.misc[0] = dmax;
    S.misc[1] = dmin;
    S.misc[3] = nan;
    int ret;
    if (nan != 0.0 || !(dmin > 1e-13 * dmax)) {
      ret = 4;
    } else {
      bool conv = true;
      for (int c = 0; c < na; ++c) {
        const double est = S.bn[c] > 0.0 ? S.res[c] / S.bn[c] : 0.0;
        if (hrow < P.hist_cap) P.proj[P.oHist + (size_t)hrow * na + c] = est;
        if (!(est <= P.tol)) conv = false;
      }
      ret = conv ? 1 : 0;
    }
    s_ret = ret;
  }
  __syncthreads();
  cstamp(P, q, 19);
  return s_ret;
}

// Y = R^-1 (Q^T rhs)[:n1] with R = [[I, Bmat], [0, R_H]] (hostls.cpp:175-182):
// y_H by a column-oriented back substitution over the packed R_H (one warp
// per right-hand side, lanes own rows), then y_top = c_top - Bmat y_H.
// Y is stored rhs-major (na x n1).
static __device__ void ctl_solve_y(const CycleArgs& P, const Ctl& S, int m) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int k = P.k, b = P.sb, ldq = P.ldq, n1 = k + m;
  double* rinv = S.cols;  // m <= b * ldq
  for (int i = threadIdx.x; i < m; i += kOrthT) {
    const int q = i / b, c = i % b;
    rinv[i] = 1.0 / S.Rp[rp_off(q, b) + (size_t)c * (q + 1) * b + i];
  }
  __syncthreads();
  for (int r = wid; r < P.na; r += kOrthT / 32) {
    double* y = S.ybuf + (size_t)r * 96;
    const double* cr = S.Cq + (size_t)r * ldq + k;
    double c[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) c[u] = (lane + 32 * u < m) ? cr[lane + 32 * u] : 0.0;
    for (int i = m - 1; i >= 0; --i) {
      const int slot = i >> 5;
      const double ci = slot == 0 ? c[0] : (slot == 1 ? c[1] : c[2]);
      const double yi = __shfl_sync(0xffffffffu, ci, i & 31) * rinv[i];
      if (lane == 0) y[i] = yi;
      const int q = i / b, cc = i % b, h = (q + 1) * b;
      const double* Rcol = S.Rp + rp_off(q, b) + (size_t)cc * h;
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int t = lane + 32 * u;
        if (t < i && t < h) c[u] -= Rcol[t] * yi;
      }
    }
    __syncwarp();
    for (int i = lane; i < m; i += 32) P.proj[P.oY + (size_t)r * n1 + k + i] = y[i];
  }
  __syncthreads();
  // y_top = c_top - Bmat y_H, Bmat staged into the (now free) packed-R space
  const size_t rp_cap = (size_t)b * b * P.nblk * (P.nblk + 1) / 2;
  const bool staged = (size_t)k * m <= rp_cap;
  double* Bs = S.Rp;
  if (staged)
    for (int x = threadIdx.x; x < k * m; x += kOrthT)
      Bs[x] = __ldcg(P.proj + P.oBmat + (size_t)(x / m) * P.cap + x % m);
  __syncthreads();
  for (int x = threadIdx.x; x < k * P.na; x += kOrthT) {
    const int i = x / P.na, r = x % P.na;
    const double* y = S.ybuf + (size_t)r * 96;
    double s = 0.0;
    if (staged) {
      for (int t = 0; t < m; ++t) s += Bs[(size_t)i * m + t] * y[t];
    } else {
      for (int t = 0; t < m; ++t) s += __ldcg(P.proj + P.oBmat + (size_t)i * P.cap + t) * y[t];
    }
    P.proj[P.oY + (size_t)r * n1 + i] = S.Cq[(size_t)r * ldq + i] - s;
  }
  __syncthreads();
}

// barrier over the worker blocks only (the control block runs on its own):
// a monotone arrival counter, target = episodes x workers
struct WBar {
  int* ctr;
  int n, epoch, wi;  // workers, episodes so far, this block's worker index
};

static __device__ __forceinline__ void wbar(WBar& w) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int target = (w.epoch + 1) * w.n;
#if PMP_BAR_ACQREL
    // release the block's writes with the arrival, acquire everyone's with
    // the final observation (no full fences)
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(w.ctr) : "memory");
    int v;
    do {
      asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(w.ctr) : "memory");
    } while (v < target);
#else
    __threadfence();
    atomicAdd(w.ctr, 1);
    while (*(volatile int*)w.ctr < target) {
    }
    __threadfence();
#endif
  }
  ++w.epoch;
  __syncthreads();
}

// grid_reduce (orth_dev.cuh) over the worker blocks of a group: block
// partials in slots 1 .. n (slot 0 belongs to the control block)
// (out of line with the barrier state by value: a WBar& parameter of an
// out-of-line function forced the callers' barrier state into local memory,
// so every barrier of the step loop paid local loads / stores)
static __device__ __noinline__ int wreduce_impl(int* ctr, int nw, int epoch, int wi, double* partial,
                                                double* gout, int K, double* G, double* out,
                                                int split, double* out2) {
  WBar wb{ctr, nw, epoch, wi};
  wbar(wb);
  const int nb = wb.n, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = wb.wi + nb * wid; o < K; o += nb * (kOrthT / 32)) {
    double s;
    if (nb <= 512) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int b = lane + 32 * u;
        v[u] = b < nb ? __ldcg(partial + (size_t)(b + 1) * K + o) : 0.0;
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
        t0 += __ldcg(partial + (size_t)(b + 1) * K + o);
        t1 += __ldcg(partial + (size_t)(b + 33) * K + o);
      }
      if (b < nb) t0 += __ldcg(partial + (size_t)(b + 1) * K + o);
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
  wbar(wb);
  for (int o = threadIdx.x; o < K; o += kOrthT) G[o] = __ldcg(gout + o);
  __syncthreads();
  return wb.epoch;
}

static __device__ __forceinline__ void wreduce(WBar& wb, double* partial, double* gout, int K,
                                               double* G, double* out, int split, double* out2) {
  wb.epoch = wreduce_impl(wb.ctr, wb.n, wb.epoch, wb.wi, partial, gout, K, G, out, split, out2);
}

// step outputs, double-buffered by step parity: B (k x sb), H1, H2 (cap x
// sb), R (sb x sb), all row-major with ld sb
struct StepBuf {
  double *B, *H1, *H2, *R;
};
static __device__ __forceinline__ StepBuf step_buf(const CycleArgs& P, int q) {
  const size_t one = (size_t)(P.kc + 2 * P.cap + P.sb) * P.sb;
  double* base = P.sbuf + (q & 1) * one;
  StepBuf s;
  s.B = base;
  s.H1 = base + (size_t)P.kc * P.sb;
  s.H2 = s.H1 + (size_t)P.cap * P.sb;
  s.R = s.H2 + (size_t)P.cap * P.sb;
  return s;
}

// flags in d_istate: [7] steps published, [8] workers done, [9] barrier
// counter, [16 + j] decision of step j (-1 until the control block posts it)
static __device__ __forceinline__ int wait_flag(const int* f, int cmp_ge) {
  __shared__ int s_v;
  if (threadIdx.x == 0) {
    int v;
    while ((v = *(volatile const int*)f) < cmp_ge) {
    }
    __threadfence();
    s_v = v;
  }
  __syncthreads();
  const int v = s_v;
  __syncthreads();
  return v;
}

// The control block: absorb each published step while the workers run the
// next one; post its decision (0 continue, 1 converged, 4 G deficient).
#ifndef PMP_CTL_NOINLINE
#define PMP_CTL_NOINLINE 1
#endif
#if PMP_CTL_NOINLINE
// (out of line, the state block by value: the control block's code no
// longer shares a register allocation with the workers' step loop)
#define PMP_CTL_RUN_ATTR __noinline__
#define PMP_CTL_REF
#else
#define PMP_CTL_RUN_ATTR
#define PMP_CTL_REF &
#endif
template <int NY>
__device__ PMP_CTL_RUN_ATTR void ctl_run(const CycleArgs& P, const Ctl PMP_CTL_REF S) {
  const int sb = P.sb;
  int hrow = 0, j = 0, total = P.ist[1];
  __shared__ int s_go;
  while (true) {
    if (threadIdx.x == 0) {
      int go;
      while (true) {
        if (*(volatile int*)(P.ist + 7) > j) {
          go = 1;
          break;
        }
        if (*(volatile int*)(P.ist + 8) != 0) {
          // workers finished: a step published just before is still absorbed
          go = *(volatile int*)(P.ist + 7) > j ? 1 : 0;
          break;
        }
      }
      __threadfence();
      s_go = go;
    }
    __syncthreads();
    if (!s_go) break;
    // this step's outputs -> shared memory
    const StepBuf sbf = step_buf(P, j);
    for (int x = threadIdx.x; x < (P.k + total) * sb; x += kOrthT)
      S.bh1[x] = x < P.k * sb ? __ldcg(sbf.B + x) : __ldcg(sbf.H1 + x - P.k * sb);
    for (int x = threadIdx.x; x < total * sb; x += kOrthT) S.h2[x] = __ldcg(sbf.H2 + x);
    for (int x = threadIdx.x; x < sb * sb; x += kOrthT) S.Rr[x] = __ldcg(sbf.R + x);
    __syncthreads();
    const int d = ctl_absorb<NY>(P, S, j, total, hrow);
    if (d != 4) ++hrow;
    if (threadIdx.x == 0) {
      __threadfence();
      *(volatile int*)(P.ist + 16 + j) = d;
    }
    ++j;
    total += sb;
  }
  // final state of the workers (written before the done flag)
  const int m = __ldcg(P.ist + 0), status = __ldcg(P.ist + 4);
  if (status != 5 && status != 4 && m > 0) ctl_solve_y(P, S, m);
  __syncthreads();
  cstamp(P, 63, 29);
  if (threadIdx.x == 0) P.ist[5] = hrow;
}


// The worker side of one cycle's inner loop (k_cycle / k_solve): steps until
// restart length, max_iters, a stop decision of the control block, or a
// Cholesky flag; the group's lead worker writes the final state and the
// done flag.  m / total / ncols / it / status are updated in place.
struct WSmem {
  double *G, *R1, *R2, *red;
  int *piv, *piv2, *flag;
  double *Xs, *Wv, *Q1;
  int ldw;
  double* ring = nullptr;  // free shared memory of a global-row worker (spmm_auto)
  int ring_doubles = 0;
};

// The block step's tall-skinny products for the shared-memory geometries:
// the scalar thread-per-row / lane-per-column forms (default), or FP64
// tensor-core fragments loaded straight from global memory (PMP_MMA=1;
// measured slower there -- c2 161 -> 176 us per block step -- the
// global-row geometry stages its operands instead, stage_dev.cuh).
#ifndef PMP_MMA
#define PMP_MMA 0
#endif
#ifndef PMP_GRAM_FLAT
#define PMP_GRAM_FLAT 1
#endif
#if PMP_MMA
#define PMP_STEP_GRAM block_gram_mma<NY>
#define PMP_STEP_UPDATE block_update_mma<NY>
#else
#define PMP_STEP_GRAM block_gram<NY>
#define PMP_STEP_UPDATE block_update<NY>
#endif

// OPT: per-instance code-generation choices of the step loop (measured per
// geometry, profiles/r02_codegen_ab.txt): kOptStamp keeps the phase stamps
// compiled in, kOptCA gathers the SpMM's X rows through L1, kOptFlat uses
// the flat Gram thread layout.
constexpr int kOptStamp = 1, kOptCA = 2, kOptFlat = 4, kOptCyc = 8, kOptFuse = 16;
template <bool CACHED, int NY, int OPT = 0>
__device__ void worker_inner(const CycleArgs& P, WBar& wb, const WSmem& S_, int r0, int nr,
                             bool lead, int& m, int& total, int& ncols, int& it, int& status) {
  double* G = S_.G;
  double* R1 = S_.R1;
  double* R2 = S_.R2;
  double* red = S_.red;
  int* piv = S_.piv;
  int* piv2 = S_.piv2;
  int* flag = S_.flag;
  double* Xs = S_.Xs;
  double* Wv = S_.Wv;
  double* Q1 = S_.Q1;
  const int ldw = S_.ldw;
  const int sb = P.sb, k = P.k, cap = P.cap, kc = P.kc, ldx = P.ldx;
  int q = 0;
  const int it_start = it;
  while (true) {
    if (it >= P.max_iters || m >= P.inner_restart) {
      status = it >= P.max_iters ? 3 : 2;
      if (q > 0) {
        const int d = wait_flag(P.ist + 16 + q - 1, 0);
        if (d == 1) status = 0;
        if (d == 4) status = 4;
      }
      break;
    }
    const int q0 = m;
    const int stp = it - it_start;
    const StepBuf sbf = step_buf(P, q);
    wstamp<(OPT & kOptStamp) != 0>(P, stp, 0);
    // ---- W = A F_0 .. F_{nfac-1} V[:, q0 : q0 + sb] ---------------------------
    const double* src = P.V + q0;
    int lds = cap;
    if ((OPT & kOptCyc) && P.wglob) {
      // tiles dealt cyclically over the group's workers; W's rows come from
      // other blocks, hence the extra group barrier
      for (int f = P.nfac - 1; f >= 0; --f) {
        double* dst = ((P.nfac - 1 - f) & 1) ? P.T1 : P.T0;
        spmm_rows_cyc<NY, (OPT & kOptCA) != 0>(P.frp[f], P.fci[f], P.fva[f], src, lds, sb, dst, P.s,
                                                P.n, wb.wi, wb.n);
        wbar(wb);
        src = dst;
        lds = P.s;
      }
      spmm_rows_cyc<NY, (OPT & kOptCA) != 0>(P.arp, P.aci, P.ava, src, lds, sb, P.W, P.s, P.n, wb.wi,
                                              wb.n);
      wbar(wb);
    } else {
    for (int f = P.nfac - 1; f >= 0; --f) {
      double* dst = ((P.nfac - 1 - f) & 1) ? P.T1 : P.T0;
      spmm_auto<NY, (OPT & kOptCA) != 0>(P.frp[f], P.fci[f], P.fva[f], src, lds, sb,
                                          dst + (size_t)r0 * P.s, P.s, r0, nr, S_.ring,
                                          S_.ring_doubles);
      wbar(wb);
      src = dst;
      lds = P.s;
    }
    spmm_auto<NY, (OPT & kOptCA) != 0>(P.arp, P.aci, P.ava, src, lds, sb, Wv, ldw, r0, nr, S_.ring,
                                        S_.ring_doubles);
    }
    __syncthreads();
    wstamp<(OPT & kOptStamp) != 0>(P, stp, 1);

    // ---- R1: [C | V]^T W --------------------------------------------------------
    const int kx = k + total;
    const Rows CV = CACHED ? Rows{Xs, ldx, kx, Xs, ldx}
                           : Rows{P.C + (size_t)r0 * kc, kc, k, P.V + (size_t)r0 * cap, cap};
    const double* Vrows = CACHED ? Xs + k : P.V + (size_t)r0 * cap;
    const int ldvr = CACHED ? ldx : cap;
    const Rows Vonly{Vrows, ldvr, total, Vrows, ldvr};
    if ((OPT & kOptFlat) && kx <= 128)
      block_gram_flat<NY>(CV, kx, Wv, ldw, sb, nr, red, P.partial, wb.wi + 1);
    else
      PMP_STEP_GRAM(CV, kx, Wv, ldw, sb, nr, red, P.partial, wb.wi + 1);
    wstamp<(OPT & kOptStamp) != 0>(P, stp, 2);
    wreduce(wb, P.partial, P.gout, kx * sb, G, sbf.B, k * sb, sbf.H1);
    wstamp<(OPT & kOptStamp) != 0>(P, stp, 3);
    PMP_STEP_UPDATE(CV, kx, Wv, ldw, sb, nr, G);
    wstamp<(OPT & kOptStamp) != 0>(P, stp, 4);
    // ---- R2: [V | W1]^T W1 ------------------------------------------------------
    const int kx2 = total + sb;
    {
      const Rows VW{Vrows, ldvr, total, Wv, ldw};
      if ((OPT & kOptFlat) && kx2 <= 128)
        block_gram_flat<NY>(VW, kx2, Wv, ldw, sb, nr, red, P.partial, wb.wi + 1);
      else
        PMP_STEP_GRAM(VW, kx2, Wv, ldw, sb, nr, red, P.partial, wb.wi + 1);
      wstamp<(OPT & kOptStamp) != 0>(P, stp, 5);
      wreduce(wb, P.partial, P.gout, kx2 * sb, G, sbf.H2, total * sb, nullptr);
      wstamp<(OPT & kOptStamp) != 0>(P, stp, 6);
    }
    // G_W = W1^T W1 - H2^T H2 (into R2 as scratch), then W2 = W1 - V H2
    const int n4 = 4 * sb * sb, lim4 = (n4 + 31) & ~31;
    for (int q4 = threadIdx.x; q4 < lim4; q4 += kOrthT) {
      const bool act = q4 < n4;
      const int qq = q4 >> 2, part = q4 & 3;
      const int i = act ? qq / sb : 0, j = act ? qq % sb : 0;
      double s = 0.0;
      if (act)
        for (int t = part; t < total; t += 4) s += G[t * sb + i] * G[t * sb + j];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (act && part == 0) R2[qq] = G[(size_t)(total + i) * sb + j] - s;
    }
    __syncthreads();
#ifdef PMP_STAMPS
    wstamp<(OPT & kOptStamp) != 0>(P, stp, 12);
#endif
    // kOptFuse (global-row instance): the Cholesky factor of G_W does not
    // depend on W2, so it is taken first (G_W symmetrised into `red`: G still
    // holds H2) and, when one Cholesky-QR pass suffices, W2 = W1 - V H2 goes
    // straight into the new V block (block_update_trsm); otherwise the
    // original order below.
    constexpr bool kFuse = (OPT & kOptFuse) != 0 && !CACHED;
    bool fused_done = false;
    if (!kFuse) PMP_STEP_UPDATE(Vonly, total, Wv, ldw, sb, nr, G);
#ifdef PMP_STAMPS
    wstamp<(OPT & kOptStamp) != 0>(P, stp, 13);
#endif
    double* Gs = kFuse ? red : G;  // the symmetrised G_W
    for (int qq = threadIdx.x; qq < sb * sb; qq += kOrthT) {
      const int i = qq / sb, j = qq % sb;
      Gs[qq] = 0.5 * (R2[i * sb + j] + R2[j * sb + i]);
    }
    __syncthreads();
#ifdef PMP_STAMPS
    wstamp<(OPT & kOptStamp) != 0>(P, stp, 14);
#endif
#ifdef PMP_STAMPS
    if (P.dbg && blockIdx.x == 1 && stp == 2)
      for (int q = threadIdx.x; q < sb * sb; q += kOrthT)
        P.dbg[(size_t)40 * 64 + q] = (unsigned long long)__double_as_longlong(G[q]);
    __syncthreads();
#endif
    if (threadIdx.x < 32) {
#ifdef PMP_STAMPS
      const long long c0 = clock64();
#endif
#ifdef PMP_CHOL_REG
      bool ok = warp_cholesky_reg<NY>(Gs, sb, R1, piv, true, kCholRatio);
#else
      bool ok = warp_cholesky_smem(Gs, sb, R1, piv, true, kCholRatio);
#endif
      if (threadIdx.x == 0) flag[0] = ok ? 0 : 1;
#ifdef PMP_STAMPS
      const long long c1 = clock64();
      if (P.dbg && blockIdx.x == 1 && threadIdx.x == 0 && stp < 64)
        P.dbg[((size_t)stp * 32 + 16) * 2 + 1] = (unsigned long long)(c1 - c0);
#endif
    }
    __syncthreads();
    wstamp<(OPT & kOptStamp) != 0>(P, stp, 7);
    bool single = false;
    if (flag[0] == 0) single = fabs(R1[0]) / fabs(R1[(sb - 1) * sb + (sb - 1)]) <= kSkipKappa;
    if (kFuse) {
      if (flag[0] == 0 && single) {
        block_update_trsm<NY>(Vonly, total, Wv, ldw, sb, nr, G, R1, piv,
                              P.V + (size_t)r0 * cap + total, cap);
        fused_done = true;
      } else {
        PMP_STEP_UPDATE(Vonly, total, Wv, ldw, sb, nr, G);
      }
    }
    if (flag[0] == 0 && !single) {
#ifdef PMP_STAMPS
      if (P.dbg && lead && threadIdx.x == 0 && stp < 64)
        P.dbg[((size_t)stp * 32 + 15) * 2 + 1] = 1;  // this step took the R3 pass
#endif
      block_trsm_rows<NY>(Wv, ldw, Q1, sb, nr, sb, R1, piv);
      const Rows Qv{Q1, sb, sb, Q1, sb};
      block_gram<NY>(Qv, sb, Q1, sb, sb, nr, red, P.partial, wb.wi + 1);
      wreduce(wb, P.partial, P.gout, sb * sb, G, nullptr, 0, nullptr);
      if (threadIdx.x < 32) {
        bool ok = warp_cholesky_smem(G, sb, R2, piv2, false, 0.0);
        if (threadIdx.x == 0) flag[0] = ok ? 0 : 1;
      }
      __syncthreads();
    }
    wstamp<(OPT & kOptStamp) != 0>(P, stp, 8);
    if (flag[0]) {
      // grid-uniform: Cholesky cannot decide the rank -> host Householder
      // (unless the previous step already converged / was deficient)
      for (int qq = threadIdx.x; qq < nr * sb; qq += kOrthT)
        P.W[(size_t)(r0 + qq / sb) * P.s + qq % sb] = Wv[(size_t)(qq / sb) * ldw + qq % sb];
      status = 5;
      if (q > 0) {
        const int d = wait_flag(P.ist + 16 + q - 1, 0);
        if (d == 1) status = 0;
        if (d == 4) status = 4;
      }
      if (status == 5 && lead && P.mirror) {
        // the step's B / H1 / H2 for the host fallback (krylov.py
        // _native_cycle status 5)
        const int lens[3] = {k * sb, total * sb, total * sb};
        const int offs[3] = {P.offB, P.offH1, P.offH2};
        const double* srcs[3] = {sbf.B, sbf.H1, sbf.H2};
        for (int a = 0; a < 3; ++a)
          for (int qq = threadIdx.x; qq < lens[a]; qq += kOrthT)
            P.mirror[offs[a] + qq] = __ldcg(srcs[a] + qq);
      }
      break;
    }
    // ---- Q -> V[:, total : total + sb] -------------------------------------------
    {
      double* qd = CACHED ? Xs + k + total : P.V + (size_t)r0 * cap + total;
      const int ldqd = CACHED ? ldx : cap;
      if (fused_done) {
        // (the new block is in V already)
      } else if (single)
        block_trsm_rows<NY>(Wv, ldw, qd, ldqd, nr, sb, R1, piv);
      else
        block_trsm_rows<NY>(Q1, sb, qd, ldqd, nr, sb, R2, nullptr);
      if (CACHED)
        for (int qq = threadIdx.x; qq < nr * sb; qq += kOrthT)
          P.V[(size_t)(r0 + qq / sb) * cap + total + qq % sb] =
              qd[(size_t)(qq / sb) * ldx + qq % sb];
    }
    if (lead) {
      // R = R2 R1 (pivoted order), un-pivoted: R[i, piv[c]] = R'[i, c]
      for (int qq = threadIdx.x; qq < sb * sb; qq += kOrthT) {
        const int i = qq / sb, c = qq % sb;
        double s = 0.0;
        if (single) {
          s = R1[i * sb + c];
        } else {
          for (int a = i; a <= c; ++a) s += R2[i * sb + a] * R1[a * sb + c];
        }
        sbf.R[i * sb + piv[c]] = (c >= i) ? s : 0.0;
      }
    }
    wstamp<(OPT & kOptStamp) != 0>(P, stp, 9);
    wbar(wb);  // new V block (and the step outputs) visible
    wstamp<(OPT & kOptStamp) != 0>(P, stp, 10);
    // the previous step's decision (the control block absorbed it meanwhile)
    if (q > 0) {
      const int d = wait_flag(P.ist + 16 + q - 1, 0);
      if (d == 1 || d == 4) {
        status = d == 1 ? 0 : 4;
        break;
      }
    }
    wstamp<(OPT & kOptStamp) != 0>(P, stp, 11);
    if (lead && threadIdx.x == 0) {
      __threadfence();
      *(volatile int*)(P.ist + 7) = q + 1;  // publish step q to the control block
    }
    ++q;
    ncols += (ncols == 0) ? k + sb : sb;
    ++it;
    m = total;
    total += sb;
  }
  if (lead && threadIdx.x == 0) {
    P.ist[0] = m;
    P.ist[1] = total;
    P.ist[2] = ncols;
    P.ist[3] = it;
    P.ist[4] = status;
    __threadfence();
    *(volatile int*)(P.ist + 8) = 1;  // done: the control block finishes up
  }
}

}  // namespace pmp
