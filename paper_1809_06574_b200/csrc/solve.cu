// Whole block-GCRO solves on the device, several systems per launch
// (krylov.py:105-275 end to end).
//
// k_cycle (cycle.cu) moved the inner loop of a cycle onto the device; the
// cycle boundaries -- projecting the residual block against the outer space
// and orthonormalising it (krylov.py:156-169), the solution / true residual
// update (krylov.py:221-234) and the outer-space fold (krylov.py:244-269) --
// still cost host round trips, and one system at a time leaves most of the
// GPU idle (every phase is latency bound).  k_solve runs complete solves:
// the grid is split into groups of blocks, one independent system per
// group (the sequence driver solves the systems of a parameter sweep in
// batches), each group = one control block (the projected least-squares
// problem, as in k_cycle) + worker blocks that own row ranges.
//
// Per cycle (group-local barriers only):
//   Z = R[:, act]; Z -= C (C^T Z); Cholesky-QR2 -> V[:, :na], S0 = R
//   inner loop (worker_inner / ctl_run, cycle_dev.cuh)
//   dX = V Y_v + U Y_u; Xt[:, act] += dX; X[:, act] = P Xt[:, act];
//   R[:, act] = B[:, act] - A X[:, act]; true residual norms; stop test
//   fold: images = V G_v Y + C G_c Y, block CGS2 against C (2 reductions),
//   Cholesky with the reference's drop test (|w2| > 1e-10 |w|), one or two
//   Cholesky-QR passes -> new C / U columns; keep the last outer_dim.
// Every decision the fast path cannot take exactly the way the reference
// does (rank-deficient blocks: krylov.py:79-95 deflation, a rank-deficient
// projected problem, a drop test inside the cancellation band) ends the
// group with status PMP_SOLVE_FALLBACK and the host re-solves that system
// on the host-driven path.
#include "stage_dev.cuh"

namespace pmp {

struct SysDesc {
  int nfac;  // factors in this system's preconditioner chain (0 .. 3)
  const int32_t* frp[3];
  const int32_t* fci[3];
  const double* fva[3];
  const int32_t* arp;
  const int32_t* aci;
  const double* ava;
  const double* B;
  double* X;
};

struct SolveArgs {
  int n, s, cap, kc, outer_dim, inner_restart, max_iters;
  int gsz, rows_per_block, ldx, hist_cap, log_cap, isz;
  int wglob;  // W rows in global memory (rows beyond shared memory)
  int stage_rows, stage_n;  // global-row geometry: staged ring (doubles per stage, stages)
  int region_doubles;       // the block's `region` of shared memory (doubles)
  double tol;
  const SysDesc* sys;
  double* ws;
  size_t wsz;
  int* ist;
  size_t oV, oC, oU, oW, oT0, oT1, oQ1, oXt, oR, oDX, oRB, oZ, oPart, oGout, oSbuf, oProj, oLog,
      oAux;
  int pBmat, pHb, pCq, pY, pRes, pBn, pHist;  // offsets inside the projected-state block
  int pCtl;        // the control block's state in GLOBAL memory (ctl_global), else unused
  int ctl_global;  // global-row geometry without the staged ring: no shared-memory region
  unsigned long long* dbg;  // diagnostics (group 0): stamps at (32 it + phase) * 2 + block
  int nsys, groups;          // systems in the queue, concurrent block groups
  int* queue;                // next-system counter (zeroed at launch)
  int* rint;                 // nsys x PMP_SOLVE_RSZ ints: per-system record
  double* rdbl;              // nsys x (2 + log_cap * s): algorithmic bytes (strict, 8(d)), residual log
};

// solve-level int state (after the cycle-level [0, 144))
enum {
  kNa = 144,
  kK = 145,
  kIt = 146,
  kStatus = 147,
  kLogRows = 148,
  kMatvecs = 149,
  kPrec = 150,
  kGbar = 151,
  kFold = 152,
  kReason = 153,  // fallback reason: 1 cycle-start QR, 2/3 inner status 4/5, 4/5 fold
  kNext = 154,    // the group's next system (taken from the queue by the control block)
  kAct = 160,  // active columns (<= 16)
};

// per-system record (PmpSolveBatch::d_result): status, reason, iterations,
// active columns left, log rows, matvecs, preconditioner applies
enum { rStatus = 0, rReason, rIt, rNa, rLogRows, rMatvecs, rPrec, PMP_SOLVE_RSZ = 8 };

constexpr int PMP_SOLVE_OK = 0, PMP_SOLVE_FALLBACK = 10;

// barrier over every block of the group (control block included)
__device__ __forceinline__ void gbar(WBar& g) { wbar(g); }

__device__ __forceinline__ int ldv(const int* p) { return *(volatile const int*)p; }

// diagnostics: cycle-level phase stamps of group 0's lead worker
__device__ __forceinline__ void sstamp(const SolveArgs& A, int grp, int cyc, int ph) {
#ifdef PMP_STAMPS
  if (A.dbg && grp == 0 && blockIdx.x == 1 && threadIdx.x == 0 && cyc < 16) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    A.dbg[((size_t)(48 + cyc) * 32 + ph) * 2 + 1] = t;
  }
#else
  (void)A;
  (void)grp;
  (void)cyc;
  (void)ph;
#endif
}

// d[c] = sum_{t < m} a[t] G[(ga + t) na + c] + sum_{t < kb} b[t] G[(gb + t) na + c]
// for c < na: one row, all outputs (each a / b element loaded once); per
// output the same summation order as the element-wise loop it replaces
template <int NY>
__device__ __forceinline__ void row_combo(const double* a, int m, int ga, const double* b, int kb,
                                          int gb, const double* G, int na, double* d) {
#pragma unroll
  for (int c = 0; c < NY; ++c) d[c] = 0.0;
#pragma unroll 4
  for (int t = 0; t < m; ++t) {
    const double x = a[t];
    const double* g = G + (size_t)(ga + t) * na;
#pragma unroll
    for (int c = 0; c < NY; ++c)
      if (c < na) d[c] += x * g[c];
  }
#pragma unroll 4
  for (int t = 0; t < kb; ++t) {
    const double x = b[t];
    const double* g = G + (size_t)(gb + t) * na;
#pragma unroll
    for (int c = 0; c < NY; ++c)
      if (c < na) d[c] += x * g[c];
  }
}

// one row of [w | z] (columns keep[a], or 0..nk-1 when keep is null) times
// T^-1 (upper, ld ldt) -> yw / yz; register arrays with static indices
template <int NY>
__device__ __forceinline__ void fold_rowsolve(const double* w, const double* z, const int* keep,
                                              int nk, const double* T, int ldt, double* yw_out,
                                              double* yz_out) {
  double yw[NY], yz[NY];
#pragma unroll
  for (int a = 0; a < NY; ++a) {
    yw[a] = 0.0;
    yz[a] = 0.0;
    if (a < nk) {
      const int col = keep ? keep[a] : a;
      double vw = w[col], vz = z[col];
#pragma unroll
      for (int b = 0; b < NY; ++b)
        if (b < a) {
          vw -= yw[b] * T[b * ldt + a];
          vz -= yz[b] * T[b * ldt + a];
        }
      yw[a] = vw / T[a * ldt + a];
      yz[a] = vz / T[a * ldt + a];
    }
  }
#pragma unroll
  for (int a = 0; a < NY; ++a)
    if (a < nk) {
      yw_out[a] = yw[a];
      yz_out[a] = yz[a];
    }
}

// The cycle boundaries' Gram products: the flat thread layout in the
// global-row instance (few columns -- k + na <= 18 -- leave half of
// block_gram's lanes idle), block_gram elsewhere.
#ifndef PMP_BOUNDARY_FLAT
#define PMP_BOUNDARY_FLAT 1
#endif
template <int NY, bool FLAT>
__device__ __forceinline__ void gram_b(const Rows X, int kx, const double* Y, int ldy, int ny,
                                       int nrows, double* red, double* partial, int slot) {
  if (FLAT && NY <= 8 && PMP_BOUNDARY_FLAT && kx <= 128)  // (s = 16: 1168 -> 1186 ms, off)
    block_gram_flat<NY>(X, kx, Y, ldy, ny, nrows, red, partial, slot);
  else
    block_gram<NY>(X, kx, Y, ldy, ny, nrows, red, partial, slot);
}

#ifndef PMP_FOLD_EXACT
#define PMP_FOLD_EXACT 1
#endif

#if PMP_FOLD_EXACT
// The fold of a block whose Gram-based drop test falls inside the
// cancellation band, column by column as the reference does it
// (krylov.py:249-265): each image column (already projected against C twice,
// as a block) is orthogonalised twice against the columns kept so far in
// this fold, its norm is recomputed from the vector and the 1e-10 drop test
// applied; kept columns go straight to C / U.  Grid reductions per column:
// a rare path (it replaced a host re-solve of the whole system).  Out of
// line, barrier state by value; returns the group barrier epoch, the number
// of kept columns in *nk_out.
template <int NY>
__device__ __noinline__ int fold_exact(int* ctr, int nwk, int epoch, int wi, double* Cr, double* Ur,
                                       int kc, int k, double* Wr, double* Zr, int s,
                                       const double* w0, int na, int nr, double* red,
                                       double* partial, double* gout, double* G, int slot,
                                       int* nk_out) {
  WBar wb{ctr, nwk, epoch, wi};
  int nk = 0;
  for (int j = 0; j < na; ++j) {
    if (w0[j] == 0.0) continue;
    for (int pass = 0; pass < 2 && nk > 0; ++pass) {
      const Rows Qc{Cr + k, kc, nk, Cr + k, kc};
      const Rows Qu{Ur + k, kc, nk, Ur + k, kc};
      block_gram<1>(Qc, nk, Wr + j, s, 1, nr, red, partial, slot);
      wreduce(wb, partial, gout, nk, G, nullptr, 0, nullptr);
      block_update<1>(Qc, nk, Wr + j, s, 1, nr, G);
      block_update<1>(Qu, nk, Zr + j, s, 1, nr, G);
    }
    const Rows Wj{Wr + j, s, 1, Wr + j, s};
    block_gram<1>(Wj, 1, Wr + j, s, 1, nr, red, partial, slot);
    wreduce(wb, partial, gout, 1, G, nullptr, 0, nullptr);
    const double nw = sqrt(fmax(G[0], 0.0));
    if (!(nw > 1e-10 * w0[j])) continue;
    for (int r = threadIdx.x; r < nr; r += kOrthT) {
      Cr[(size_t)r * kc + k + nk] = Wr[(size_t)r * s + j] / nw;
      Ur[(size_t)r * kc + k + nk] = Zr[(size_t)r * s + j] / nw;
    }
    __syncthreads();
    ++nk;
  }
  if (threadIdx.x == 0) *nk_out = nk;
  __syncthreads();
  return wb.epoch;
}
#endif

template <bool CACHED, int NY, bool WG>
#ifndef PMP_MINB
#define PMP_MINB 2
#endif
__global__ void __launch_bounds__(kOrthT, PMP_MINB) k_solve(SolveArgs A) {
  extern __shared__ __align__(16) double sh[];
  const int grp = blockIdx.x / A.gsz, lb = blockIdx.x % A.gsz;
  const bool ctl = lb == 0;
  const bool lead = lb == 1;
  const int wi = lb - 1, nw = A.gsz - 1;
  double* ws = A.ws + (size_t)grp * A.wsz;
  int* ist = A.ist + (size_t)grp * A.isz;
  const int n = A.n, s = A.s, cap = A.cap, kc = A.kc;
  const int r0 = ctl ? 0 : wi * A.rows_per_block;
  const int r1 = ctl ? 0 : min(n, r0 + A.rows_per_block);
  const int nr = max(0, r1 - r0);

  const int kmax = (kc + cap + s) * s;
  double* p = sh;
  double* G = p;
  p += kmax;
  double* R1 = p;
  p += s * s;
  double* R2 = p;
  p += s * s;
  double* red = p;
  p += 8 * 32 * s;
  int* piv = reinterpret_cast<int*>(p);
  int* piv2 = piv + 16;
  int* flag = piv + 32;
  p += 20;
  double* region = p;

  double* V = ws + A.oV;
  double* C = ws + A.oC;
  double* U = ws + A.oU;
  double* W = ws + A.oW;
  double* Xt = ws + A.oXt;
  double* Rr = ws + A.oR;
  double* DX = ws + A.oDX;
  double* RB = ws + A.oRB;
  double* Z = ws + A.oZ;
  double* partial = ws + A.oPart;
  double* gout = ws + A.oGout;
  double* proj = ws + A.oProj;
  double* logp = ws + A.oLog;
  double* aux = ws + A.oAux;
  double* bn = aux;          // s: |B[:, c]|
  double* pn = aux + 16;     // s: |R[:, c]| at the last true residual
  double* lrel = aux + 32;   // s: last relative residual row
  double* img = aux + 64;    // (kc + cap) x s: G Y (fold images), row-major ld s
  // The control block's projected-problem state: its shared-memory region, or
  // (global-row geometry without the staged ring) global memory.  There the
  // workers use no region at all, so keeping the ~60 KB out of every block's
  // shared memory leaves the SM a 4x larger L1 for the workers' row gathers
  // (measured on c4: profiles/r02_ctl_global_ab.txt); the control block runs
  // one step behind the workers and a step lasts milliseconds at these sizes,
  // so its slower state is invisible.
  double* ctl_mem = A.ctl_global ? proj + A.pCtl : region;
  int* act = ist + kAct;

  // the per-group argument block lives in SHARED memory: as a local struct
  // it sat in the (L1-starved) stack and every field read in the step loop
  // became an L2 round trip
  __shared__ CycleArgs L;
  __shared__ int acts[16];

  WBar wb{ist + 9, nw, 0, wi};
  WBar gb{ist + kGbar, A.gsz, 0, lb};
  const int slot = lb;  // partial slot of a worker (1 .. nw)

  // groups take systems from a queue: the first `groups` statically, the
  // rest in completion order (no group idles while a launch has systems
  // left; a launch lasts ~ the mean, not the max, of its solves)
  for (int sys = grp; sys < A.nsys;) {
  const SysDesc D = A.sys[sys];
  if (threadIdx.x == 0) {
  L.n = n;
  L.s = s;
  L.cap = cap;
  L.kc = kc;
  L.nfac = D.nfac;
  for (int i = 0; i < 3; ++i) {
    L.frp[i] = D.frp[i];
    L.fci[i] = D.fci[i];
    L.fva[i] = D.fva[i];
  }
  L.arp = D.arp;
  L.aci = D.aci;
  L.ava = D.ava;
  L.V = V;
  L.W = W;
  L.T0 = ws + A.oT0;
  L.T1 = ws + A.oT1;
  L.C = C;
  L.small = nullptr;
  L.mirror = nullptr;
  L.offB = L.offH1 = L.offH2 = L.offR = 0;
  L.partial = partial;
  L.gout = gout;
  L.Q1g = ws + A.oQ1;
  L.sbuf = ws + A.oSbuf;
  L.rows_per_block = A.rows_per_block;
  L.ldx = A.ldx;
  L.max_iters = A.max_iters;
  L.inner_restart = A.inner_restart;
  L.hist_cap = A.hist_cap;
  L.tol = A.tol;
  L.proj = proj;
  L.oBmat = A.pBmat;
  L.oHb = A.pHb;
  L.oQR = 0;
  L.oTau = 0;
  L.oCq = A.pCq;
  L.oY = A.pY;
  L.oRes = A.pRes;
  L.oBn = A.pBn;
  L.oHist = A.pHist;
  L.ist = ist;
  L.dbg = nullptr;
  L.wglob = A.wglob;
  }
  __syncthreads();

  // ---- setup: X = Xt = 0, R = B, column norms of B -----------------------------
  if (!ctl) {
    for (int q = threadIdx.x; q < nr * s; q += kOrthT) {
      const size_t o = (size_t)r0 * s + q;
      D.X[o] = 0.0;
      Xt[o] = 0.0;
      Rr[o] = D.B[o];
    }
    const double* Bv = D.B + (size_t)r0 * s;
    const Rows BB{Bv, s, s, Bv, s};
    gram_b<NY, WG>(BB, s, Bv, s, s, nr, red, partial, slot);
    wreduce(wb, partial, gout, s * s, G, nullptr, 0, nullptr);
    if (lead && threadIdx.x == 0) {
      int na = 0;
      for (int c = 0; c < s; ++c) {
        const double b = sqrt(fmax(G[c * s + c], 0.0));
        if (c == 0) aux[48] = aux[49] = 0.0;
        bn[c] = b;
        pn[c] = b;
        lrel[c] = b > 0.0 ? 1.0 : 0.0;
        logp[c] = lrel[c];
        if (b > 0.0) act[na++] = c;
      }
      ist[kNa] = na;
      ist[kK] = 0;
      ist[kIt] = 0;
      ist[kStatus] = PMP_SOLVE_OK;
      ist[kLogRows] = 1;
      ist[kMatvecs] = 0;
      ist[kPrec] = 0;
      ist[kReason] = 0;
    }
  }
  gbar(gb);

  int cyc = 0;
  while (true) {
    const int na = ldv(ist + kNa), k = ldv(ist + kK);
    int it = ldv(ist + kIt);
    const int it0 = it;
    if (na == 0 || it >= A.max_iters || ldv(ist + kStatus) != PMP_SOLVE_OK) break;
    const int ldq = k + cap;
    if (threadIdx.x == 0) {
      L.k = k;
      L.na = na;
      L.sb = na;
      L.ldq = ldq;
      L.nblk = (A.inner_restart + na - 1) / na + 1;
      // (diagnostic stamps of group 0, indexed by the global iteration)
      L.dbg = (A.dbg && grp == 0 && !ctl && it < 48) ? A.dbg + (size_t)it * 32 * 2 : nullptr;
      for (int c = 0; c < na; ++c) acts[c] = ldv(act + c);
    }
    __syncthreads();

    // ---- cycle start: Z = R[:, act] - C (C^T R[:, act]); QR -> V[:, :na] -------
    sstamp(A, grp, cyc, 0);
    if (!ctl) {
      double* Zw = W + (size_t)r0 * s;
      for (int q = threadIdx.x; q < nr * na; q += kOrthT) {
        const int r = q / na, c = q % na;
        Zw[(size_t)r * s + c] = Rr[(size_t)(r0 + r) * s + acts[c]];
      }
      __syncthreads();
      const StepBuf sbf = step_buf(L, 0);
      if (k > 0) {
        const Rows CV{C + (size_t)r0 * kc, kc, k, C + (size_t)r0 * kc, kc};
        gram_b<NY, WG>(CV, k, Zw, s, na, nr, red, partial, slot);
        wreduce(wb, partial, gout, k * na, G, sbf.B, k * na, nullptr);
        block_update<NY>(CV, k, Zw, s, na, nr, G);
      }
      {
        const Rows ZZ{Zw, s, na, Zw, s};
        gram_b<NY, WG>(ZZ, na, Zw, s, na, nr, red, partial, slot);
        wreduce(wb, partial, gout, na * na, G, nullptr, 0, nullptr);
      }
      for (int q = threadIdx.x; q < na * na; q += kOrthT) {
        const int i = q / na, j = q % na;
        R2[q] = 0.5 * (G[i * na + j] + G[j * na + i]);
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        const bool ok = warp_cholesky_smem(R2, na, R1, piv, true, kCholRatio);
        if (threadIdx.x == 0) flag[0] = ok ? 0 : 1;
      }
      __syncthreads();
      bool single = false;
      if (flag[0] == 0) single = fabs(R1[0]) / fabs(R1[(na - 1) * na + (na - 1)]) <= kSkipKappa;
      double* Q1 = L.Q1g + (size_t)r0 * na;
      if (flag[0] == 0 && !single) {
        block_trsm_rows<NY>(Zw, s, Q1, na, nr, na, R1, piv);
        const Rows Qv{Q1, na, na, Q1, na};
        gram_b<NY, WG>(Qv, na, Q1, na, na, nr, red, partial, slot);
        wreduce(wb, partial, gout, na * na, G, nullptr, 0, nullptr);
        if (threadIdx.x < 32) {
          const bool ok = warp_cholesky_smem(G, na, R2, piv2, false, 0.0);
          if (threadIdx.x == 0) flag[0] = ok ? 0 : 1;
        }
        __syncthreads();
      }
      if (flag[0]) {
        if (lead && threadIdx.x == 0) { ist[kStatus] = PMP_SOLVE_FALLBACK; ist[kReason] = 1; }
      } else {
        double* Vr = V + (size_t)r0 * cap;
        if (single)
          block_trsm_rows<NY>(Zw, s, Vr, cap, nr, na, R1, piv);
        else
          block_trsm_rows<NY>(Q1, na, Vr, cap, nr, na, R2, nullptr);
        if (lead) {
          // S0 = R2 R1 (pivoted order), un-pivoted
          for (int q = threadIdx.x; q < na * na; q += kOrthT) {
            const int i = q / na, c = q % na;
            double t = 0.0;
            if (single) {
              t = R1[i * na + c];
            } else {
              for (int a = i; a <= c; ++a) t += R2[i * na + a] * R1[a * na + c];
            }
            sbf.R[i * na + piv[c]] = (c >= i) ? t : 0.0;
          }
          if (threadIdx.x == 0) {
            ist[0] = 0;
            ist[1] = na;
            ist[2] = 0;
            ist[3] = it;
            ist[7] = 0;
            ist[8] = 0;
          }
        }
        if (CACHED) {
          double* Xs = region;
          const int kx0 = k + na;
          for (int q = threadIdx.x; q < nr * kx0; q += kOrthT) {
            const int r = q / kx0, t = q % kx0;
            Xs[(size_t)r * A.ldx + t] = t < k ? C[(size_t)(r0 + r) * kc + t]
                                              : Vr[(size_t)r * cap + t - k];
          }
        }
      }
    }
    sstamp(A, grp, cyc, 1);
    gbar(gb);
    sstamp(A, grp, cyc, 2);
    if (ldv(ist + kStatus) != PMP_SOLVE_OK) break;

    // ---- control block: projected problem of the cycle ---------------------------
    if (ctl) {
      const Ctl S = ctl_layout(ctl_mem, na, L.nblk, ldq, na);
      const StepBuf sbf = step_buf(L, 0);
      for (int q = threadIdx.x; q < ldq * na; q += kOrthT) {
        const int c = q / ldq, i = q % ldq;
        double v = 0.0;
        if (i < k)
          v = __ldcg(sbf.B + i * na + c);
        else if (i < k + na)
          v = __ldcg(sbf.R + (i - k) * na + c);
        S.Cq[q] = v;
      }
      // the fold images start from rhs0 = [rhs_c; S0; 0] (img = rhs0 - Q [0; t])
      for (int q = threadIdx.x; q < (k + cap) * na; q += kOrthT) {
        const int i = q / na, c = q % na;
        double v = 0.0;
        if (i < k)
          v = __ldcg(sbf.B + i * na + c);
        else if (i < k + na)
          v = __ldcg(sbf.R + (i - k) * na + c);
        img[(size_t)i * s + c] = v;
      }
      for (int c = threadIdx.x; c < na; c += kOrthT) S.bn[c] = bn[acts[c]];
      if (threadIdx.x == 0) {
        S.misc[0] = k > 0 ? 1.0 : 0.0;
        S.misc[1] = k > 0 ? 1.0 : INFINITY;
        S.misc[3] = 0.0;
      }
      for (int q = threadIdx.x; q < k * cap; q += kOrthT) proj[A.pBmat + q] = 0.0;
      for (int q = threadIdx.x; q < cap * cap; q += kOrthT) proj[A.pHb + q] = 0.0;
      for (int q = threadIdx.x; q < 128; q += kOrthT) ist[16 + q] = -1;
      __syncthreads();
    }
    gbar(gb);

    // ---- inner loop ---------------------------------------------------------------
    if (ctl) {
      const Ctl S = ctl_layout(ctl_mem, na, L.nblk, ldq, na);
      ctl_run<NY>(L, S);
      // the cycle's estimate rows -> the full-width log; fold images G Y
      const int hrow = ldv(ist + 5), m = ldv(ist + 0), total = ldv(ist + 1), st = ldv(ist + 4);
      {
        // the cycle's estimate rows -> full-width log rows (thread per column)
        const int lr0 = ldv(ist + kLogRows);
        const int nh = min(hrow, A.log_cap - lr0);
        for (int col = threadIdx.x; col < s; col += kOrthT) {
          int pos = -1;
          for (int c = 0; c < na; ++c)
            if (acts[c] == col) pos = c;
          double last = lrel[col];
          for (int h = 0; h < nh; ++h) {
            if (pos >= 0) last = proj[A.pHist + (size_t)h * na + pos];
            logp[(size_t)(lr0 + h) * s + col] = last;
          }
          lrel[col] = last;
        }
        __syncthreads();
        if (threadIdx.x == 0) ist[kLogRows] = lr0 + max(nh, 0);
      }
      if (st != 4 && st != 5 && m > 0) {
        // fold images G Y = rhs0 - (rhs0 - G Y), and the least-squares
        // residual rhs0 - G Y = Q [0; t] with t the tail of Q^T rhs0: apply
        // the steps' window transforms Q_p = M_p^T backwards (cheap, all in
        // shared memory) instead of multiplying G (global) by Y
        const int nrows = k + total, n1 = k + m, nq = m / na, b2 = 2 * na;
        double* z = S.cols;  // na x ldq, column-major
        for (int x = threadIdx.x; x < na * ldq; x += kOrthT) {
          const int i = x % ldq;
          z[x] = (i >= n1 && i < nrows) ? S.Cq[x] : 0.0;
        }
        __syncthreads();
        const int nout = na * b2;
        for (int pq = nq - 1; pq >= 0; --pq) {
          const double* M = S.Mq + (size_t)pq * b2 * b2;
          const int w0 = k + pq * na;
          double o[2] = {0.0, 0.0};
          for (int u = 0; u < 2; ++u) {
            const int x = threadIdx.x + u * kOrthT;
            if (x < nout) {
              const int c = x / b2, i = x % b2;
              const double* zc = z + (size_t)c * ldq + w0;
              double t = 0.0;
              for (int j = 0; j < b2; ++j) t += M[i * b2 + j] * zc[j];
              o[u] = t;
            }
          }
          __syncthreads();
          for (int u = 0; u < 2; ++u) {
            const int x = threadIdx.x + u * kOrthT;
            if (x < nout) z[(size_t)(x / b2) * ldq + w0 + x % b2] = o[u];
          }
          __syncthreads();
        }
        for (int x = threadIdx.x; x < nrows * na; x += kOrthT) {
          const int i = x / na, c = x % na;
          img[(size_t)i * s + c] -= z[(size_t)c * ldq + i];
        }
      }
      __syncthreads();
    } else {
      int m = 0, total = na, ncols = 0, status = 0;
      // W rows in shared memory, or (rows beyond shared memory) in global
      // (a compile-time choice: the shared-memory instances keep LDS / STS)
      const int ldw = WG ? s : odd_ld(na);
      double* Wv = WG ? W + (size_t)r0 * s : region + (CACHED ? (size_t)nr * A.ldx : 0);
      WSmem wsm{G, R1, R2, red, piv, piv2, flag, region, Wv, L.Q1g + (size_t)r0 * na, ldw};
      if constexpr (WG) {
        // (the control block's state lives in `region` of block 0 only: a
        // global-row worker's region is free between its passes)
        wsm.ring = A.ctl_global ? nullptr : region;
        wsm.ring_doubles = A.ctl_global ? 0 : A.region_doubles;
      }
      bool staged = false;
      if constexpr (WG) {
        if (A.stage_rows > 0) {
          // (the control block's state lives in `region` of block 0 only:
          // the workers' region is free for the staging ring)
          const Ring ring{region, A.stage_n, A.stage_rows, kc, cap, s};
          worker_inner_staged<NY>(L, wb, wsm, ring, r0, nr, lead, m, total, ncols, it, status);
          staged = true;
        }
      }
#ifndef PMP_WG_OPT
#define PMP_WG_OPT (kOptStamp | kOptCA | kOptFlat | kOptCyc | kOptFuse)
#endif
#ifndef PMP_SM_OPT
#define PMP_SM_OPT kOptFlat
#endif
      if (!staged)
        worker_inner<CACHED, NY, WG ? PMP_WG_OPT : PMP_SM_OPT>(L, wb, wsm, r0, nr, lead, m, total,
                                                               ncols, it, status);
      sstamp(A, grp, cyc, 3);
    }
    gbar(gb);
    sstamp(A, grp, cyc, 4);
    {
      const int st = ldv(ist + 4);
      if (st == 4 || st == 5) {
        if (lead && threadIdx.x == 0) { ist[kStatus] = PMP_SOLVE_FALLBACK; ist[kReason] = st == 4 ? 2 : 3; }
        break;
      }
    }
    const int m = ldv(ist + 0), total = ldv(ist + 1), it_new = ldv(ist + 3);
    if (m == 0) break;  // no step ran (iteration budget): nothing to fold in

    // ---- cycle end: dX, X, true residuals (workers) -----------------------------------
    if (!ctl) {
      const int n1 = k + m;
      // Y (rhs-major na x n1) -> smem G as row-major n1 x na
      const double* Yg = proj + A.pY;
      for (int q = threadIdx.x; q < n1 * na; q += kOrthT) {
        const int t = q / na, c = q % na;
        G[q] = __ldcg(Yg + (size_t)c * n1 + t);
      }
      __syncthreads();
      for (int r = threadIdx.x; r < nr; r += kOrthT) {
        const size_t row = (size_t)(r0 + r);
        // (V rows from the block's shared-memory copy when cached)
        const double* vr = CACHED ? region + (size_t)r * A.ldx + k : V + row * cap;
        double d[NY];
        row_combo<NY>(vr, m, k, U + row * kc, k, 0, G, na, d);
#pragma unroll
        for (int c = 0; c < NY; ++c)
          if (c < na) {
            DX[row * s + c] = d[c];
            const double xt = Xt[row * s + acts[c]] + d[c];
            Xt[row * s + acts[c]] = xt;
            Z[row * s + c] = xt;
          }
      }
      // Xa = P Z (factor chain right to left)
      const double* src = Z;
      constexpr int kOpt = WG ? PMP_WG_OPT : PMP_SM_OPT;
      // tiles dealt cyclically (spmm_rows_cyc); 8-column blocks only (s = 16: 1168 -> 1179 ms)
      constexpr bool kCyc = WG && NY <= 8 && (kOpt & kOptCyc) != 0;
      for (int f = D.nfac - 1; f >= 0; --f) {
        wbar(wb);
        double* dst = ((D.nfac - 1 - f) & 1) ? L.T1 : L.T0;
        if (kCyc)
          spmm_rows_cyc<NY, (kOpt & kOptCA) != 0>(D.frp[f], D.fci[f], D.fva[f], src, s, na, dst, s, n,
                                                  wb.wi, wb.n);
        else
          spmm_auto<NY, (kOpt & kOptCA) != 0>(D.frp[f], D.fci[f], D.fva[f], src, s, na,
                                              dst + (size_t)r0 * s, s, r0, nr,
                                              (WG && !A.ctl_global) ? region : nullptr,
                                              A.region_doubles);
        src = dst;
      }
      if (kCyc && D.nfac > 0) wbar(wb);  // this block's rows of P Z came from other blocks
      __syncthreads();
      for (int q = threadIdx.x; q < nr * na; q += kOrthT) {
        const int r = q / na, c = q % na;
        const size_t row = (size_t)(r0 + r);
        D.X[row * s + acts[c]] = src[row * s + c];
      }
      wbar(wb);
      // Rb = B[:, act] - A Xa -> R[:, act], RB
      if (kCyc) {
        spmm_rows_cyc<NY, (kOpt & kOptCA) != 0>(D.arp, D.aci, D.ava, src, s, na, RB, s, n, wb.wi,
                                                wb.n);
        wbar(wb);
      } else {
        spmm_auto<NY, (kOpt & kOptCA) != 0>(D.arp, D.aci, D.ava, src, s, na, RB + (size_t)r0 * s, s,
                                            r0, nr, (WG && !A.ctl_global) ? region : nullptr,
                                            A.region_doubles);
      }
      __syncthreads();
      for (int q = threadIdx.x; q < nr * na; q += kOrthT) {
        const int r = q / na, c = q % na;
        const size_t row = (size_t)(r0 + r);
        const double rb = D.B[row * s + acts[c]] - RB[row * s + c];
        RB[row * s + c] = rb;
        Rr[row * s + acts[c]] = rb;
      }
      __syncthreads();
      const double* RBr = RB + (size_t)r0 * s;
      const Rows RR{RBr, s, na, RBr, s};
      gram_b<NY, WG>(RR, na, RBr, s, na, nr, red, partial, slot);
      wreduce(wb, partial, gout, na * na, G, nullptr, 0, nullptr);
      if (lead && threadIdx.x == 0) {
        const int steps = it_new - it0;
        // algorithmic HBM bytes of the cycle's block steps (roofline):
        // every operator matrix once (12 B / nonzero + row pointers), the
        // gathered and written n x na blocks, [C | V] once per step
        double mb = 0.0;
        for (int f = 0; f < D.nfac; ++f)
          mb += 12.0 * __ldg(D.frp[f] + n) + 4.0 * (n + 1) + 16.0 * n * na;
        mb += 12.0 * __ldg(D.arp + n) + 4.0 * (n + 1) + 16.0 * n * na;
        // aux[48]: every operand once per step (the strict figure round 1
        // reported); aux[49]: SURVEY.md 8(d)'s unit for block CGS2 -- two
        // Gram products and two updates per step read [C | V] -- 32 n total +
        // 48 n s_b + 16 n k on top of the operator chain
        double by = 0.0, by2 = 0.0;
        for (int j = 0; j < steps; ++j) {
          const double tot = (double)na * (j + 1);
          by += mb + 8.0 * n * (k + tot) + 32.0 * n * na;
          by2 += mb + 32.0 * n * tot + 48.0 * n * na + 16.0 * n * k;
        }
        aux[48] += by;
        aux[49] += by2;
        ist[kIt] = it_new;
        ist[kMatvecs] += na * steps + na;
        if (D.nfac) ist[kPrec] += na * steps + na;
        int lr = ist[kLogRows];
        int still = 0;
        for (int c = 0; c < na; ++c) {
          const double tn = sqrt(fmax(G[c * na + c], 0.0));
          const int col = acts[c];
          pn[col] = tn;
          const double rel = bn[col] > 0.0 ? tn / bn[col] : 0.0;
          lrel[col] = rel;
          if (rel > A.tol) act[still++] = col;
        }
        if (lr < A.log_cap) {
          for (int c = 0; c < s; ++c) logp[(size_t)lr * s + c] = lrel[c];
          ++lr;
        }
        ist[kLogRows] = lr;
        ist[kNa] = still;
        // fold only when another cycle can run (krylov.py:244)
        ist[kFold] = (still > 0 && it_new < A.max_iters) ? 1 : 0;
      }
    }
    sstamp(A, grp, cyc, 5);
    gbar(gb);
    sstamp(A, grp, cyc, 6);
    if (!ldv(ist + kFold)) {
      ++cyc;
      continue;
    }

    // ---- fold (workers): images -> block CGS2 against C -> new C / U columns ---------
    if (!ctl) {
      // RB = V[:, :total] img_v + C[:, :k] img_c  (own rows)
      for (int q = threadIdx.x; q < (k + total) * na; q += kOrthT) G[q] = __ldcg(img + (size_t)(q / na) * s + q % na);
      __syncthreads();
      for (int r = threadIdx.x; r < nr; r += kOrthT) {
        const size_t row = (size_t)(r0 + r);
        const double* vr = CACHED ? region + (size_t)r * A.ldx + k : V + row * cap;
        const double* cr = CACHED ? region + (size_t)r * A.ldx : C + row * kc;
        double d[NY];
        row_combo<NY>(vr, total, k, cr, k, 0, G, na, d);
#pragma unroll
        for (int c = 0; c < NY; ++c)
          if (c < na) RB[row * s + c] = d[c];
      }
      __syncthreads();
      double* Wr = RB + (size_t)r0 * s;
      double* Zr = DX + (size_t)r0 * s;
      const Rows Cr{C + (size_t)r0 * kc, kc, k, Wr, s};
      const Rows Conly{C + (size_t)r0 * kc, kc, k, C + (size_t)r0 * kc, kc};
      const Rows Uonly{U + (size_t)r0 * kc, kc, k, U + (size_t)r0 * kc, kc};
      // pass 1: [C | W]^T W -> H1, M0 = W^T W
      gram_b<NY, WG>(Cr, k + na, Wr, s, na, nr, red, partial, slot);
      wreduce(wb, partial, gout, (k + na) * na, G, nullptr, 0, nullptr);
      double* w0 = R1;  // |w_c| (before any projection)
      for (int c = threadIdx.x; c < na; c += kOrthT) w0[c] = sqrt(fmax(G[(k + c) * na + c], 0.0));
      double* Mf = R2;  // na x na: W2^T W2 (built below)
      if (k > 0) {
        block_update<NY>(Conly, k, Wr, s, na, nr, G);
        block_update<NY>(Uonly, k, Zr, s, na, nr, G);
        // pass 2: [C | W1]^T W1 -> H2, M1; M = M1 - H2^T H2
        gram_b<NY, WG>(Cr, k + na, Wr, s, na, nr, red, partial, slot);
        wreduce(wb, partial, gout, (k + na) * na, G, nullptr, 0, nullptr);
        for (int q = threadIdx.x; q < na * na; q += kOrthT) {
          const int i = q / na, j = q % na;
          double h = 0.0;
          for (int t = 0; t < k; ++t) h += G[t * na + i] * G[t * na + j];
          Mf[q] = G[(k + i) * na + j] - h;
        }
        __syncthreads();
        block_update<NY>(Conly, k, Wr, s, na, nr, G);
        block_update<NY>(Uonly, k, Zr, s, na, nr, G);
      } else {
        for (int q = threadIdx.x; q < na * na; q += kOrthT) Mf[q] = G[q];
        __syncthreads();
      }
      // sequential drop test + Cholesky of the kept columns (thread 0; tiny)
      __shared__ int s_keep[16];
      __shared__ int s_nk, s_amb;
      double* T = G;  // nk x nk upper (row-major), reuse of the reduction buffer
      if (threadIdx.x == 0) {
        int nk = 0, amb = 0;
        for (int j = 0; j < na; ++j) {
          if (w0[j] == 0.0) continue;
          // d = M_jj - sum over kept i of T_ij^2, with T_ij for the kept i
          double tcol[16];
          double d = Mf[j * na + j];
          for (int a = 0; a < nk; ++a) {
            const int i = s_keep[a];
            double v = Mf[i * na + j];
            for (int b = 0; b < a; ++b) v -= T[b * 16 + a] * tcol[b];
            v /= T[a * 16 + a];
            tcol[a] = v;
            d -= v * v;
          }
          const double mjj = Mf[j * na + j];
          if (!(d > 1e-4 * mjj)) {
            // cancellation: the reference's exact recomputation decides
            amb = 1;
            break;
          }
          const double nwj = sqrt(d);
          if (!(nwj > 1e-10 * w0[j])) continue;
          for (int a = 0; a < nk; ++a) T[a * 16 + nk] = tcol[a];
          T[nk * 16 + nk] = nwj;
          s_keep[nk++] = j;
        }
        s_nk = nk;
        s_amb = amb;
      }
      __syncthreads();
      int nk = s_nk;
      if (s_amb) {
#if PMP_FOLD_EXACT
        wb.epoch = fold_exact<NY>(wb.ctr, wb.n, wb.epoch, wb.wi, C + (size_t)r0 * kc,
                                  U + (size_t)r0 * kc, kc, k, Wr, Zr, s, w0, na, nr, red,
                                  partial, gout, G, slot, &s_nk);
        nk = s_nk;
        if (threadIdx.x == 0) s_amb = 0;
        __syncthreads();
#else
        if (lead && threadIdx.x == 0) { ist[kStatus] = PMP_SOLVE_FALLBACK; ist[kReason] = 4; }
#endif
      } else if (nk > 0) {
        // Q = W2[:, keep] T^-1 and the directions alike (own rows), in place
        // into the next C / U columns
        double tmin = INFINITY, tmax = 0.0;
        for (int a = 0; a < nk; ++a) {
          tmin = fmin(tmin, T[a * 16 + a]);
          tmax = fmax(tmax, T[a * 16 + a]);
        }
        for (int r = threadIdx.x; r < nr; r += kOrthT) {
          const size_t row = (size_t)(r0 + r);
          fold_rowsolve<NY>(RB + row * s, DX + row * s, s_keep, nk, T, 16,
                            C + row * kc + k, U + row * kc + k);
        }
        __syncthreads();
        if (!(tmax <= kSkipKappa * tmin)) {
          // second Cholesky-QR pass over the new columns
          const Rows Qn{C + (size_t)r0 * kc + k, kc, nk, C + (size_t)r0 * kc + k, kc};
          gram_b<NY, WG>(Qn, nk, C + (size_t)r0 * kc + k, kc, nk, nr, red, partial, slot);
          wreduce(wb, partial, gout, nk * nk, G, nullptr, 0, nullptr);
          if (threadIdx.x < 32) {
            const bool ok = warp_cholesky_smem(G, nk, R1, piv2, false, 0.0);
            if (threadIdx.x == 0) flag[0] = ok ? 0 : 1;
          }
          __syncthreads();
          if (flag[0]) {
            if (lead && threadIdx.x == 0) { ist[kStatus] = PMP_SOLVE_FALLBACK; ist[kReason] = 5; }
          } else {
            for (int r = threadIdx.x; r < nr; r += kOrthT) {
              const size_t row = (size_t)(r0 + r);
              fold_rowsolve<NY>(C + row * kc + k, U + row * kc + k, nullptr, nk, R1, nk,
                                C + row * kc + k, U + row * kc + k);
            }
          }
        }
      }
      // truncation: keep the last outer_dim columns (krylov.py:267-269)
      const int kk = k + nk;
      if (!s_amb && kk > A.outer_dim) {
        const int drop = kk - A.outer_dim;
        for (int r = threadIdx.x; r < nr; r += kOrthT) {
          const size_t row = (size_t)(r0 + r);
          for (int t = 0; t < A.outer_dim; ++t) {
            C[row * kc + t] = C[row * kc + t + drop];
            U[row * kc + t] = U[row * kc + t + drop];
          }
        }
      }
      if (lead && threadIdx.x == 0 && !s_amb) ist[kK] = kk > A.outer_dim ? A.outer_dim : kk;
    }
    sstamp(A, grp, cyc, 7);
    gbar(gb);
    sstamp(A, grp, cyc, 8);
    ++cyc;
  }

  // ---- system done: its record, then the next system from the queue ------------
  gbar(gb);
  if (lead) {
    int* rec = A.rint + (size_t)sys * PMP_SOLVE_RSZ;
    double* rd = A.rdbl + (size_t)sys * (2 + (size_t)A.log_cap * s);
    const int lr = ldv(ist + kLogRows);
    if (threadIdx.x == 0) {
      rec[rStatus] = ldv(ist + kStatus);
      rec[rReason] = ldv(ist + kReason);
      rec[rIt] = ldv(ist + kIt);
      rec[rNa] = ldv(ist + kNa);
      rec[rLogRows] = lr;
      rec[rMatvecs] = ldv(ist + kMatvecs);
      rec[rPrec] = ldv(ist + kPrec);
      rd[0] = __ldcg(aux + 48);
      rd[1] = __ldcg(aux + 49);
    }
    for (int q = threadIdx.x; q < lr * s; q += kOrthT) rd[2 + q] = __ldcg(logp + q);
  }
  if (ctl && threadIdx.x == 0) ist[kNext] = A.groups + atomicAdd(A.queue, 1);
  gbar(gb);
  sys = ldv(ist + kNext);
  }
}

}  // namespace pmp

// cycle.cu
namespace pmp {
size_t cycle_region_doubles(int rows, int ldx, int sb, int ldq, int na, int restart, int cached);
size_t cycle_ctl_doubles(int sb, int ldq, int na, int restart);
size_t cycle_work_doubles(int rows, int ldx, int sb, int cached);
}

using namespace pmp;

// the staged ring runs from PMP_STAGE_MIN_S block columns up (measured,
// profiles/r02_stage_ab_c3_c4.txt: it wins at s = 16 -- c3 block step 13.1 ->
// 8.4 ms -- and loses at s = 8 -- c4 12.5 -> 13.9 ms, 16-24-row tiles)
#ifndef PMP_STAGE
#define PMP_STAGE 1
#endif
static bool solve_staged(int s, int kc, int cap, int cached) {
  static const int stage_min_s = [] {
    const char* e = getenv("PMP_STAGE_MIN_S");
    return e ? atoi(e) : 9;
  }();
  return PMP_STAGE && cached == 2 && s >= stage_min_s && (s % 2) == 0 && (kc % 2) == 0 &&
         (cap % 2) == 0;
}
// global-row geometry without the ring: the control state lives in global
// memory and the blocks carry no region (PMP_CTL_GLOBAL=0 keeps it in smem)
static bool solve_ctl_global(int s, int kc, int cap, int cached) {
  static const int on = [] {
    const char* e = getenv("PMP_CTL_GLOBAL");
    return e ? atoi(e) : 1;
  }();
  if (on >= 2 && cached == 0) return true;  // (experiment: W rows only in the region)
  // staged geometry (s >= 9: c3): with the control state in global memory the
  // blocks need only the ring, and two of them fit an SM instead of one
  // (PMP_STAGE_CTLG; measured in profiles/r02_codegen_ab.txt)
  static const int stg = [] {
    const char* e = getenv("PMP_STAGE_CTLG");
    return e ? atoi(e) : 1;
  }();
  if (cached == 2 && solve_staged(s, kc, cap, cached)) return on && stg != 0;
  return on && cached == 2;
}

// doubles of a block's shared-memory region: the control state and / or the
// workers' rows (cycle_region_doubles), only the workers' rows when the
// control state is in global memory, or -- staged geometry with the control
// state in global memory -- a ring that fills a two-blocks-per-SM budget
static size_t solve_region_doubles(int rows, int ldx, int kc, int cap, int s, int restart,
                                   int cached) {
  if (!solve_ctl_global(s, kc, cap, cached))
    return cycle_region_doubles(rows, ldx, s, kc + cap, s, restart, cached);
  if (solve_staged(s, kc, cap, cached)) {
    const size_t fixed = (size_t)(kc + cap + s) * s + 2 * (size_t)s * s + 8 * 32 * (size_t)s + 20;
    const size_t budget = (size_t)108 * 1024 / sizeof(double);
    return budget > fixed + 2048 ? ((budget - fixed) & ~(size_t)1) : 2048;
  }
  return cycle_work_doubles(rows, ldx, s, cached);
}

static size_t solve_smem_bytes(int rows, int ldx, int kc, int cap, int s, int restart,
                               int cached) {
  size_t d = (size_t)(kc + cap + s) * s + 2 * (size_t)s * s + 8 * 32 * (size_t)s + 20;
  d += solve_region_doubles(rows, ldx, kc, cap, s, restart, cached);
  return d * sizeof(double);
}

static void* solve_kernel(int s, int cached) {
  if (s <= 8)
    return cached == 1 ? (void*)k_solve<true, 8, false>
                       : (cached == 2 ? (void*)k_solve<false, 8, true> : (void*)k_solve<false, 8, false>);
  return cached == 1 ? (void*)k_solve<true, 16, false>
                     : (cached == 2 ? (void*)k_solve<false, 16, true> : (void*)k_solve<false, 16, false>);
}

extern "C" {

int pmp_solve_geometry(int n, int s, int cap, int kc, int restart, int groups, int* gsz,
                       int* rows, int* cached, size_t* smem) {
  const int sms = orth_max_grid() / 2;
  const int ldx = odd_ld(kc + cap);
  if (groups < 1 || s < 1 || s > 16) return PMP_ERR_ARG;
  // cached 1: [C | V] and W rows in shared memory; 0: W rows only; 2: none
  const int order[6][2] = {{2, 1}, {1, 1}, {2, 0}, {1, 0}, {2, 2}, {1, 2}};
  for (int a = 0; a < 6; ++a) {
    const int bps = order[a][0], cach = order[a][1];
    const int g = bps * sms / groups;
    if (g < 2) continue;
    int workers = g - 1;
    const int need = (n + 31) / 32;
    if (need < workers) workers = need;
    const int r = (n + workers - 1) / workers;
    const size_t sm = solve_smem_bytes(r, ldx, kc, cap, s, restart, cach);
    if (sm > (size_t)(bps == 2 ? 110 : 220) * 1024) continue;
    // registers may cap residency below what shared memory allows
    if (prepare_smem(solve_kernel(s, cach), sm, kOrthT) < bps) continue;
    *gsz = workers + 1;
    *rows = r;
    *cached = cach;
    *smem = sm;
    return PMP_OK;
  }
  return PMP_ERR_ARG;
}

size_t pmp_solve_ctl_doubles(int s, int kc, int cap, int restart) {
  return cycle_ctl_doubles(s, kc + cap, s, restart);
}

int pmp_solve_batch(PmpSolveBatch* b) {
  if (!b || b->groups < 1 || b->nsys < 1 || !b->d_queue || !b->d_result || !b->d_result_log ||
      b->s < 1 || b->s > 16 || 
      b->inner_restart + b->s > 96 || b->outer_dim < 0 || b->outer_dim + b->s > b->kc) {
    set_error("pmp_solve_batch: bad arguments");
    return PMP_ERR_ARG;
  }
  int gsz, rows, cached;
  size_t smem;
  if (pmp_solve_geometry(b->n, b->s, b->cap, b->kc, b->inner_restart, b->groups, &gsz, &rows,
                         &cached, &smem) != PMP_OK) {
    set_error("pmp_solve_batch: no co-resident geometry (n=%d s=%d groups=%d)", b->n, b->s,
              b->groups);
    return PMP_ERR_ARG;
  }
  if (gsz != b->gsz || rows != b->rows_per_block) {
    set_error("pmp_solve_batch: geometry mismatch (query pmp_solve_geometry first)");
    return PMP_ERR_ARG;
  }
  void* fn = solve_kernel(b->s, cached);
  const int occ = prepare_smem(fn, smem, kOrthT);
  if (occ * (orth_max_grid() / 2) < gsz * (b->groups < b->nsys ? b->groups : b->nsys)) {
    set_error("pmp_solve_batch: grid not co-resident (%d blocks/SM)", occ);
    return PMP_ERR_ARG;
  }
  SolveArgs A;
  A.n = b->n;
  A.s = b->s;
  A.cap = b->cap;
  A.kc = b->kc;
  A.outer_dim = b->outer_dim;
  A.inner_restart = b->inner_restart;
  A.max_iters = b->max_iters;
  A.gsz = gsz;
  A.rows_per_block = rows;
  A.ldx = odd_ld(b->kc + b->cap);
  A.hist_cap = b->hist_cap;
  A.log_cap = b->log_cap;
  A.isz = b->isz;
  A.tol = b->tol;
  A.wglob = cached == 2;
  A.stage_rows = 0;
  A.stage_n = 0;
  A.region_doubles = (int)solve_region_doubles(rows, A.ldx, b->kc, b->cap, b->s,
                                               b->inner_restart, cached);
  A.ctl_global = solve_ctl_global(b->s, b->kc, b->cap, cached) ? 1 : 0;
  A.pCtl = b->pCtl;
  if (A.ctl_global && b->pCtl <= 0) {
    set_error("pmp_solve_batch: pCtl not set (pmp_solve_ctl_doubles sizes it)");
    return PMP_ERR_ARG;
  }
  if (solve_staged(b->s, b->kc, b->cap, cached)) {
    // ring of S stages x R rows of [C | V | W] in the workers' region
    const size_t region = (size_t)A.region_doubles;
    // (stage_rows carries the stage size in doubles: a pass packs as many
    // rows as its columns allow, >= 8 even at full width)
    const size_t row = (size_t)bank_pad(b->kc) + bank_pad(b->cap) + bank_pad(b->s);
    for (int S = 4; S >= 2 && A.stage_rows == 0; --S) {
      const size_t stage = (region / S) & ~(size_t)1;
      if (stage >= 8 * row) {
        A.stage_rows = (int)stage;
        A.stage_n = S;
      }
    }
  }
  A.sys = reinterpret_cast<const SysDesc*>(b->d_sys);
  A.ws = b->d_ws;
  A.wsz = b->wsz;
  A.ist = b->d_istate;
  A.oV = b->oV;
  A.oC = b->oC;
  A.oU = b->oU;
  A.oW = b->oW;
  A.oT0 = b->oT0;
  A.oT1 = b->oT1;
  A.oQ1 = b->oQ1;
  A.oXt = b->oXt;
  A.oR = b->oR;
  A.oDX = b->oDX;
  A.oRB = b->oRB;
  A.oZ = b->oZ;
  A.oPart = b->oPart;
  A.oGout = b->oGout;
  A.oSbuf = b->oSbuf;
  A.oProj = b->oProj;
  A.oLog = b->oLog;
  A.oAux = b->oAux;
  A.pBmat = b->pBmat;
  A.pHb = b->pHb;
  A.pCq = b->pCq;
  A.pY = b->pY;
  A.pRes = b->pRes;
  A.pBn = b->pBn;
  A.pHist = b->pHist;
  A.dbg = cycle_dbg_take();
  A.nsys = b->nsys;
  A.groups = b->groups < b->nsys ? b->groups : b->nsys;
  A.queue = b->d_queue;
  A.rint = b->d_result;
  A.rdbl = b->d_result_log;
  if (cudaMemsetAsync(A.queue, 0, sizeof(int), reinterpret_cast<cudaStream_t>(b->stream)) !=
      cudaSuccess)
    return cuda_status("pmp_solve_batch");
  void* args[] = {&A};
  cudaError_t e = coop_launch(fn, gsz * A.groups, args, smem,
                              reinterpret_cast<cudaStream_t>(b->stream));
  if (e != cudaSuccess) {
    set_error("pmp_solve_batch: %s", cudaGetErrorString(e));
    return PMP_ERR_CUDA;
  }
  return cuda_status("pmp_solve_batch");
}

}  // extern "C"
