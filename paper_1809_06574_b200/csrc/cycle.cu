// Device-resident inner loop of one block-GCRO cycle (krylov.py:184-216).
//
// pmp_gcro_inner drives a cycle from the host: per block step it launches
// the operator chain and the fused orthogonalisation, waits for the small
// results in mapped memory and folds them into the projected least-squares
// problem.  At BASELINE sizes (c2: n = 32768, s = 8) the device work of a
// step is tens of microseconds while launch gaps + the host round trip add
// ~100 us, so the step is latency bound on the HOST.  k_cycle removes the
// host from the loop: one persistent cooperative launch runs every step of
// the cycle.
//
//   per step j (nfac preconditioner factors):
//     T0 = F_{nfac-1} V[:, q0:q0+sb]        control block meanwhile absorbs
//     grid barrier                            step j-1 and publishes the stop
//                                             decision read after the barrier
//     T1 = F_{nfac-2} T0 ... (barrier each)
//     W  = A T_last                           own rows -> shared memory
//     R1: [C | V]^T W  (reduce, 2 barriers)  W1 = W - C B - V H1
//     R2: [V | W1]^T W1 (reduce, 2 barriers) W2 = W1 - V H2
//     pivoted Cholesky of W2^T W2 (every block, redundantly)
//     [R3: Cholesky-QR2 second pass when kappa > 4 (2 barriers)]
//     Q = W2 P R^-1 -> V[:, total:total+sb]
//     grid barrier (new V block visible)
//
// Projected problem (control block 0, owns no rows).  G = [[I, Bmat], [0,
// Hb]] is block upper Hessenberg, so the Householder QR the host path
// computes column by column (hostls.cpp pmp_host_hls_append) is, for step
// q, b = sb reflectors acting only on the 2b-row window k + [q b, (q+2) b).
// The kernel keeps each step's window transform explicitly, M_q = Q_q^T
// (2b x 2b), so bringing a new block column up to date is q small dense
// mat-vecs (parallel over the block's columns) instead of q b sequential
// reflector applications; the window itself is factored with one thread
// per column (the block's b columns, the 2b identity columns that become
// M_q, and the na right-hand sides), registers only.  The arithmetic of the
// window factorisation is the host's (larfg / dot / update order); the
// packed R (block columns of height (q+1) b) stays in shared memory for the
// final back substitution.  On a host fallback (status 4 / 5) the host
// re-factors G from Bmat / Hb (the same minimiser).
#include "cycle_dev.cuh"

namespace pmp {

template <bool CACHED, int NY, bool WG>
__global__ void __launch_bounds__(kOrthT, 2) k_cycle(CycleArgs P) {
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

  cstamp(P, 63, 31);
  if (ctl) {
    const Ctl S = ctl_layout(region, sb, P.nblk, ldq, P.na);
    for (int q = threadIdx.x; q < ldq * P.na; q += kOrthT) S.Cq[q] = P.proj[P.oCq + q];
    for (int q = threadIdx.x; q < P.na; q += kOrthT) S.bn[q] = P.proj[P.oBn + q];
    if (threadIdx.x == 0) {
      S.misc[0] = k > 0 ? 1.0 : 0.0;  // the identity columns' R_jj
      S.misc[1] = k > 0 ? 1.0 : INFINITY;
      S.misc[3] = 0.0;
    }
    for (int q = threadIdx.x; q < k * cap; q += kOrthT) P.proj[P.oBmat + q] = 0.0;
    for (int q = threadIdx.x; q < cap * cap; q += kOrthT) P.proj[P.oHb + q] = 0.0;
    __syncthreads();
    ctl_run<NY>(P, S);
    return;
  }

  // ---- workers -----------------------------------------------------------------
  const int ldx = P.ldx;
  // W rows in shared memory, or (rows beyond shared memory) in global
  const int ldw = WG ? P.s : odd_ld(sb);
  double* Xs = region;
  double* Wv = WG ? P.W + (size_t)r0 * P.s : region + (CACHED ? (size_t)nr * ldx : 0);
  double* Q1 = P.Q1g + (size_t)r0 * sb;
  WBar wb{P.ist + 9, (int)gridDim.x - 1, 0, (int)blockIdx.x - 1};

  int m = P.ist[0], total = P.ist[1], ncols = P.ist[2], it = P.ist[3];
  if (CACHED) {
    const int kx0 = k + total;
    for (int q = threadIdx.x; q < nr * kx0; q += kOrthT) {
      const int r = q / kx0, t = q % kx0;
      Xs[(size_t)r * ldx + t] = t < k ? P.C[(size_t)(r0 + r) * kc + t]
                                      : P.V[(size_t)(r0 + r) * cap + t - k];
    }
  }
  __syncthreads();
  cstamp(P, 63, 30);

  int status = 0;
  WSmem wsm{G, R1, R2, red, piv, piv2, flag, Xs, Wv, Q1, ldw};
  worker_inner<CACHED, NY>(P, wb, wsm, r0, nr, blockIdx.x == 1, m, total, ncols, it, status);
}

int cycle_nblk(int restart, int sb) { return (restart + sb - 1) / sb + 1; }

// doubles of the control block's projected-problem state (ctl_layout)
size_t cycle_ctl_doubles(int sb, int ldq, int na, int restart) {
  const size_t nb = cycle_nblk(restart, sb);
  return nb * 4 * sb * sb + (size_t)sb * sb * nb * (nb + 1) / 2 + (size_t)ldq * na +
         (size_t)sb * ldq + sb * sb + 16 * 96 + 32 + 8 + 16 + 16 +
         (size_t)(2 * sb + 1) * (3 * sb + na) + (size_t)2 * ldq * sb + 8;
}

// doubles of a worker's rows kept in shared memory (cached: 1 = [C | V] and W
// rows, 0 = W rows only, 2 = none)
size_t cycle_work_doubles(int rows, int ldx, int sb, int cached) {
  return (size_t)rows * ((cached == 1 ? ldx : 0) + (cached == 2 ? 0 : odd_ld(sb)));
}

size_t cycle_region_doubles(int rows, int ldx, int sb, int ldq, int na, int restart, int cached) {
  size_t ctl = cycle_ctl_doubles(sb, ldq, na, restart);
  // cached: 1 = [C | V] rows (and W rows) in shared memory, 0 = W rows
  // only, 2 = none (W rows in global memory: large n per block)
  size_t work = (size_t)rows * ((cached == 1 ? ldx : 0) + (cached == 2 ? 0 : odd_ld(sb)));
  return ctl > work ? ctl : work;
}

size_t cycle_smem_bytes(int rows, int ldx, int k, int cap, int sb, int ldq, int na, int restart,
                        int cached) {
  size_t d = (size_t)(k + cap + sb) * sb + 2 * sb * sb + 8 * 32 * sb + 20;
  d += cycle_region_doubles(rows, ldx, sb, ldq, na, restart, cached);
  return d * sizeof(double);
}

}  // namespace pmp

using namespace pmp;

static unsigned long long* g_cdbg = nullptr;
static int g_cdbg_left = 0;

// next diagnostics record (4096 stamps) or nullptr (solve.cu uses it too)
unsigned long long* pmp::cycle_dbg_take() {
  if (!g_cdbg || g_cdbg_left <= 0) return nullptr;
  unsigned long long* p = g_cdbg;
  g_cdbg += 4096;
  --g_cdbg_left;
  return p;
}

extern "C" {

// Diagnostics: the next `records` cycle kernels write %globaltimer stamps
// (blocks 0 and 1) into d_stamps[4096 * launch + (32 * step + phase) * 2 + block].
int pmp_cycle_debug_stamps(unsigned long long* d_stamps, int records) {
  g_cdbg = d_stamps;
  g_cdbg_left = d_stamps ? records : 0;
  return PMP_OK;
}

size_t pmp_cycle_workspace(int n, int cap, int kc, int s) {
  const int g = orth_max_grid();
  const size_t kmax = (size_t)(kc + cap + s) * s;
  return 256 + sizeof(double) * ((size_t)g * kmax + kmax + (size_t)n * s +
                                 2 * (size_t)(kc + 2 * cap + s) * s + 64);
}

int pmp_gcro_cycle_dev(PmpGcroCycle* c) {
  if (!c || c->n < 1 || c->sb < 1 || c->sb > 16 || c->na < 1 || c->na > 16 || c->nfac < 0 ||
      c->nfac > 3 || c->s < c->sb || c->k < 0 || c->k > c->kc || c->ldq < c->k + c->cap ||
      c->inner_restart < 1 || c->inner_restart + c->sb > 96) {
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
    if (NYsel == 8)
      return cached == 1 ? (void*)k_cycle<true, 8, false>
                         : (cached == 2 ? (void*)k_cycle<false, 8, true> : (void*)k_cycle<false, 8, false>);
    return cached == 1 ? (void*)k_cycle<true, 16, false>
                       : (cached == 2 ? (void*)k_cycle<false, 16, true> : (void*)k_cycle<false, 16, false>);
  };
  // geometry: 1 control block + workers; prefer the cached layout with two
  // blocks per SM, then one, then streaming rows from global memory
  // (blocks_per_sm = 1 puts the one-per-SM layouts first)
  int g = 0, rows = 0;
  size_t smem = 0;
  void* fn = nullptr;
  const int order2[6][2] = {{2, 1}, {1, 1}, {2, 0}, {1, 0}, {2, 2}, {1, 2}};
  const int order1[6][2] = {{1, 1}, {2, 1}, {1, 0}, {2, 0}, {1, 2}, {2, 2}};
  const int(*order)[2] = c->blocks_per_sm == 1 ? order1 : order2;
  int wglob = 0;
  for (int attempt = 0; attempt < 6 && !fn; ++attempt) {
    const int bps = order[attempt][0], cach = order[attempt][1];
    const int gb = bps * sms;
    int workers = gb - 1;
    const int need = (c->n + 31) / 32;
    if (need < workers) workers = need;
    const int r = (c->n + workers - 1) / workers;
    const size_t sm = cycle_smem_bytes(r, ldx, c->kc, c->cap, c->sb, c->ldq, c->na,
                                       c->inner_restart, cach);
    if (sm > (size_t)(bps == 2 ? 110 : 220) * 1024) continue;
    void* f = pick(cach);
    const int occ = prepare_smem(f, sm, kOrthT);
    if (occ * sms < workers + 1) continue;
    fn = f;
    g = workers + 1;
    rows = r;
    smem = sm;
    wglob = cach == 2;
  }
  if (!fn) {
    set_error("pmp_gcro_cycle_dev: no co-resident geometry (n=%d ldq=%d)", c->n, c->ldq);
    return PMP_ERR_ARG;
  }
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
  P.wglob = wglob;
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
  P.sbuf = P.Q1g + (size_t)c->n * c->s;
  P.rows_per_block = rows;
  P.ldx = ldx;
  P.max_iters = c->max_iters;
  P.inner_restart = c->inner_restart;
  P.hist_cap = c->hist_cap;
  P.nblk = cycle_nblk(c->inner_restart, c->sb);
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
  P.dbg = cycle_dbg_take();
  void* args[] = {&P};
  cudaError_t e = coop_launch(fn, g, args, smem, reinterpret_cast<cudaStream_t>(c->stream));
  if (e != cudaSuccess) {
    set_error("pmp_gcro_cycle_dev: %s", cudaGetErrorString(e));
    return PMP_ERR_CUDA;
  }
  return cuda_status("pmp_gcro_cycle_dev");
}

}  // extern "C"
