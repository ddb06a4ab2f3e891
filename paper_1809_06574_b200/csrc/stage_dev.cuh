// Block step of the persistent solve for the GLOBAL-ROW geometry (large n:
// c3 / c4 / c5 -- W rows in HBM), with the tall-skinny products fed by
// bulk asynchronous copies (cp.async.bulk, the TMA engine's 1-D form) into a
// shared-memory ring, and computed by FP64 tensor-core fragments (DMMA
// m8n8k4) from shared memory.
//
// Why: at these sizes every phase of the block step streams the block's rows
// of [C | V] and W from HBM.  The thread-per-row / lane-per-column loops keep
// only a few loads in flight per warp at 16 warps per SM (the kernel's
// register and shared-memory footprint), so the Gram / update phases ran at
// 2-3 TB/s (ncu: 0.29 eligible warps per scheduler, L1 hit 55 %, 35 %
// excess sectors).  Here one thread posts the copies of tile i + S - 1 while
// the block computes tile i: S x R rows (tens of KB) in flight per block, no
// register cost, whole 16-byte-aligned rows.
//
// The CGS2 step (krylov.py:186-196) becomes three streaming passes over the
// block's rows instead of four:
//   pass 1   [C | V]^T W                                 -> reduce -> B, H1
//   pass 2   W1 = W - [C | V] [B; H1], then [V | W1]^T W1  -> reduce -> H2, W1^T W1
//            (the Pythagorean G_W = W1^T W1 - H2^T H2 is factored before pass 3)
//   pass 3   W2 = W1 - V H2 and, when the Cholesky-QR needs one pass
//            (kappa <= 4), the new block Q = W2 P R^-1 straight into V
// Same operations as the scalar path (cycle_dev.cuh worker_inner), different
// (fixed) summation order.
#pragma once

#include "cycle_dev.cuh"

namespace pmp {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra "
      "WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// generic-proxy writes (this block's stores of W / V / C rows) before
// async-proxy reads of the same global memory (the bulk copies)
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// One ring of S stages of `stage` doubles each in the workers' shared
// memory.  A pass lays its tile out per stage as [C rows | V rows | W rows]
// with padded strides (8 m + 4 doubles: the 4 rows of a DMMA half-warp
// fragment land 8 banks apart) and as many rows as fit the columns it
// actually needs (more rows per tile early in a cycle, when V is narrow).
struct Ring {
  double* base;
  int S, stage;       // stages, doubles per stage
  int kc, cap, s;     // global leading dimensions of C, V, W rows
};

__host__ __device__ __forceinline__ int bank_pad(int w) { return ((w + 3) & ~7) + 4; }

struct Tile {
  int R;               // rows per tile
  int cst, vst, wst;   // strides of the C / V / W parts (0: part absent)
  int ccols, vcols, wcols;  // columns copied (even)
  __device__ __forceinline__ double* Cs(const Ring& g, int st) const {
    return g.base + (size_t)st * g.stage;
  }
  __device__ __forceinline__ double* Vs(const Ring& g, int st) const {
    return Cs(g, st) + (size_t)R * cst;
  }
  __device__ __forceinline__ double* Ws(const Ring& g, int st) const {
    return Vs(g, st) + (size_t)R * vst;
  }
};

__device__ __forceinline__ Tile make_tile(const Ring& g, bool c, int vcols, bool w) {
  Tile t;
  t.ccols = c ? g.kc : 0;
  t.vcols = (vcols + 1) & ~1;
  t.wcols = w ? g.s : 0;
  t.cst = c ? bank_pad(g.kc) : 0;
  t.vst = bank_pad(t.vcols);
  t.wst = w ? bank_pad(g.s) : 0;
  int R = (g.stage / (t.cst + t.vst + t.wst)) & ~7;
  t.R = R > 64 ? 64 : R;
  return t;
}

// which global rows a pass stages
struct StageSpec {
  const double* C;  // this block's C rows (ld kc), or null
  const double* V;  // this block's V rows (ld cap)
  const double* W;  // this block's W rows (ld s), or null
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait(int pending) {
  switch (pending) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
  }
}

// every thread: its share of the 16-byte copies of tile `tile` into stage st
__device__ __forceinline__ void ring_issue(const Ring& g, const Tile& T, const StageSpec& sp,
                                           int tile, int nr, int st) {
  const int ra = tile * T.R, nt = min(T.R, nr - ra);
  const int cc = T.ccols >> 1, vc = T.vcols >> 1, wc = T.wcols >> 1;
  const int nc = nt * cc, nv = nt * vc, nw = nt * wc;
  double* Cd = T.Cs(g, st);
  double* Vd = T.Vs(g, st);
  double* Wd = T.Ws(g, st);
  for (int q = threadIdx.x; q < nc + nv + nw; q += kOrthT) {
    if (q < nc) {
      const int r = q / cc, c = q - r * cc;
      cp_async16(Cd + (size_t)r * T.cst + 2 * c, sp.C + (size_t)(ra + r) * g.kc + 2 * c);
    } else if (q < nc + nv) {
      const int x = q - nc, r = x / vc, c = x - r * vc;
      cp_async16(Vd + (size_t)r * T.vst + 2 * c, sp.V + (size_t)(ra + r) * g.cap + 2 * c);
    } else {
      const int x = q - nc - nv, r = x / wc, c = x - r * wc;
      cp_async16(Wd + (size_t)r * T.wst + 2 * c, sp.W + (size_t)(ra + r) * g.s + 2 * c);
    }
  }
}

// run `body(tile, stage, rows)` over the block's nr rows, S - 1 tiles ahead
template <class F>
__device__ __forceinline__ void ring_pass(const Ring& g, const Tile& T, const StageSpec& sp,
                                          int nr, F body) {
  const int ntiles = (nr + T.R - 1) / T.R;
  __syncthreads();  // this block's earlier writes of the rows are done
  for (int i = 0; i < g.S - 1; ++i) {
    if (i < ntiles) ring_issue(g, T, sp, i, nr, i % g.S);
    cp_async_commit();
  }
  for (int i = 0; i < ntiles; ++i) {
    const int st = i % g.S;
    if (i + g.S - 1 < ntiles) ring_issue(g, T, sp, i + g.S - 1, nr, (i + g.S - 1) % g.S);
    cp_async_commit();          // (possibly empty: the group count stays in step)
    cp_async_wait(g.S - 1);     // tile i's group is complete
    __syncthreads();
    body(i, st, min(T.R, nr - i * T.R));
    __syncthreads();            // stage st is free again
  }
}

// acc[j][e] (t-tile w + 8 j of the warp, chain e = 4-row chunk parity) +=
// sum over the tile's rows of X(r, t) Y[r][c]; X = [a (ka cols, ld lda) |
// b (ld ldb)], Y ld ldy, rows nt (a multiple of 8 except for the last tile)
template <int NY, int NT>
__device__ __forceinline__ void tile_gram(double (&acc)[NT][2][(NY + 7) / 8][2], const double* xa,
                                          int lda, int ka, const double* xb, int ldb, int kx,
                                          const double* Y, int ldy, int ny, int nt) {
  constexpr int NH = (NY + 7) / 8;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int t = (wid + 8 * j) * 8 + g;
    if ((wid + 8 * j) * 8 >= kx) break;  // warp-uniform
    const bool tok = t < kx;
    const double* xc = tok ? (t < ka ? xa + t : xb + (t - ka)) : xa;
    const int ldc = (tok && t >= ka) ? ldb : lda;
    for (int r0 = 0; r0 < nt; r0 += 8) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = r0 + 4 * e + t4;
        const bool ok = r < nt;
        const double a = (ok && tok) ? xc[(size_t)r * ldc] : 0.0;
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int c = h * 8 + g;
          const double b = (ok && c < ny) ? Y[(size_t)r * ldy + c] : 0.0;
          dmma884(acc[j][e][h], a, b);
        }
      }
    }
  }
}

template <int NY, int NT>
__device__ __forceinline__ void acc_zero(double (&acc)[NT][2][(NY + 7) / 8][2]) {
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int h = 0; h < (NY + 7) / 8; ++h) acc[j][e][h][0] = acc[j][e][h][1] = 0.0;
}

// partial[t * ny + c] <- acc (the warp's t-tiles; chains summed 0 + 1)
template <int NY, int NT>
__device__ __forceinline__ void tile_gram_store(const double (&acc)[NT][2][(NY + 7) / 8][2],
                                                int kx, int ny, double* part) {
  constexpr int NH = (NY + 7) / 8;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int t = (wid + 8 * j) * 8 + g;
    if (t >= kx) continue;
#pragma unroll
    for (int h = 0; h < NH; ++h)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int c = h * 8 + 2 * t4 + i;
        if (c < ny) part[t * ny + c] = acc[j][0][h][i] + acc[j][1][h][i];
      }
  }
}

// Y[r][c] -= sum_t X(r, t) G[t][c] for the tile's rows (8-row blocks over the
// warps); X = [a (ka, lda) | b (ldb)], kx columns; G row-major ld ny (smem)
template <int NY>
__device__ __forceinline__ void tile_update(const double* xa, int lda, int ka, const double* xb,
                                            int ldb, int kx, const double* G, double* Y, int ldy,
                                            int ny, int nt) {
  constexpr int NH = (NY + 7) / 8;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int nch = (kx + 3) >> 2;
  for (int rb = wid * 8; rb < nt; rb += (kOrthT / 32) * 8) {
    const int r = rb + g;
    const bool rok = r < nt;
    const double* ra = xa + (size_t)(rok ? r : 0) * lda;
    const double* rbp = xb + (size_t)(rok ? r : 0) * ldb - ka;
    // four independent accumulator chains (chunk mod 4), summed in a fixed
    // order: the DMMA latency is not serialised over kx / 4 chunks
    double acc4[4][NH][2];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int h = 0; h < NH; ++h) acc4[u][h][0] = acc4[u][h][1] = 0.0;
    for (int ch0 = 0; ch0 < nch; ch0 += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = (ch0 + u) * 4 + t4;
        const double a = (rok && t < kx) ? (t < ka ? ra[t] : rbp[t]) : 0.0;
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int c = h * 8 + g;
          const double b = (t < kx && c < ny) ? G[t * ny + c] : 0.0;
          dmma884(acc4[u][h], a, b);
        }
      }
    }
    double acc[NH][2];
#pragma unroll
    for (int h = 0; h < NH; ++h)
#pragma unroll
      for (int i = 0; i < 2; ++i)
        acc[h][i] = (acc4[0][h][i] + acc4[1][h][i]) + (acc4[2][h][i] + acc4[3][h][i]);
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
}

// y = x[piv] R^-1 for the tile's rows (thread per row): the new V block
template <int NY>
__device__ __forceinline__ void tile_trsm(const double* X, int ldx, double* Y, int ldy, int nt,
                                          int m, const double* R, const int* piv,
                                          const double* rinv) {
  for (int r = threadIdx.x; r < nt; r += kOrthT) {
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
}

// pass 1: part[t * sb + c] = sum over the block's rows of [C | V](r, t) W[r][c]
template <int NY>
__device__ __noinline__ void staged_gram1(Ring g, const double* C, int k, const double* V,
                                          int total, const double* W, int sb, int nr,
                                          double* part) {
  constexpr int NT = 2;
  const int kx = k + total;
  double acc[NT][2][(NY + 7) / 8][2];
  acc_zero<NY, NT>(acc);
  const Tile T = make_tile(g, k > 0, total, true);
  const StageSpec sp{C, V, W};
  ring_pass(g, T, sp, nr, [&](int, int st, int nt) {
    tile_gram<NY, NT>(acc, T.Cs(g, st), T.cst, k, T.Vs(g, st), T.vst, kx, T.Ws(g, st), T.wst,
                      sb, nt);
  });
  tile_gram_store<NY, NT>(acc, kx, sb, part);
  __syncthreads();
}

// pass 2: W1 = W - [C | V] G (G = [B; H1], kx x sb, smem), written back to
// W; part2[t * sb + c] = sum of [V | W1](r, t) W1[r][c] (t < total + sb)
template <int NY>
__device__ __noinline__ void staged_upd1_gram2(Ring g, const double* C, int k, const double* V,
                                               int total, double* W, int sb, int nr,
                                               const double* G, double* part) {
  constexpr int NT = 2;
  const int kx = k + total, kx2 = total + sb;
  double acc[NT][2][(NY + 7) / 8][2];
  acc_zero<NY, NT>(acc);
  const Tile T = make_tile(g, k > 0, total, true);
  const StageSpec sp{C, V, W};
  ring_pass(g, T, sp, nr, [&](int tile, int st, int nt) {
    double* Wt = T.Ws(g, st);
    tile_update<NY>(T.Cs(g, st), T.cst, k, T.Vs(g, st), T.vst, kx, G, Wt, T.wst, sb, nt);
    __syncthreads();
    // W1 rows back to HBM (pass 3 and the cycle end read them)
    double* Wg = W + (size_t)tile * T.R * g.s;
    for (int q = threadIdx.x; q < nt * sb; q += kOrthT) {
      const int r = q / sb, c = q - r * sb;
      Wg[(size_t)r * g.s + c] = Wt[(size_t)r * T.wst + c];
    }
    tile_gram<NY, NT>(acc, T.Vs(g, st), T.vst, total, Wt, T.wst, kx2, Wt, T.wst, sb, nt);
  });
  tile_gram_store<NY, NT>(acc, kx2, sb, part);
  __syncthreads();
}

// pass 3: W2 = W1 - V H2 (H2: total x sb, smem); with `Rq` (one Cholesky-QR
// pass suffices) the new block Q = W2[:, piv] R^-1 goes straight to Vq (ld
// cap); otherwise W2 is written back to W for the second pass
template <int NY>
__device__ __noinline__ void staged_upd2(Ring g, const double* V, int total, double* W, int sb,
                                         int nr, const double* H2, const double* Rq,
                                         const int* piv, double* Vq) {
  __shared__ double rinv[16];
  if (Rq && threadIdx.x < sb) rinv[threadIdx.x] = 1.0 / Rq[threadIdx.x * sb + threadIdx.x];
  const Tile T = make_tile(g, false, total, true);
  const StageSpec sp{nullptr, V, W};
  ring_pass(g, T, sp, nr, [&](int tile, int st, int nt) {
    double* Wt = T.Ws(g, st);
    tile_update<NY>(T.Vs(g, st), T.vst, total, T.Vs(g, st), T.vst, total, H2, Wt, T.wst, sb,
                    nt);
    __syncthreads();
    if (Rq) {
      tile_trsm<NY>(Wt, T.wst, Vq + (size_t)tile * T.R * g.cap, g.cap, nt, sb, Rq, piv, rinv);
    } else {
      double* Wg = W + (size_t)tile * T.R * g.s;
      for (int q = threadIdx.x; q < nt * sb; q += kOrthT) {
        const int r = q / sb, c = q - r * sb;
        Wg[(size_t)r * g.s + c] = Wt[(size_t)r * T.wst + c];
      }
    }
  });
  __syncthreads();
}

}  // namespace pmp

namespace pmp {

// The worker side of one cycle's inner loop for the global-row geometry
// (worker_inner in cycle_dev.cuh with the Gram / update phases replaced by
// the three staged passes above).  Same contract: steps until restart
// length, max_iters, a stop decision of the control block, or a Cholesky
// flag; the lead worker writes the final state and the done flag.
#ifndef PMP_STAGED_ATTR
#define PMP_STAGED_ATTR __noinline__
#endif
template <int NY>
__device__ PMP_STAGED_ATTR void worker_inner_staged(const CycleArgs& P, WBar& wb, const WSmem& S_, Ring ring,
                                    int r0, int nr, bool lead, int& m, int& total, int& ncols,
                                    int& it, int& status) {
  double* G = S_.G;
  double* R1 = S_.R1;
  double* R2 = S_.R2;
  double* red = S_.red;
  int* piv = S_.piv;
  int* piv2 = S_.piv2;
  int* flag = S_.flag;
  double* Wv = S_.Wv;  // this block's W rows in HBM (ld P.s)
  double* Q1 = S_.Q1;
  const int ldw = S_.ldw;
  const int sb = P.sb, k = P.k, cap = P.cap, kc = P.kc;
  double* Cr = const_cast<double*>(P.C) + (size_t)r0 * kc;
  double* Vr = P.V + (size_t)r0 * cap;
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
    cstamp(P, stp, 0);
    // ---- W = A F_0 .. F_{nfac-1} V[:, q0 : q0 + sb] ---------------------------
    const double* src = P.V + q0;
    int lds = cap;
#ifndef PMP_STAGED_CYC
#define PMP_STAGED_CYC 0
#endif
    if (PMP_STAGED_CYC) {
      // tiles dealt cyclically over the group's workers (spmm_rows_cyc)
      for (int f = P.nfac - 1; f >= 0; --f) {
        double* dst = ((P.nfac - 1 - f) & 1) ? P.T1 : P.T0;
        spmm_rows_cyc<NY, false>(P.frp[f], P.fci[f], P.fva[f], src, lds, sb, dst, P.s, P.n, wb.wi,
                                 wb.n);
        wbar(wb);
        src = dst;
        lds = P.s;
      }
      spmm_rows_cyc<NY, false>(P.arp, P.aci, P.ava, src, lds, sb, P.W, P.s, P.n, wb.wi, wb.n);
      wbar(wb);
    } else {
#ifndef PMP_STAGED_CA
#define PMP_STAGED_CA 1
#endif
    for (int f = P.nfac - 1; f >= 0; --f) {
      double* dst = ((P.nfac - 1 - f) & 1) ? P.T1 : P.T0;
      spmm_rows<NY, PMP_STAGED_CA != 0>(P.frp[f], P.fci[f], P.fva[f], src, lds, sb,
                                        dst + (size_t)r0 * P.s, P.s, r0, nr);
      wbar(wb);
      src = dst;
      lds = P.s;
    }
    spmm_rows<NY, PMP_STAGED_CA != 0>(P.arp, P.aci, P.ava, src, lds, sb, Wv, ldw, r0, nr);
    }
    cstamp(P, stp, 1);

    // ---- pass 1: [C | V]^T W ---------------------------------------------------
    const int kx = k + total;
    staged_gram1<NY>(ring, Cr, k, Vr, total, Wv, sb, nr,
                     P.partial + (size_t)(wb.wi + 1) * kx * sb);
    cstamp(P, stp, 2);
    wreduce(wb, P.partial, P.gout, kx * sb, G, sbf.B, k * sb, sbf.H1);
    cstamp(P, stp, 3);
    // ---- pass 2: W1 = W - [C | V] G, then [V | W1]^T W1 -------------------------
    const int kx2 = total + sb;
    staged_upd1_gram2<NY>(ring, Cr, k, Vr, total, Wv, sb, nr, G,
                          P.partial + (size_t)(wb.wi + 1) * kx2 * sb);
    cstamp(P, stp, 4);
    cstamp(P, stp, 5);
    wreduce(wb, P.partial, P.gout, kx2 * sb, G, sbf.H2, total * sb, nullptr);
    cstamp(P, stp, 6);
    // G_W = W1^T W1 - H2^T H2 (R2), symmetrised into red, factored before
    // pass 3 (it does not depend on W2)
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
    for (int qq = threadIdx.x; qq < sb * sb; qq += kOrthT) {
      const int i = qq / sb, j = qq % sb;
      red[qq] = 0.5 * (R2[i * sb + j] + R2[j * sb + i]);
    }
    __syncthreads();
    cstamp(P, stp, 12);
    if (threadIdx.x < 32) {
      bool ok = warp_cholesky_smem(red, sb, R1, piv, true, kCholRatio);
      if (threadIdx.x == 0) flag[0] = ok ? 0 : 1;
    }
    __syncthreads();
    bool single = false;
    if (flag[0] == 0) single = fabs(R1[0]) / fabs(R1[(sb - 1) * sb + (sb - 1)]) <= kSkipKappa;
    cstamp(P, stp, 13);
    // ---- pass 3: W2 = W1 - V H2 (and Q = W2 P R^-1 -> V when single) -------------
    staged_upd2<NY>(ring, Vr, total, Wv, sb, nr, G, (flag[0] == 0 && single) ? R1 : nullptr,
                    piv, Vr + total);
    cstamp(P, stp, 14);
    cstamp(P, stp, 7);
    if (flag[0] == 0 && !single) {
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
    cstamp(P, stp, 8);
    if (flag[0]) {
      // W2 is in P.W (this block's rows): the host Householder fallback
      status = 5;
      if (q > 0) {
        const int d = wait_flag(P.ist + 16 + q - 1, 0);
        if (d == 1) status = 0;
        if (d == 4) status = 4;
      }
      if (status == 5 && lead && P.mirror) {
        const int lens[3] = {k * sb, total * sb, total * sb};
        const int offs[3] = {P.offB, P.offH1, P.offH2};
        const double* srcs[3] = {sbf.B, sbf.H1, sbf.H2};
        for (int a = 0; a < 3; ++a)
          for (int qq = threadIdx.x; qq < lens[a]; qq += kOrthT)
            P.mirror[offs[a] + qq] = __ldcg(srcs[a] + qq);
      }
      break;
    }
    if (!single) block_trsm_rows<NY>(Q1, sb, Vr + total, cap, nr, sb, R2, nullptr);
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
    cstamp(P, stp, 9);
    wbar(wb);  // new V block (and the step outputs) visible
    cstamp(P, stp, 10);
    if (q > 0) {
      const int d = wait_flag(P.ist + 16 + q - 1, 0);
      if (d == 1 || d == 4) {
        status = d == 1 ? 0 : 4;
        break;
      }
    }
    cstamp(P, stp, 11);
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
