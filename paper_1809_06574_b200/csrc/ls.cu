// Kernels 3/4: batched per-column least squares for the SPAI build
// (spai.py:229-292, min ||e_j - A p||) and the SPAI update (update.py:66-75,
// min ||a1_j - A_l q||), plus the level-1 pattern augmentation
// (spai.py:210-222).
//
// One "team" (a warp, or a 128/256-thread CTA) owns one column at a time.
// Per column it
//   1. gathers J = unique(target rows U rows(A(:,k)), k in I_j)
//      (spai.py:237-240) by a bitonic sort + compaction in team memory,
//   2. scatters the dense |J| x |I| block A(J, I) and the target into team
//      memory (column-major, leading dimension |J|),
//   3. runs a column-pivoted Householder QR on it (LAPACK geqp3/dlarfg
//      conventions), decides the rank by |R_kk| > eps |R_00| (gelsy uses
//      rcond = eps, spai.py:250), back-substitutes -- or, when rank
//      deficient, applies the RZ complete orthogonal factorisation to get
//      gelsy's minimum-norm solution,
//   4. recomputes the residual ||t - A(J,I) z||_2 explicitly (spai.py:252),
//   5. writes z into the CSC slots of column j.
// Team memory is shared memory (warp / CTA tiers) or a global-memory slice
// (columns whose dense block exceeds shared memory).  All reductions are
// fixed-order, so results are bitwise reproducible.
#include <float.h>
#include <stdlib.h>

#include "common.cuh"

namespace pmp {

struct LsParams {
  int mode;  // 0 solve, 1 plan (|J|), 2 export J, 3 SNE, 4 solve + record the
             // symbolic plan, 5 solve from a recorded plan, 6 record only
  int ncols;
  const int* cols;
  int n;
  const int* iptr;
  const int* iidx;
  const int* acolptr;
  const int* arowidx;
  const double* avals;
  const int* tcolptr;  // NULL => identity target
  const int* trowidx;
  const double* tvals;
  double* coef;
  double* resid;
  int* flags;
  int* msize;
  const int* jptr;
  int* jidx;
  int lcap, mcap, ncap;
  size_t team_bytes;
  char* gws;
  // symbolic plan of the listed columns (modes 4 / 5): per column c at
  // plan + plan_ptr[c]: |J|, tot (entries of A(:, I_j)), tl, off[0..|I_j|],
  // then (value index, pos | col << 16) for the tot A entries and the tl
  // target entries (value index -1 for the identity target)
  int* plan;
  const int* plan_ptr;
};

// several systems sharing the plan's structures (segmented tier): their
// values and outputs, passed by value in the kernel parameters (no device
// pointer arrays); nsys <= 1 uses LsParams' avals / coef / resid / flags
constexpr int kLsMaxSys = PMP_LS_MAX_SYSTEMS;
struct LsMulti {
  int nsys;
  const double* avals[kLsMaxSys];
  double* coef[kLsMaxSys];
  double* resid[kLsMaxSys];
  int* flags[kLsMaxSys];
};

// team memory layout --------------------------------------------------------
struct LsMem {
  double* M;     // mcap * (ncap + 1)
  double* nrm;   // ncap + 1
  double* w;     // ncap + 1
  double* z;     // ncap + 1
  double* tau;   // ncap + 1
  double* red;   // 16
  int* list;     // lcap
  int* sup;      // ncap + 1
  int* perm;     // ncap + 1
  int* off;      // ncap + 2
  int* misc;     // 16
};

__host__ __device__ inline size_t align16(size_t b) { return (b + 15) & ~(size_t)15; }

__host__ __device__ inline size_t ls_team_bytes(int lcap, int mcap, int ncap) {
  size_t d = (size_t)mcap * (ncap + 1) + 4 * (size_t)(ncap + 1) + 16;
  size_t i = (size_t)lcap + 3 * (size_t)(ncap + 1) + 1 + 16;
  return align16(d * sizeof(double)) + align16(i * sizeof(int));
}

__device__ inline LsMem ls_carve(char* base, int lcap, int mcap, int ncap) {
  LsMem m;
  double* d = reinterpret_cast<double*>(base);
  m.M = d;
  d += (size_t)mcap * (ncap + 1);
  m.nrm = d;
  d += ncap + 1;
  m.w = d;
  d += ncap + 1;
  m.z = d;
  d += ncap + 1;
  m.tau = d;
  d += ncap + 1;
  m.red = d;
  d += 16;
  size_t dbytes = align16(((size_t)mcap * (ncap + 1) + 4 * (size_t)(ncap + 1) + 16) * sizeof(double));
  int* i = reinterpret_cast<int*>(base + dbytes);
  m.list = i;
  i += lcap;
  m.sup = i;
  i += ncap + 1;
  m.perm = i;
  i += ncap + 1;
  m.off = i;
  i += ncap + 2;
  m.misc = i;
  return m;
}

// in-place exclusive prefix of a[0..len) into a[0..len] (a[len] = total);
// executed by warp 0 of the team, the caller syncs afterwards
__device__ inline void warp0_exclusive_scan(int* a, int len, int tid) {
  if (tid >= 32) return;
  int carry = 0;
  for (int base = 0; base < len; base += 32) {
    int i = base + tid;
    int v = i < len ? a[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (tid >= o) x += y;
    }
    if (i < len) a[i] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (tid == 0) a[len] = carry;
}

template <int T>
__device__ inline void bitonic_sort(int* a, int lp2, const Team<T>& tm) {
  for (int k = 2; k <= lp2; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int i = tm.tid; i < lp2; i += T) {
        int ixj = i ^ jj;
        if (ixj > i) {
          int x = a[i], y = a[ixj];
          bool asc = (i & k) == 0;
          if ((x > y) == asc) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      tm.sync();
    }
  }
}

// stable in-place compaction of a[0..len) keeping keep(i, value) == true;
// returns the kept count (all team threads).  cnt: >= T/32 + 2 ints of team
// scratch.  keep() may read a[i-1] through `prev` (the original value).
template <int T, class K>
__device__ inline int team_compact(int* a, double* wv, int len, const Team<T>& tm, int* cnt, K keep) {
  const int lane = tm.tid & 31, wid = tm.tid >> 5;
  int running = 0;
  int carry_prev = kIntMax;  // original value of a[base - 1]
  for (int base = 0; base < len; base += T) {
    int i = base + tm.tid;
    int v = i < len ? a[i] : kIntMax;
    double wval = (wv && i < len) ? wv[i] : 0.0;
    int prev = (tm.tid == 0) ? carry_prev : ((i - 1 < len) ? a[i - 1] : kIntMax);
    bool f = (i < len) && keep(i, v, prev, wval);
    unsigned b = __ballot_sync(0xffffffffu, f);
    int wpre = __popc(b & ((1u << lane) - 1u));
    int woff = 0, total = __popc(b);
    int last_orig = __shfl_sync(0xffffffffu, v, 31);
    if (T > 32) {
      if (lane == 0) cnt[wid] = __popc(b);
      if (tm.tid == T - 1) cnt[T / 32] = v;
      __syncthreads();
      total = 0;
      for (int q = 0; q < T / 32; ++q) {
        if (q < wid) woff += cnt[q];
        total += cnt[q];
      }
      last_orig = cnt[T / 32];
      __syncthreads();
    } else {
      __syncwarp();
    }
    if (f) {
      a[running + woff + wpre] = v;
      if (wv) wv[running + woff + wpre] = wval;
    }
    running += total;
    carry_prev = last_orig;
    tm.sync();
  }
  return running;
}

// gather the row list for column j: target rows + rows of A(:, sup[c]);
// returns its length; pads to a power of two with kIntMax and sorts.
template <int T>
__device__ inline int gather_sorted_rows(const LsParams& P, int j, const LsMem& m, int nI, int t0,
                                         int tl, const Team<T>& tm, int* lp2_out) {
  for (int c = tm.tid; c < nI; c += T) {
    int k = m.sup[c];
    m.off[c] = P.acolptr[k + 1] - P.acolptr[k];
  }
  tm.sync();
  warp0_exclusive_scan(m.off, nI, tm.tid);
  tm.sync();
  const int L = tl + m.off[nI];
  int lp2 = 1;
  while (lp2 < L) lp2 <<= 1;
  for (int q = tm.tid; q < lp2; q += T) {
    int r;
    if (q >= L) {
      r = kIntMax;
    } else if (q < tl) {
      r = (t0 < 0) ? j : P.trowidx[t0 + q];
    } else {
      int qq = q - tl;
      // last c with off[c] <= qq
      int lo = 0, hi = nI;  // off[0] = 0 <= qq < off[nI]
      while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (m.off[mid] <= qq)
          lo = mid;
        else
          hi = mid;
      }
      int k = m.sup[lo];
      r = P.arowidx[P.acolptr[k] + (qq - m.off[lo])];
    }
    m.list[q] = r;
  }
  tm.sync();
  bitonic_sort<T>(m.list, lp2, tm);
  *lp2_out = lp2;
  return L;
}

// rank (gelsy rcond = eps) and the minimum-norm / back-substituted solution
// of the factored column block M (ld mm, R on top, Q^T t in column n):
// z -> m.w (original support order), rank -> m.misc[1].  Warp 0 works.
template <int T>
__device__ void ls_rank_solve(const LsMem& m, double* M, int mm, int n, int K, int tid) {
  if (tid < 32) {
    const int lane = tid;
    int r = 0;
    const double r00 = K > 0 ? fabs(M[0]) : 0.0;
    if (r00 > 0.0) {
      r = 1;
      while (r < K && fabs(M[r + (size_t)r * mm]) > DBL_EPSILON * r00) ++r;
    }
    double* y = m.z;  // y[0..n)
    for (int i = lane; i < n; i += 32) y[i] = (i < r) ? M[i + (size_t)n * mm] : 0.0;
    __syncwarp();
    if (r < n) {
      // RZ: annihilate R[i, r:n] for i = r-1 .. 0 (dtzrzf)
      for (int i = r - 1; i >= 0; --i) {
        double s2 = 0.0;
        for (int c = r + lane; c < n; c += 32) {
          double v = M[i + (size_t)c * mm];
          s2 += v * v;
        }
        s2 = warp_sum(s2);
        double alpha = M[i + (size_t)i * mm];
        double tz = 0.0, scal = 0.0, beta = alpha;
        if (s2 > 0.0) {
          beta = -copysign(hypot(alpha, sqrt(s2)), alpha);
          tz = (beta - alpha) / beta;
          scal = 1.0 / (alpha - beta);
        }
        __syncwarp();
        if (tz != 0.0) {
          for (int c = r + lane; c < n; c += 32) M[i + (size_t)c * mm] *= scal;
          __syncwarp();
          if (lane == 0) M[i + (size_t)i * mm] = beta;
          // rows l < i: w = R[l,i] + sum_c R[l,c] v_c
          for (int l = lane; l < i; l += 32) {
            double wl = M[l + (size_t)i * mm];
            for (int c = r; c < n; ++c) wl += M[l + (size_t)c * mm] * M[i + (size_t)c * mm];
            M[l + (size_t)i * mm] -= tz * wl;
            for (int c = r; c < n; ++c) M[l + (size_t)c * mm] -= tz * wl * M[i + (size_t)c * mm];
          }
        }
        if (lane == 0) m.tau[i] = tz;
        __syncwarp();
      }
    }
    // back substitution on the leading r x r triangle (column oriented)
    for (int k = r - 1; k >= 0; --k) {
      double zk = y[k] / M[k + (size_t)k * mm];
      __syncwarp();
      if (lane == 0) y[k] = zk;
      for (int i = lane; i < k; i += 32) y[i] -= M[i + (size_t)k * mm] * zk;
      __syncwarp();
    }
    if (r < n) {
      // x = H_{r-1} ... H_0 [y; 0]
      for (int i = 0; i < r; ++i) {
        double tz = m.tau[i];
        if (tz == 0.0) continue;
        double s = 0.0;
        for (int c = r + lane; c < n; c += 32) s += M[i + (size_t)c * mm] * y[c];
        s = warp_sum(s) + y[i];
        __syncwarp();
        if (lane == 0) y[i] -= tz * s;
        for (int c = r + lane; c < n; c += 32) y[c] -= tz * s * M[i + (size_t)c * mm];
        __syncwarp();
      }
    }
    // un-permute into w[] (original support order)
    for (int k = lane; k < n; k += 32) m.w[m.perm[k]] = y[k];
    if (lane == 0) m.misc[1] = r;
  }
}

// explicit residual t - A(J, I) z (spai.py:252) and the column's outputs;
// the caller synchronised the team after the solve
template <int T>
__device__ void ls_residual_store(const LsParams& P, const LsMem& m, const int* J, int mm, int n,
                                  int i0, int j, int t0, int tl, int tot, const int* ent,
                                  int tid) {
  Team<T> tm{tid, m.red};
  const int rank = m.misc[1];
  double* res = m.M;  // reuse
  for (int i = tid; i < mm; i += T) res[i] = 0.0;
  tm.sync();
  if (ent) {
    // same updates in the same order, positions from the plan
    for (int q = tid; q < tl; q += T) {
      const int e = ent[2 * (tot + q)];
      res[ent[2 * (tot + q) + 1] & 0xffff] = e < 0 ? 1.0 : P.tvals[e];
    }
    tm.sync();
    // The column loop below is sequential (columns share rows; its order
    // fixes the rounding) with only |A(:, c)| <= T entries of work per
    // column: with the plan entries and values read from global memory
    // inside it, every column paid two dependent L2 round trips (ncu: 19 %
    // of the team kernel's stall samples at c3).  Stage them once -- every
    // load in flight together -- behind `res` in the dead block M when they
    // fit; same updates in the same order.
    const size_t mcells = (size_t)P.mcap * (P.ncap + 1);
    double* sv = res + mm;
    int* sp = reinterpret_cast<int*>(sv + tot);
    if (T > 32 && (size_t)mm + tot + (tot + 1) / 2 <= mcells) {
      for (int q = tid; q < tot; q += T) {
        sv[q] = P.avals[ent[2 * q]];
        sp[q] = ent[2 * q + 1] & 0xffff;
      }
      tm.sync();
      for (int c = 0; c < n; ++c) {
        const double zc = m.w[c];
        for (int q = m.off[c] + tid; q < m.off[c + 1]; q += T) res[sp[q]] -= sv[q] * zc;
        tm.sync();
      }
    } else {
      for (int c = 0; c < n; ++c) {
        const double zc = m.w[c];
        for (int q = m.off[c] + tid; q < m.off[c + 1]; q += T)
          res[ent[2 * q + 1] & 0xffff] -= P.avals[ent[2 * q]] * zc;
        tm.sync();
      }
    }
  } else {
    for (int q = tid; q < tl; q += T) {
      int r = (t0 < 0) ? j : P.trowidx[t0 + q];
      res[lower_bound_i(J, mm, r)] = (t0 < 0) ? 1.0 : P.tvals[t0 + q];
    }
    tm.sync();
    for (int c = 0; c < n; ++c) {
      const double zc = m.w[c];
      const int k = m.sup[c];
      const int lo = P.acolptr[k], hi = P.acolptr[k + 1];
      for (int e = lo + tid; e < hi; e += T)
        res[lower_bound_i(J, mm, P.arowidx[e])] -= P.avals[e] * zc;
      tm.sync();
    }
  }
  double part = 0.0;
  for (int i = tid; i < mm; i += T) part += res[i] * res[i];
  const double rn2 = tm.sum(part);
  for (int c = tid; c < n; c += T) P.coef[i0 + c] = m.w[c];
  if (tid == 0) {
    P.resid[j] = sqrt(rn2);
    P.flags[j] = (rank < n) ? 1 : 0;
  }
  tm.sync();
}

// Column-pivoted Householder QR of the team's dense block M (mm x (n + 1),
// column-major, the target in column n) for the multi-warp teams (c3: 125 x
// 27 per column, 128 threads).  Same factorisation as the loop in ls_column
// (which the warp tier keeps), organised for fewer team barriers per
// reflector -- 5 instead of 11:
//  * trailing column norms are computed once and DOWNDATED with the finished
//    row of R (|a_j|^2 -= r_kj^2, recomputed exactly when the downdate has
//    cancelled below sqrt(eps) of the last exact value: xGEQP3's safeguard,
//    the pivoting the reference's gelsy itself uses) instead of being
//    recomputed from the window every step;
//  * warp 0 downdates, re-norms and finds the pivot with shuffles (first
//    maximum wins, like the sequential scan);
//  * every thread forms the reflector's scalars itself from the team sum, the
//    reflector is applied unscaled (w_j = a_kj + scal * sum x_i a_ij) so no
//    scaling pass separates the two sweeps, and the vector below the
//    diagonal is not stored (only R and Q^T t are used afterwards).
#ifndef PMP_LS_TEAM_QR
#define PMP_LS_TEAM_QR 1
#endif
template <int T>
__device__ void ls_qr_team(const LsMem& m, double* M, int mm, int n, const Team<T>& tm) {
  const int tid = tm.tid, lane = tid & 31, wid = tid >> 5;
  const unsigned full = 0xffffffffu;
  const int K = mm < n ? mm : n;
  tm.colsum(
      n, 0, mm,
      [&](int c, int i) {
        const double v = M[i + (size_t)c * mm];
        return v * v;
      },
      m.nrm);
  tm.sync();
  for (int c = tid; c < n; c += T) m.z[c] = m.nrm[c];  // last exactly computed values
  tm.sync();
  for (int k = 0; k < K; ++k) {
    if (wid == 0) {
      double best = -1.0;
      int bi = n;
      for (int c0 = k; c0 < n; c0 += 32) {
        const int c = c0 + lane;
        double v = -1.0;
        bool redo = false;
        if (c < n) {
          v = m.nrm[c];
          if (k > 0) {
            const double r = M[(k - 1) + (size_t)c * mm];
            v -= r * r;
            redo = !(v > 1.4901161193847656e-8 * m.z[c]);
          }
        }
        unsigned todo = __ballot_sync(full, redo);
        while (todo) {
          const int b = __ffs(todo) - 1;
          todo &= todo - 1;
          const int cb = c0 + b;
          double s2 = 0.0;
          for (int i = k + lane; i < mm; i += 32) {
            const double x = M[i + (size_t)cb * mm];
            s2 += x * x;
          }
          s2 = warp_sum(s2);
          if (lane == b) {
            v = s2;
            m.z[c] = s2;
          }
        }
        if (c < n) {
          m.nrm[c] = v;
          if (v > best) {
            best = v;
            bi = c;
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(full, best, o);
        const int oi = __shfl_xor_sync(full, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      __syncwarp();
      if (lane == 0) {
        const int p = bi < n ? bi : k;
        m.misc[0] = p;
        if (p != k) {
          const int t = m.perm[k];
          m.perm[k] = m.perm[p];
          m.perm[p] = t;
          m.nrm[p] = m.nrm[k];
          m.z[p] = m.z[k];
        }
      }
    }
    tm.sync();
    const int p = m.misc[0];
    double part = 0.0;
    for (int i = tid; i < mm; i += T) {
      double a = M[i + (size_t)k * mm];
      if (p != k) {
        const double b = M[i + (size_t)p * mm];
        M[i + (size_t)p * mm] = a;
        M[i + (size_t)k * mm] = b;
        a = b;
      }
      if (i > k) part += a * a;
    }
    part = warp_sum(part);
    if (lane == 0) m.red[wid] = part;
    tm.sync();
    double xn2 = 0.0;
#pragma unroll
    for (int i = 0; i < T / 32; ++i) xn2 += m.red[i];
    const double alpha = M[k + (size_t)k * mm];
    tm.sync();
    double tau = 0.0, scal = 0.0;
    if (xn2 > 0.0) {
      const double beta = -copysign(hypot(alpha, sqrt(xn2)), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
      if (tid == 0) M[k + (size_t)k * mm] = beta;
    }
    if (tid == 0) m.tau[k] = tau;
    if (tau != 0.0) {
      // w_j = a_kj + scal * sum_{i > k} x_i a_ij, j = k + 1 .. n (target included)
      {
        const int ncols = n - k;
        int g = 32;
        while (g > 1 && g * ncols > T) g >>= 1;
        const int groups = T / g;
        const int gid = tid / g, lig = tid % g;
        const int rounds = (ncols + groups - 1) / groups;
        const double* xk = M + (size_t)k * mm;
        for (int rd = 0; rd < rounds; ++rd) {
          const int c = rd * groups + gid;
          double s0 = 0.0, s1 = 0.0;
          if (c < ncols) {
            const double* aj = M + (size_t)(k + 1 + c) * mm;
            int i = k + 1 + lig;
            for (; i + g < mm; i += 2 * g) {
              s0 += xk[i] * aj[i];
              s1 += xk[i + g] * aj[i + g];
            }
            if (i < mm) s0 += xk[i] * aj[i];
          }
          double sv = s0 + s1;
          for (int o = g >> 1; o > 0; o >>= 1) sv += __shfl_xor_sync(full, sv, o);
          if (c < ncols && lig == 0) m.w[k + 1 + c] = M[k + (size_t)(k + 1 + c) * mm] + scal * sv;
        }
      }
      tm.sync();
      const int rows = mm - k, ncol = n - k;
      const int tpc = rows < T ? rows : T, ngr = T / tpc;
      const int r = tid % tpc, g2 = tid / tpc;
      if (g2 < ngr)
        for (int i0 = r; i0 < rows; i0 += tpc) {
          const int i = k + i0;
          const double vi = (i0 == 0) ? 1.0 : scal * M[i + (size_t)k * mm];
          const double tv = tau * vi;
          for (int jj = k + 1 + g2; jj <= k + ncol; jj += ngr) M[i + (size_t)jj * mm] -= tv * m.w[jj];
        }
      tm.sync();
    }
  }
}

template <int T>
__device__ void ls_column(const LsParams& P, int j, int cpos, char* mem, int tid) {
  LsMem m = ls_carve(mem, P.lcap, P.mcap, P.ncap);
  Team<T> tm{tid, m.red};
  const int i0 = P.iptr[j];
  const int nI = P.iptr[j + 1] - i0;
  int t0, tl;
  if (P.tcolptr) {
    t0 = P.tcolptr[j];
    tl = P.tcolptr[j + 1] - t0;
  } else {
    t0 = -1;
    tl = 1;
  }
  for (int c = tid; c < nI; c += T) m.sup[c] = P.iidx[i0 + c];
  int* pl = (P.mode >= 4) ? P.plan + P.plan_ptr[cpos] : nullptr;
  int mJ;
  const int* J = m.list;
  if (P.mode == 5) {
    // the recorded symbolic work of this column (same structure): no gather,
    // sort or searches
    for (int c = tid; c <= nI; c += T) m.off[c] = pl[3 + c];
    tm.sync();
    mJ = pl[0];
  } else {
    tm.sync();
    int lp2;
    const int L = gather_sorted_rows<T>(P, j, m, nI, t0, tl, tm, &lp2);
    (void)L;
    mJ = team_compact<T>(m.list, nullptr, lp2, tm, m.misc + 4,
                         [](int i, int v, int prev, double) {
                           return v != kIntMax && (i == 0 || v != prev);
                         });
  }

  if (P.mode == 1) {
    if (tid == 0) P.msize[j] = mJ;
    tm.sync();
    return;
  }
  if (P.mode == 2) {
    int o = P.jptr[j];
    for (int i = tid; i < mJ; i += T) P.jidx[o + i] = J[i];
    tm.sync();
    return;
  }

  // ---- degenerate sizes (spai.py:241-242) -----------------------------------
  if (nI == 0 || mJ == 0) {
    double s = 0.0;
    for (int q = tid; q < tl; q += T) {
      double v = (t0 < 0) ? 1.0 : P.tvals[t0 + q];
      s += v * v;
    }
    s = tm.sum(s);
    for (int c = tid; c < nI; c += T) P.coef[i0 + c] = 0.0;
    if (tid == 0) {
      P.resid[j] = sqrt(s);
      P.flags[j] = 0;
    }
    tm.sync();
    return;
  }

  const int mm = mJ, n = nI;
  double* M = m.M;
  const size_t msz = (size_t)mm * (n + 1);
  for (size_t q = tid; q < msz; q += T) M[q] = 0.0;
  for (int c = tid; c <= n; c += T) m.perm[c] = c;
  tm.sync();
  // scatter A(J, I) (off[] still holds the per-column prefix) and the target
  const int tot = m.off[n];
  int* ent = pl ? pl + 4 + n : nullptr;  // (value index, pos | col << 16) pairs
  if (P.mode == 5) {
    for (int q = tid; q < tot + tl; q += T) {
      const int e = ent[2 * q], pc = ent[2 * q + 1];
      const int pos = pc & 0xffff, col = pc >> 16;
      M[pos + (size_t)col * mm] = q < tot ? P.avals[e] : (e < 0 ? 1.0 : P.tvals[e]);
    }
  } else {
    if (pl && tid == 0) {
      pl[0] = mJ;
      pl[1] = tot;
      pl[2] = tl;
    }
    for (int c = tid; pl && c <= n; c += T) pl[3 + c] = m.off[c];
    for (int q = tid; q < tot + tl; q += T) {
      if (q < tot) {
        int lo = 0, hi = n;
        while (hi - lo > 1) {
          int mid = (lo + hi) >> 1;
          if (m.off[mid] <= q)
            lo = mid;
          else
            hi = mid;
        }
        int e = P.acolptr[m.sup[lo]] + (q - m.off[lo]);
        int pos = lower_bound_i(J, mm, P.arowidx[e]);
        M[pos + (size_t)lo * mm] = P.avals[e];
        if (ent) {
          ent[2 * q] = e;
          ent[2 * q + 1] = pos | (lo << 16);
        }
      } else {
        int qq = q - tot;
        int r = (t0 < 0) ? j : P.trowidx[t0 + qq];
        double v = (t0 < 0) ? 1.0 : P.tvals[t0 + qq];
        const int pos = lower_bound_i(J, mm, r);
        M[pos + (size_t)n * mm] = v;
        if (ent) {
          ent[2 * q] = (t0 < 0) ? -1 : t0 + qq;
          ent[2 * q + 1] = pos | (n << 16);
        }
      }
    }
  }
  tm.sync();
  if (P.mode == 6) return;  // symbolic record only (the register tier solves)

  // ---- column-pivoted Householder QR ----------------------------------------
  const int K = mm < n ? mm : n;
  if (T > 32 && PMP_LS_TEAM_QR) {
    ls_qr_team<T>(m, M, mm, n, tm);
  } else
  for (int k = 0; k < K; ++k) {
    // squared norms of the trailing columns over rows k..m-1
    tm.colsum(
        n - k, k, mm,
        [&](int c, int i) {
          double v = M[i + (size_t)(k + c) * mm];
          return v * v;
        },
        m.nrm + k);
    tm.sync();
    if (tid == 0) {
      int p = k;
      double best = m.nrm[k];
      for (int c = k + 1; c < n; ++c)
        if (m.nrm[c] > best) {
          best = m.nrm[c];
          p = c;
        }
      m.misc[0] = p;
      if (p != k) {
        int t = m.perm[k];
        m.perm[k] = m.perm[p];
        m.perm[p] = t;
      }
    }
    tm.sync();
    const int p = m.misc[0];
    if (p != k) {
      for (int i = tid; i < mm; i += T) {
        double a = M[i + (size_t)k * mm];
        M[i + (size_t)k * mm] = M[i + (size_t)p * mm];
        M[i + (size_t)p * mm] = a;
      }
      tm.sync();
    }
    // dlarfg on M[k:m, k]
    double part = 0.0;
    for (int i = k + 1 + tid; i < mm; i += T) {
      double v = M[i + (size_t)k * mm];
      part += v * v;
    }
    const double xn2 = tm.sum(part);
    if (tid == 0) {
      double alpha = M[k + (size_t)k * mm];
      double tau = 0.0, scal = 0.0;
      if (xn2 > 0.0) {
        double beta = -copysign(hypot(alpha, sqrt(xn2)), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
        M[k + (size_t)k * mm] = beta;
      }
      m.tau[k] = tau;
      m.w[n] = scal;  // temporary slot
    }
    tm.sync();
    const double tau = m.tau[k];
    if (tau != 0.0) {
      const double scal = m.w[n];
      for (int i = k + 1 + tid; i < mm; i += T) M[i + (size_t)k * mm] *= scal;
      tm.sync();
      // w_j = M[k,j] + sum_{i>k} v_i M[i,j] for j = k+1..n (rhs included)
      tm.colsum(
          n - k, k + 1, mm,
          [&](int c, int i) { return M[i + (size_t)k * mm] * M[i + (size_t)(k + 1 + c) * mm]; },
          m.w + k + 1);
      tm.sync();
      for (int c = tid; c < n - k; c += T) m.w[k + 1 + c] += M[k + (size_t)(k + 1 + c) * mm];
      tm.sync();
      const int rows = mm - k, ncol = n - k;
      // threads over the window's rows (v_k = 1 implicitly), column groups
      // when the window is shorter than the team: one division per step
      // instead of a division and a modulo per element; same arithmetic
      const int tpc = rows < T ? rows : T, ngr = T / tpc;
      const int r = tid % tpc, g = tid / tpc;
      if (g < ngr)
        for (int i0 = r; i0 < rows; i0 += tpc) {
          const int i = k + i0;
          const double vi = (i0 == 0) ? 1.0 : M[i + (size_t)k * mm];
          for (int jj = k + 1 + g; jj <= k + ncol; jj += ngr)
            M[i + (size_t)jj * mm] -= tau * m.w[jj] * vi;
        }
      tm.sync();
    }
  }

  ls_rank_solve<T>(m, M, mm, n, K, tid);
  tm.sync();
  ls_residual_store<T>(P, m, J, mm, n, i0, j, t0, tl, tot, ent, tid);
}

template <int T, bool GLOBAL>
__global__ void k_ls(LsParams P) {
  extern __shared__ __align__(16) char smem[];
  const int per_block = blockDim.x / T;
  const int team = threadIdx.x / T;
  const int tid = threadIdx.x % T;
  char* mem = GLOBAL ? (P.gws + (size_t)blockIdx.x * P.team_bytes) : (smem + (size_t)team * P.team_bytes);
  for (int c = blockIdx.x * per_block + team; c < P.ncols; c += gridDim.x * per_block) {
    const int j = P.cols ? P.cols[c] : c;
    ls_column<T>(P, j, c, mem, tid);
  }
}

// ---------------------------------------------------------------------------
// Segmented register tier for columns with a plan (modes 4 / 5) whose dense
// block is small: |J| <= MR rows, |I| < SEG columns (c1 13 x 5, c2/c4 25 x 7,
// their boundary columns).  A warp solves 32 / SEG columns at once, one
// SEG-lane segment per column and ONE LANE PER COLUMN of [A(J, I) | t]:
// lane c keeps column c (all its rows) in registers, so norms, reflector
// applications and updates are lane-local FMA chains; only the pivot choice
// (3-4 shuffle steps) and the reflector broadcast (one shuffle per row) cross
// lanes.  Same algorithm as ls_column: column pivoting on the trailing norms
// (largest, earliest position on ties), LAPACK dlarfg reflectors, rank by
// |R_kk| > eps |R_00|, column-oriented back substitution, explicit residual
// over the original block in the original support order.  Columns that turn
// out rank deficient (or |J| < |I|) are finished by the whole warp with the
// team-memory RZ code (ls_rank_solve / ls_residual_store).
//
// Several systems per launch (nsys > 1): problem g = sys * ncols + c solves
// column c of the shared plan against system sys's values (sys_avals[sys])
// into sys_coef / sys_resid / sys_flags[sys] -- one launch builds the SPAI
// updates of a whole window of systems that share their structures.
// ---------------------------------------------------------------------------

// double reciprocal / square root without libm slow-path calls: hardware
// approximations refined by Newton steps to ~1 ulp (finite, normal inputs)
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__device__ __forceinline__ double sqrt_nr(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-0.5 * x * r, r, 1.5);
  r = r * fma(-0.5 * x * r, r, 1.5);
  const double s = x * r;
  return fma(fma(-s, s, x), 0.5 * r, s);
}

#ifndef PMP_LSSEG_ILP
#define PMP_LSSEG_ILP 1
#endif

template <int MR, int SEG>
struct SegLayout {
  static constexpr int kTile = MR * SEG + 8;  // original block [MR][SEG] (+pad: bank spread)
  // R rows 0..SEG-1 (ld SEG; the reflector buffer during the QR), then z /
  // Q^T t (SEG), the position -> column map (SEG ints), +1 pad so the
  // segments' broadcast reads fall in different banks
  static constexpr int kRyMain = SEG * SEG > MR ? SEG * SEG : MR;
  static constexpr int kRy = kRyMain + SEG + SEG / 2 + 1;
  static constexpr int kPPW = 32 / SEG;
  __host__ __device__ static size_t gen_bytes() { return ls_team_bytes(1, MR, SEG); }
  __host__ __device__ static size_t warp_bytes() {
    return align16((size_t)kPPW * (kTile + kRy) * sizeof(double) + 16) + gen_bytes();
  }
};

template <int MR, int SEG>
__global__ void __launch_bounds__(256, 2) k_ls_seg(const LsParams P, const LsMulti S) {
  using Lay = SegLayout<MR, SEG>;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int PPW = Lay::kPPW;
  extern __shared__ __align__(16) char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int seg = lane / SEG, sl = lane % SEG;
  char* wmem = smem + (size_t)wid * Lay::warp_bytes();
  double* A = reinterpret_cast<double*>(wmem) + (size_t)seg * (Lay::kTile + Lay::kRy);
  double* RY = A + Lay::kTile;
  double* Z = RY + Lay::kRyMain;
  int* wflag = reinterpret_cast<int*>(reinterpret_cast<double*>(wmem) +
                                      (size_t)PPW * (Lay::kTile + Lay::kRy));
  const LsMem gm = ls_carve(wmem + Lay::warp_bytes() - Lay::gen_bytes(), 1, MR, SEG);

  const int nsys = S.nsys > 0 ? S.nsys : 1;
  const long long total = (long long)P.ncols * nsys;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long base = ((long long)blockIdx.x * (blockDim.x >> 5) + wid) * PPW; base < total;
       base += nwarps * PPW) {
    const long long g = base + seg;
    const bool valid = g < total;
    int sys = 0, c = 0;
    if (valid) {
      sys = (int)(g / P.ncols);
      c = (int)(g - (long long)sys * P.ncols);
    }
    const double* avals = nsys > 1 ? S.avals[sys] : P.avals;
    double* coef = nsys > 1 ? S.coef[sys] : P.coef;
    double* resid = nsys > 1 ? S.resid[sys] : P.resid;
    int* flags = nsys > 1 ? S.flags[sys] : P.flags;
    int j = 0, i0 = 0, n = 0, mm = 0, tot = 0, tl = 0, t0 = -1;
    const int* pl = nullptr;
    if (valid) {
      j = P.cols ? P.cols[c] : c;
      i0 = P.iptr[j];
      n = P.iptr[j + 1] - i0;
      pl = P.plan + P.plan_ptr[c];
      mm = pl[0];
      tot = pl[1];
      tl = pl[2];
      t0 = P.tcolptr ? P.tcolptr[j] : -1;
    }
    const bool degen = valid && (n == 0 || mm == 0);
    bool fast = valid && !degen;
    const int* ent = fast ? pl + 4 + n : nullptr;

    // ---- original block [A(J, I) | t] -> tile (row-major, ld SEG) -> registers
    if (fast)
      for (int i = 0; i < mm; ++i) A[i * SEG + sl] = 0.0;
    __syncwarp();
#if PMP_LSSEG_ILP
    // batches of 8 entries per lane: every plan load of a batch, then every
    // value gather, then the smem stores (two dependent round trips per
    // batch instead of two per entry)
    if (fast)
      for (int q0 = sl; q0 < tot + tl; q0 += 8 * SEG) {
        int ee[8], pp[8];
        double vv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int q = q0 + u * SEG;
          const bool ok = q < tot + tl;
          ee[u] = ok ? ent[2 * q] : 0;
          pp[u] = ok ? ent[2 * q + 1] : -1;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int q = q0 + u * SEG;
          vv[u] = pp[u] < 0 ? 0.0 : (q < tot ? avals[ee[u]] : (ee[u] < 0 ? 1.0 : P.tvals[ee[u]]));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (pp[u] >= 0) A[(pp[u] & 0xffff) * SEG + (pp[u] >> 16)] = vv[u];
      }
#else
    if (fast)
      for (int q = sl; q < tot + tl; q += SEG) {
        const int e = ent[2 * q], pc = ent[2 * q + 1];
        A[(pc & 0xffff) * SEG + (pc >> 16)] =
            q < tot ? avals[e] : (e < 0 ? 1.0 : P.tvals[e]);
      }
#endif
    __syncwarp();
    double a[MR];
#pragma unroll
    for (int i = 0; i < MR; ++i) a[i] = (fast && i < mm) ? A[i * SEG + sl] : 0.0;
    const bool iscol = fast && sl < n;
    const bool isrhs = fast && sl == n;
    int mypos = sl;  // current position of this lane's column (pivoting)
    const int K = mm < n ? mm : n;

    // ---- column-pivoted Householder QR ------------------------------------
#pragma unroll
    for (int k = 0; k < SEG - 1; ++k) {
      const bool act = fast && k < K;
      // trailing norms over rows k.. (rows > k summed first: the pivot's
      // dlarfg needs that part alone)
#if PMP_LSSEG_ILP
      // four interleaved partial sums: the 31-long dependent FMA chain was
      // the step's critical path
      double sq[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = k + 1; i < MR; ++i) sq[(i - k - 1) & 3] += a[i] * a[i];
      const double sgt = (sq[0] + sq[1]) + (sq[2] + sq[3]);
#else
      double sgt = 0.0;
#pragma unroll
      for (int i = k + 1; i < MR; ++i) sgt += a[i] * a[i];
#endif
      const bool cand = act && iscol && mypos >= k;
      double bv = cand ? a[k] * a[k] + sgt : -1.0;
      int bp = cand ? mypos : 0x7fffffff;
      int bl = sl;
#pragma unroll
      for (int o = 1; o < SEG; o <<= 1) {
        const double ov = __shfl_xor_sync(FULL, bv, o);
        const int op = __shfl_xor_sync(FULL, bp, o);
        const int ol = __shfl_xor_sync(FULL, bl, o);
        if (ov > bv || (ov == bv && op < bp)) {
          bv = ov;
          bp = op;
          bl = ol;
        }
      }
      // swap positions k <-> bp
      if (act) {
        if (sl == bl)
          mypos = k;
        else if (iscol && mypos == k)
          mypos = bp;
      }
      // dlarfg on the pivot lane's column, rows k..
      double tau = 0.0, scal = 0.0;
      if (act && sl == bl) {
        const double alpha = a[k];
        if (sgt > 0.0) {
          // (call-free sqrt / reciprocal: a libm slow-path call here would
          // spill the register-resident column around every step)
          const double beta = -copysign(sqrt_nr(fma(alpha, alpha, sgt)), alpha);
          tau = (beta - alpha) * rcp_nr(beta);
          scal = rcp_nr(alpha - beta);
          a[k] = beta;
        }
        if (tau != 0.0) {
#pragma unroll
          for (int i = k + 1; i < MR; ++i) a[i] *= scal;
        }
      }
      tau = __shfl_sync(FULL, tau, seg * SEG + bl);
      // the reflector v (rows > k) -> the segment's broadcast buffer
      if (act && sl == bl) {
#pragma unroll
        for (int i = k + 1; i < MR; ++i) RY[i] = a[i];
      }
      __syncwarp();
      // w = a[k] + sum_{i > k} v_i a[i];  a -= tau w v  (columns right of the
      // pivot and the right-hand side)
      if (act && tau != 0.0 && ((iscol && mypos > k) || isrhs)) {
#if PMP_LSSEG_ILP
        double wq[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int i = k + 1; i < MR; ++i) wq[(i - k - 1) & 3] += RY[i] * a[i];
        double w = (wq[0] + wq[1]) + (wq[2] + wq[3]);
#else
        double w = 0.0;
#pragma unroll
        for (int i = k + 1; i < MR; ++i) w += RY[i] * a[i];
#endif
        w += a[k];
        a[k] -= tau * w;
        // re-read v (volatile) instead of holding all of it in registers:
        // that doubles the live set and spills the column
        const volatile double* vv = RY;
#pragma unroll
        for (int i = k + 1; i < MR; ++i) a[i] -= tau * w * vv[i];
      }
      __syncwarp();
    }

    // ---- R, Q^T t -> smem; rank and back substitution (segment leader) ------
    if (iscol) {
#pragma unroll
      for (int i = 0; i < SEG - 1; ++i)
        if (i < n) RY[i * SEG + mypos] = a[i];
      reinterpret_cast<int*>(Z + SEG)[mypos] = sl;
    }
    if (isrhs) {
#pragma unroll
      for (int i = 0; i < SEG - 1; ++i)
        if (i < n) Z[i] = a[i];
    }
    __syncwarp();
#if PMP_LSSEG_ILP
    // rank (leading |R_ii| > eps |R_00|, hostls.cpp) by a segment ballot and
    // the back substitution across the segment's lanes: lane i keeps z_i,
    // each step broadcasts z_k / R_kk (reciprocal of lane k's diagonal) and
    // the lanes above subtract; the fixed SEG - 1 steps keep every shuffle
    // warp-uniform (segments have different n)
    {
      const double r00 = (fast && K > 0) ? fabs(RY[0]) : 0.0;
      const bool okd = fast && sl < K && r00 > 0.0 &&
                       (sl == 0 || fabs(RY[sl * SEG + sl]) > DBL_EPSILON * r00);
      const unsigned bal = __ballot_sync(FULL, okd);
      const unsigned sbits = (bal >> (seg * SEG)) & ((SEG == 32) ? 0xffffffffu : ((1u << SEG) - 1u));
      const int r = __ffs(~sbits) - 1;
      const bool full = fast && r == n;
      double z = (full && sl < n) ? Z[sl] : 0.0;
      const double rd = (full && sl < n) ? 1.0 / RY[sl * SEG + sl] : 0.0;
#pragma unroll
      for (int k = SEG - 2; k >= 0; --k) {
        const double zk = __shfl_sync(FULL, z * rd, seg * SEG + k);
        if (full && k < n) {
          if (sl == k) z = zk;
          else if (sl < k) z -= RY[sl * SEG + k] * zk;
        }
      }
      if (full && sl < n) Z[sl] = z;
      __syncwarp();
      if (valid && !degen) fast = full;
    }
#else
    if (fast && sl == 0) {
      int r = 0;
      const double r00 = K > 0 ? fabs(RY[0]) : 0.0;
      if (r00 > 0.0) {
        r = 1;
        while (r < K && fabs(RY[r * SEG + r]) > DBL_EPSILON * r00) ++r;
      }
      if (r == n) {
        for (int k = r - 1; k >= 0; --k) {
          const double zk = Z[k] / RY[k * SEG + k];
          Z[k] = zk;
          for (int i = 0; i < k; ++i) Z[i] -= RY[i * SEG + k] * zk;
        }
      } else {
        fast = false;  // (leader only; shared below)
      }
      wflag[seg] = fast ? 0 : 1;
    }
    __syncwarp();
    if (valid && !degen) fast = wflag[seg] == 0;
#endif

    // ---- coefficients (original support order) and the explicit residual
    //      t - A(J, I) z over the original block, columns in support order --
    double zo = 0.0;
    if (fast && iscol) zo = Z[mypos];
    __syncwarp();
    if (fast && iscol) {
      RY[sl] = zo;
      coef[i0 + sl] = zo;
    }
    if (degen)
      for (int q = sl; q < n; q += SEG) coef[i0 + q] = 0.0;
    __syncwarp();
    double part = 0.0;
    if (fast) {
#if PMP_LSSEG_ILP
      // the lane's rows together (independent chains interleave); per row
      // and for the sum over rows the same order as the row loop
      constexpr int RU = (MR + SEG - 1) / SEG;
      double res[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const int i = sl + u * SEG;
        res[u] = i < mm ? A[i * SEG + n] : 0.0;
      }
      for (int cc = 0; cc < n; ++cc) {
        const double zc = RY[cc];
#pragma unroll
        for (int u = 0; u < RU; ++u) {
          const int i = sl + u * SEG;
          if (i < mm) res[u] -= A[i * SEG + cc] * zc;
        }
      }
#pragma unroll
      for (int u = 0; u < RU; ++u)
        if (sl + u * SEG < mm) part += res[u] * res[u];
#else
      for (int i = sl; i < mm; i += SEG) {
        double res = A[i * SEG + n];
        for (int cc = 0; cc < n; ++cc) res -= A[i * SEG + cc] * RY[cc];
        part += res * res;
      }
#endif
    } else if (degen) {
      for (int q = sl; q < tl; q += SEG) {
        const double v = (t0 < 0) ? 1.0 : P.tvals[t0 + q];
        part += v * v;
      }
    }
#pragma unroll
    for (int o = SEG >> 1; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
    if ((fast || degen) && sl == 0) {
      resid[j] = sqrt(part);
      flags[j] = 0;
    }

    // ---- rank-deficient columns: the whole warp, team-memory RZ path --------
    // (from the segment's R rows and Q^T t in shared memory: the RZ solve
    // reads rows < |I| only, the residual the plan and the values)
    const bool defic = valid && !degen && !fast;
    unsigned need = __ballot_sync(FULL, defic && sl == 0);
    while (need) {
      const int L = __ffs(need) - 1;
      need &= need - 1;
      const int ss = L / SEG;
      const int mm_s = __shfl_sync(FULL, mm, L), n_s = __shfl_sync(FULL, n, L);
      const int K_s = mm_s < n_s ? mm_s : n_s;
      const int i0_s = __shfl_sync(FULL, i0, L), j_s = __shfl_sync(FULL, j, L);
      const int t0_s = __shfl_sync(FULL, t0, L), tl_s = __shfl_sync(FULL, tl, L);
      const int tot_s = __shfl_sync(FULL, tot, L), sys_s = __shfl_sync(FULL, sys, L);
      const int* pl_s = reinterpret_cast<const int*>(
          __shfl_sync(FULL, reinterpret_cast<unsigned long long>(pl), L));
      __syncwarp();
      const double* RYs = reinterpret_cast<double*>(wmem) + (size_t)ss * (Lay::kTile + Lay::kRy) +
                          Lay::kTile;
      const double* Zs = RYs + Lay::kRyMain;
      const int* perm_s = reinterpret_cast<const int*>(Zs + SEG);
      const int rows_s = K_s;
      for (int q = lane; q < rows_s * n_s; q += 32) {
        const int i = q % rows_s, cq = q / rows_s;
        gm.M[i + cq * mm_s] = RYs[i * SEG + cq];
      }
      for (int q = lane; q < rows_s; q += 32) gm.M[q + n_s * mm_s] = Zs[q];
      for (int q = lane; q < n_s; q += 32) gm.perm[q] = perm_s[q];
      for (int q = lane; q <= n_s; q += 32) gm.off[q] = pl_s[3 + q];
      __syncwarp();
      LsParams Q = P;
      if (nsys > 1) {
        Q.avals = S.avals[sys_s];
        Q.coef = S.coef[sys_s];
        Q.resid = S.resid[sys_s];
        Q.flags = S.flags[sys_s];
      }
      ls_rank_solve<32>(gm, gm.M, mm_s, n_s, K_s, lane);
      __syncwarp();
      ls_residual_store<32>(Q, gm, nullptr, mm_s, n_s, i0_s, j_s, t0_s, tl_s, tot_s,
                            pl_s + 4 + n_s, lane);
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// Large columns (dense A(J, I) beyond shared memory, e.g. the power-law
// config c5: median 2450 x 30, tail 10948 x 230 while each column of A(J, I)
// holds only ~40 nonzeros): corrected semi-normal equations.  G = M^T M and
// M^T t come from sparse dot products of the CSC columns (merge
// intersections), never forming the dense block; pivoted Cholesky of G; one
// step of iterative refinement on the explicit residual r = t - M z over J
// (which also gives the reported residual, spai.py:252).  With
// kappa(M) sqrt(eps) << 1 this matches the Householder solution to ~kappa
// eps; a (near) rank-deficient G (min R_kk <= 1e-6 R_00) flags the column
// (flags bit 1) so the host re-solves it with the dense pivoted-QR kernel.
// ---------------------------------------------------------------------------

__host__ __device__ inline size_t sne_team_bytes(int lcap, int mcap, int ncap) {
  size_t d = (size_t)mcap + (size_t)ncap * ncap + 5 * (size_t)(ncap + 1) + 16;
  size_t i = (size_t)lcap + 3 * (size_t)(ncap + 1) + 1 + 16;
  return align16(d * sizeof(double)) + align16(i * sizeof(int));
}

// sparse dot of two sorted CSC columns
__device__ inline double col_dot(const LsParams& P, int a, int b) {
  int i = P.acolptr[a], ie = P.acolptr[a + 1];
  int j = P.acolptr[b], je = P.acolptr[b + 1];
  double s = 0.0;
  while (i < ie && j < je) {
    const int ra = P.arowidx[i], rb = P.arowidx[j];
    if (ra == rb) {
      s += P.avals[i] * P.avals[j];
      ++i;
      ++j;
    } else if (ra < rb) {
      ++i;
    } else {
      ++j;
    }
  }
  return s;
}

// dot of CSC column a with the target column j (identity: e_j)
__device__ inline double col_dot_target(const LsParams& P, int a, int j) {
  int i = P.acolptr[a], ie = P.acolptr[a + 1];
  if (!P.tcolptr) {
    int pos = i + lower_bound_i(P.arowidx + i, ie - i, j);
    return (pos < ie && P.arowidx[pos] == j) ? P.avals[pos] : 0.0;
  }
  int t = P.tcolptr[j], te = P.tcolptr[j + 1];
  double s = 0.0;
  while (i < ie && t < te) {
    const int ra = P.arowidx[i], rt = P.trowidx[t];
    if (ra == rt) {
      s += P.avals[i] * P.tvals[t];
      ++i;
      ++t;
    } else if (ra < rt) {
      ++i;
    } else {
      ++t;
    }
  }
  return s;
}

template <int T>
__device__ void sne_column(const LsParams& P, int j, char* mem, int tid) {
  const int lcap = P.lcap, mcap = P.mcap, ncap = P.ncap;
  double* d = reinterpret_cast<double*>(mem);
  double* r = d;
  d += mcap;
  double* G = d;
  d += (size_t)ncap * ncap;
  double* z = d;
  d += ncap + 1;
  double* dz = d;
  d += ncap + 1;
  double* bt = d;
  d += ncap + 1;
  double* gd = d;  // diagonal scratch
  d += ncap + 1;
  double* red = d + (ncap + 1);
  const size_t dbytes =
      align16(((size_t)mcap + (size_t)ncap * ncap + 5 * (size_t)(ncap + 1) + 16) * sizeof(double));
  int* ib = reinterpret_cast<int*>(mem + dbytes);
  LsMem m;
  m.list = ib;
  m.sup = ib + lcap;
  m.perm = m.sup + ncap + 1;
  m.off = m.perm + ncap + 1;
  m.misc = m.off + ncap + 2;
  Team<T> tm{tid, red};
  const int i0 = P.iptr[j];
  const int n = P.iptr[j + 1] - i0;
  int t0, tl;
  if (P.tcolptr) {
    t0 = P.tcolptr[j];
    tl = P.tcolptr[j + 1] - t0;
  } else {
    t0 = -1;
    tl = 1;
  }
  for (int c = tid; c < n; c += T) {
    m.sup[c] = P.iidx[i0 + c];
    m.perm[c] = c;
  }
  tm.sync();
  int lp2;
  gather_sorted_rows<T>(P, j, m, n, t0, tl, tm, &lp2);
  const int mJ = team_compact<T>(m.list, nullptr, lp2, tm, m.misc + 4,
                                 [](int i, int v, int prev, double) {
                                   return v != kIntMax && (i == 0 || v != prev);
                                 });
  const int* J = m.list;
  // G = M^T M (upper triangle computed, mirrored), bt = M^T t
  const int npairs = n * (n + 1) / 2;
  for (int q = tid; q < npairs; q += T) {
    // q -> (a, b), a <= b, row-major upper triangle
    int a = (int)((2.0 * n + 1.0 - sqrt((2.0 * n + 1.0) * (2.0 * n + 1.0) - 8.0 * q)) / 2.0);
    while (a > 0 && a * n - a * (a - 1) / 2 > q) --a;
    while ((a + 1) * n - (a + 1) * a / 2 <= q) ++a;
    const int b = a + (q - (a * n - a * (a - 1) / 2));
    const double v = col_dot(P, m.sup[a], m.sup[b]);
    G[a * ncap + b] = v;
    G[b * ncap + a] = v;
  }
  for (int c = tid; c < n; c += T) bt[c] = col_dot_target(P, m.sup[c], j);
  tm.sync();
  // pivoted Cholesky in place (upper factor in G's upper triangle; the
  // permutation acts symmetrically: perm[k] = original column at position k)
  int ok = 1;
  const double g00 = 1.0;
  (void)g00;
  double r00 = 0.0;
  for (int k = 0; k < n; ++k) {
    if (tid == 0) {
      int p = k;
      double best = G[k * ncap + k];
      for (int c = k + 1; c < n; ++c)
        if (G[c * ncap + c] > best) {
          best = G[c * ncap + c];
          p = c;
        }
      m.misc[0] = p;
    }
    tm.sync();
    const int p = m.misc[0];
    if (p != k) {
      for (int c = tid; c < n; c += T) {  // swap rows k, p
        double t = G[k * ncap + c];
        G[k * ncap + c] = G[p * ncap + c];
        G[p * ncap + c] = t;
      }
      tm.sync();
      for (int c = tid; c < n; c += T) {  // swap columns k, p
        double t = G[c * ncap + k];
        G[c * ncap + k] = G[c * ncap + p];
        G[c * ncap + p] = t;
      }
      if (tid == 0) {
        int t = m.perm[k];
        m.perm[k] = m.perm[p];
        m.perm[p] = t;
      }
      tm.sync();
    }
    const double dkk = G[k * ncap + k];
    if (k == 0) r00 = sqrt(fmax(dkk, 0.0));
    if (!(dkk > 0.0) || sqrt(dkk) <= 1e-6 * r00) {
      ok = 0;
      break;
    }
    const double rkk = sqrt(dkk);
    for (int c = k + tid; c < n; c += T) gd[c] = (c == k) ? rkk : G[k * ncap + c] / rkk;
    tm.sync();
    for (int c = k + tid; c < n; c += T) G[k * ncap + c] = gd[c];
    const int w = n - k - 1;
    for (int q = tid; q < w * w; q += T) {
      const int a = k + 1 + q / w, b = k + 1 + q % w;
      if (b >= a) {
        G[a * ncap + b] -= gd[a] * gd[b];
        if (b != a) G[b * ncap + a] = G[a * ncap + b];
      }
    }
    tm.sync();
  }
  if (!ok) {
    // leave the column to the dense pivoted-QR path
    if (tid == 0) P.flags[j] = 2;
    tm.sync();
    return;
  }
  // z = P R^-1 R^-T P^T bt ; two passes: solve, residual, refine
  for (int pass = 0; pass < 2; ++pass) {
    double* y = pass == 0 ? z : dz;
    // rhs (permuted) into y: y = P^T (pass 0: bt, pass 1: M^T r)
    if (pass == 1) {
      for (int c = tid; c < n; c += T) {
        const int k = m.sup[c];
        double s = 0.0;
        for (int e = P.acolptr[k]; e < P.acolptr[k + 1]; ++e)
          s += P.avals[e] * r[lower_bound_i(J, mJ, P.arowidx[e])];
        bt[c] = s;
      }
      tm.sync();
    }
    for (int c = tid; c < n; c += T) y[c] = bt[m.perm[c]];
    tm.sync();
    if (tid < 32) {
      // forward (R^T y' = y) then backward (R x = y'), warp 0
      for (int k = 0; k < n; ++k) {
        const double yk = y[k] / G[k * ncap + k];
        __syncwarp();
        if (tid == 0) y[k] = yk;
        for (int c = k + 1 + tid; c < n; c += 32) y[c] -= G[k * ncap + c] * yk;
        __syncwarp();
      }
      for (int k = n - 1; k >= 0; --k) {
        const double yk = y[k] / G[k * ncap + k];
        __syncwarp();
        if (tid == 0) y[k] = yk;
        for (int c = tid; c < k; c += 32) y[c] -= G[c * ncap + k] * yk;
        __syncwarp();
      }
    }
    tm.sync();
    // back to support order: gd[perm[c]] = y[c]; accumulate into z (support order)
    for (int c = tid; c < n; c += T) gd[m.perm[c]] = y[c];
    tm.sync();
    if (pass == 0) {
      for (int c = tid; c < n; c += T) z[c] = gd[c];
    } else {
      for (int c = tid; c < n; c += T) z[c] += gd[c];
    }
    tm.sync();
    // explicit residual r = t - M z over J
    for (int i = tid; i < mJ; i += T) r[i] = 0.0;
    tm.sync();
    for (int q = tid; q < tl; q += T) {
      const int row = (t0 < 0) ? j : P.trowidx[t0 + q];
      r[lower_bound_i(J, mJ, row)] = (t0 < 0) ? 1.0 : P.tvals[t0 + q];
    }
    tm.sync();
    for (int c = 0; c < n; ++c) {
      const double zc = z[c];
      const int k = m.sup[c];
      for (int e = P.acolptr[k] + tid; e < P.acolptr[k + 1]; e += T)
        r[lower_bound_i(J, mJ, P.arowidx[e])] -= P.avals[e] * zc;
      tm.sync();
    }
  }
  double part = 0.0;
  for (int i = tid; i < mJ; i += T) part += r[i] * r[i];
  const double rn2 = tm.sum(part);
  for (int c = tid; c < n; c += T) P.coef[i0 + c] = z[c];
  if (tid == 0) {
    P.resid[j] = sqrt(rn2);
    P.flags[j] = 0;
  }
  tm.sync();
}

template <int T, bool GLOBAL>
__global__ void k_ls_sne(LsParams P) {
  extern __shared__ __align__(16) char smem[];
  char* mem = GLOBAL ? (P.gws + (size_t)blockIdx.x * P.team_bytes) : smem;
  for (int c = blockIdx.x; c < P.ncols; c += gridDim.x) {
    const int j = P.cols ? P.cols[c] : c;
    sne_column<T>(P, j, mem, threadIdx.x);
  }
}

__global__ void k_ls_bound(int ncols, const int* cols, const int* iptr, const int* iidx,
                           const int* acolptr, const int* tcolptr, int* lsize) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  int j = cols ? cols[c] : c;
  int L = tcolptr ? tcolptr[j + 1] - tcolptr[j] : 1;
  for (int e = iptr[j]; e < iptr[j + 1]; ++e) {
    int k = iidx[e];
    L += acolptr[k + 1] - acolptr[k];
  }
  lsize[c] = L;
}

// ---------------------------------------------------------------------------
// level-1 augmentation (spai.py:210-222)
// ---------------------------------------------------------------------------

struct AugParams {
  int mode;
  int ncols;
  const int* cols;
  int max_fill;
  const int* iptr;
  const int* iidx;
  const int* acolptr;
  const int* arowidx;
  const double* avals;
  int* newsize;
  const int* newptr;
  int* newidx;
  int lcap;
  size_t team_bytes;
  char* gws;
};

__host__ __device__ inline size_t aug_team_bytes(int lcap) {
  return align16(((size_t)lcap + 16) * sizeof(double)) +
         align16((2 * (size_t)lcap + 64 + 16) * sizeof(int));
}

// |A(r, k)| by binary search in CSC column k (0 if structurally absent)
__device__ inline double abs_entry(const AugParams& P, int r, int k) {
  int lo = P.acolptr[k], hi = P.acolptr[k + 1];
  int pos = lo + lower_bound_i(P.arowidx + lo, hi - lo, r);
  return (pos < hi && P.arowidx[pos] == r) ? fabs(P.avals[pos]) : 0.0;
}

template <int T>
__device__ void aug_column(const AugParams& P, int c, char* mem, int tid) {
  double* w = reinterpret_cast<double*>(mem);
  double* red = w + P.lcap;
  int* list = reinterpret_cast<int*>(mem + align16(((size_t)P.lcap + 16) * sizeof(double)));
  int* off = list + P.lcap;    // 64 + 16 ints: misc
  int* keepf = off + 80;       // lcap ints: top-k keep flags
  Team<T> tm{tid, red};
  const int j = P.cols ? P.cols[c] : c;
  const int b0 = P.iptr[j], nb = P.iptr[j + 1] - b0;
  const int* base = P.iidx + b0;
  const int klo = P.acolptr[j], khi = P.acolptr[j + 1];
  // two-hop candidate rows: rows(A(:, k)) for k in rows(A(:, j))
  int L = 0;
  for (int e = klo; e < khi; ++e) {
    int k = P.arowidx[e];
    L += P.acolptr[k + 1] - P.acolptr[k];
  }
  int lp2 = 1;
  while (lp2 < L) lp2 <<= 1;
  for (int q = tid; q < lp2; q += T) {
    int r = kIntMax;
    if (q < L) {
      int acc = 0;
      for (int e = klo; e < khi; ++e) {
        int k = P.arowidx[e];
        int len = P.acolptr[k + 1] - P.acolptr[k];
        if (q < acc + len) {
          r = P.arowidx[P.acolptr[k] + (q - acc)];
          break;
        }
        acc += len;
      }
    }
    list[q] = r;
  }
  tm.sync();
  bitonic_sort<T>(list, lp2, tm);
  int C0 = team_compact<T>(list, nullptr, lp2, tm, off, [](int i, int v, int prev, double) {
    return v != kIntMax && (i == 0 || v != prev);
  });
  // weights in the reference's order: k ascending over rows(A(:, j)), each
  // product and partial sum rounded (csc_matmat), exact zeros dropped
  for (int q = tid; q < C0; q += T) {
    int r = list[q];
    double acc = 0.0;
    for (int e = klo; e < khi; ++e) {
      int k = P.arowidx[e];
      double ark = abs_entry(P, r, k);
      if (ark != 0.0) acc = __dadd_rn(acc, __dmul_rn(ark, fabs(P.avals[e])));
    }
    bool in_base = false;
    int pb = lower_bound_i(base, nb, r);
    if (pb < nb && base[pb] == r) in_base = true;
    w[q] = (in_base || acc == 0.0) ? -1.0 : acc;  // -1 marks "not a candidate"
  }
  tm.sync();
  int C = team_compact<T>(list, w, C0, tm, off, [](int, int, int, double wv) { return wv >= 0.0; });
  const int room = P.max_fill - nb > 0 ? P.max_fill - nb : 0;
  int kept = C;
  if (C > room) {
    // keep the first `room` by (w desc, row asc): rank by counting
    for (int q = tid; q < C; q += T) {
      double wq = w[q];
      int rq = list[q];
      int rank = 0;
      for (int t = 0; t < C; ++t) {
        double wt = w[t];
        rank += (wt > wq) || (wt == wq && list[t] < rq);
      }
      keepf[q] = rank < room;
    }
    tm.sync();
    kept = team_compact<T>(list, w, C, tm, off,
                           [keepf](int i, int, int, double) { return keepf[i] != 0; });
  }
  if (P.mode == 0) {
    if (tid == 0) P.newsize[j] = nb + kept;
    tm.sync();
    return;
  }
  // union of two disjoint sorted lists: merge by rank
  int* out = P.newidx + P.newptr[j];
  for (int q = tid; q < nb; q += T) {
    int v = base[q];
    out[q + lower_bound_i(list, kept, v)] = v;
  }
  for (int q = tid; q < kept; q += T) {
    int v = list[q];
    out[q + lower_bound_i(base, nb, v)] = v;
  }
  tm.sync();
}

template <int T, bool GLOBAL>
__global__ void k_aug(AugParams P) {
  extern __shared__ __align__(16) char smem[];
  const int per_block = blockDim.x / T;
  const int team = threadIdx.x / T;
  const int tid = threadIdx.x % T;
  char* mem = GLOBAL ? (P.gws + (size_t)blockIdx.x * P.team_bytes) : (smem + (size_t)team * P.team_bytes);
  for (int c = blockIdx.x * per_block + team; c < P.ncols; c += gridDim.x * per_block)
    aug_column<T>(P, c, mem, tid);
}

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// PMP_LS_REG=0 disables the register warp tier (A/B experiments)
static bool ls_reg_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("PMP_LS_REG");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on != 0;
}

template <int T, bool G>
static int launch_ls(LsParams P, cudaStream_t st, size_t ws_bytes) {
  const size_t tb = P.team_bytes;
  if (G) {
    int grid = num_sms() * 2;
    if (grid > P.ncols) grid = P.ncols;
    if ((size_t)grid * tb > ws_bytes) grid = (int)(ws_bytes / tb);
    if (grid < 1) {
      set_error("pmp_ls_columns: global workspace too small (%zu < %zu)", ws_bytes, tb);
      return PMP_ERR_WORKSPACE;
    }
    k_ls<T, true><<<grid, T, 0, st>>>(P);
  } else {
    int per_block = (T == 32) ? 8 : 1;
    while (per_block > 1 && per_block * tb > 96 * 1024) per_block >>= 1;
    size_t sm = per_block * tb;
    if (sm > 227 * 1024) {
      set_error("pmp_ls_columns: team needs %zu B of shared memory", sm);
      return PMP_ERR_ARG;
    }
    prepare_smem((const void*)k_ls<T, false>, sm, T * per_block);
    int grid = ceil_div(P.ncols, per_block);
    k_ls<T, false><<<grid, T * per_block, sm, st>>>(P);
  }
  return cuda_status("pmp_ls_columns");
}

template <int MR, int SEG>
static int launch_seg(const LsParams& P, const LsMulti& S, cudaStream_t st) {
  const size_t wb = SegLayout<MR, SEG>::warp_bytes();
  const size_t sm = 8 * wb;
  prepare_smem((const void*)k_ls_seg<MR, SEG>, sm, 256);
  const long long total = (long long)P.ncols * (S.nsys > 0 ? S.nsys : 1);
  const long long per_block = 8LL * (32 / SEG);
  long long grid = (total + per_block - 1) / per_block;
  const long long cap = (long long)num_sms() * 64;
  if (grid > cap) grid = cap;
  k_ls_seg<MR, SEG><<<(int)grid, 256, sm, st>>>(P, S);
  return cuda_status("pmp_ls_columns");
}

static int launch_ls_seg(const LsParams& P, const LsMulti& S, int mcap, int ncap,
                         cudaStream_t st) {
  // (MR = 28 covers the 25-row interior subproblems of the 7-point
  // stencils without 7 rows of zero padding in every unrolled row loop)
  if (ncap <= 7)
    return mcap <= 16 ? launch_seg<16, 8>(P, S, st)
                      : (mcap <= 28 ? launch_seg<28, 8>(P, S, st) : launch_seg<32, 8>(P, S, st));
  return mcap <= 16 ? launch_seg<16, 16>(P, S, st) : launch_seg<32, 16>(P, S, st);
}

static bool seg_eligible(int mode, int team, int use_global, int mcap, int ncap) {
  return (mode == 4 || mode == 5) && team == 32 && !use_global && mcap <= 32 && ncap <= 15 &&
         ls_reg_enabled();
}

template <int T, bool G>
static int launch_aug(AugParams P, cudaStream_t st, size_t ws_bytes) {
  const size_t tb = P.team_bytes;
  if (G) {
    int grid = num_sms() * 2;
    if (grid > P.ncols) grid = P.ncols;
    if ((size_t)grid * tb > ws_bytes) grid = (int)(ws_bytes / tb);
    if (grid < 1) {
      set_error("pmp_augment: global workspace too small");
      return PMP_ERR_WORKSPACE;
    }
    k_aug<T, true><<<grid, T, 0, st>>>(P);
  } else {
    int per_block = (T == 32) ? 8 : 1;
    while (per_block > 1 && per_block * tb > 96 * 1024) per_block >>= 1;
    size_t sm = per_block * tb;
    if (sm > 227 * 1024) {
      set_error("pmp_augment: team needs %zu B of shared memory", sm);
      return PMP_ERR_ARG;
    }
    prepare_smem((const void*)k_aug<T, false>, sm, T * per_block);
    k_aug<T, false><<<ceil_div(P.ncols, per_block), T * per_block, sm, st>>>(P);
  }
  return cuda_status("pmp_augment");
}

}  // namespace pmp

using namespace pmp;

extern "C" {

size_t pmp_ls_team_bytes(int team, int lcap, int mcap, int ncap) {
  // team == 0 queries the semi-normal-equations (mode 3) layout
  if (team == 0) return sne_team_bytes(lcap, mcap, ncap);
  return ls_team_bytes(lcap, mcap, ncap);
}

int pmp_ls_bound(int ncols, const int32_t* cols, const int32_t* iptr, const int32_t* iidx,
                 const int32_t* acolptr, const int32_t* tcolptr, int32_t* lsize, void* st) {
  if (ncols <= 0) return PMP_OK;
  k_ls_bound<<<ceil_div(ncols, 256), 256, 0, reinterpret_cast<cudaStream_t>(st)>>>(
      ncols, cols, iptr, iidx, acolptr, tcolptr, lsize);
  return cuda_status("pmp_ls_bound");
}

static int ls_columns(int mode, int team, int use_global, int lcap, int mcap, int ncap, int ncols,
                      const int32_t* cols, int n, const int32_t* iptr, const int32_t* iidx,
                      const int32_t* acolptr, const int32_t* arowidx, const double* avals,
                      const int32_t* tcolptr, const int32_t* trowidx, const double* tvals,
                      double* coef, double* resid, int32_t* flags, int32_t* msize,
                      const int32_t* jptr, int32_t* jidx, int32_t* plan, const int32_t* plan_ptr,
                      void* ws, size_t ws_bytes, void* st) {
  if (mode < 0 || mode > 5 || (team != 32 && team != 128 && team != 256) || lcap < 1 ||
      mcap < 0 || ncap < 0 || ncols < 0 || (lcap & (lcap - 1)) ||
      (mode >= 4 && (!plan || !plan_ptr || mcap >= 65536 || ncap >= 32768))) {
    set_error("pmp_ls_columns: bad arguments (mode=%d team=%d lcap=%d)", mode, team, lcap);
    return PMP_ERR_ARG;
  }
  if (ncols == 0) return PMP_OK;
  LsParams P;
  P.plan = plan;
  P.plan_ptr = plan_ptr;
  P.mode = mode;
  P.ncols = ncols;
  P.cols = cols;
  P.n = n;
  P.iptr = iptr;
  P.iidx = iidx;
  P.acolptr = acolptr;
  P.arowidx = arowidx;
  P.avals = avals;
  P.tcolptr = tcolptr;
  P.trowidx = trowidx;
  P.tvals = tvals;
  P.coef = coef;
  P.resid = resid;
  P.flags = flags;
  P.msize = msize;
  P.jptr = jptr;
  P.jidx = jidx;
  P.lcap = lcap;
  P.mcap = (mode == 0 || mode >= 3) ? mcap : 0;
  P.ncap = ncap;
  P.team_bytes = ls_team_bytes(lcap, P.mcap, ncap);
  P.gws = (char*)ws;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(st);
  if (mode == 3) {
    // large columns: corrected semi-normal equations, CTA of 256 per column
    P.team_bytes = sne_team_bytes(lcap, mcap, ncap);
    const size_t tb = P.team_bytes;
    if (use_global) {
      int grid = num_sms() * 2;
      if (grid > ncols) grid = ncols;
      if ((size_t)grid * tb > ws_bytes) grid = (int)(ws_bytes / tb);
      if (grid < 1) {
        set_error("pmp_ls_columns: global workspace too small (%zu < %zu)", ws_bytes, tb);
        return PMP_ERR_WORKSPACE;
      }
      k_ls_sne<256, true><<<grid, 256, 0, s>>>(P);
    } else {
      if (tb > 227 * 1024) {
        set_error("pmp_ls_columns: SNE team needs %zu B of shared memory", tb);
        return PMP_ERR_ARG;
      }
      prepare_smem((const void*)k_ls_sne<256, false>, tb, 256);
      k_ls_sne<256, false><<<ncols, 256, tb, s>>>(P);
    }
    return cuda_status("pmp_ls_columns");
  }
  if (seg_eligible(mode, team, use_global, mcap, ncap)) {
    // small columns with a plan: segmented register tier.  A recording call
    // first records the plan only (mode 6), so the first and every replayed
    // build of a structure compute bitwise the same numbers.
    if (mode == 4) {
      P.mode = 6;
      const int rc = launch_ls<32, false>(P, s, ws_bytes);
      if (rc != PMP_OK) return rc;
    }
    P.mode = 5;
    LsMulti S;
    S.nsys = 1;
    return launch_ls_seg(P, S, mcap, ncap, s);
  }
  if (use_global) {
    if (team == 32) return launch_ls<32, true>(P, s, ws_bytes);
    if (team == 128) return launch_ls<128, true>(P, s, ws_bytes);
    return launch_ls<256, true>(P, s, ws_bytes);
  }
  if (team == 32) return launch_ls<32, false>(P, s, ws_bytes);
  if (team == 128) return launch_ls<128, false>(P, s, ws_bytes);
  return launch_ls<256, false>(P, s, ws_bytes);
}

int pmp_ls_columns(int mode, int team, int use_global, int lcap, int mcap, int ncap, int ncols,
                   const int32_t* cols, int n, const int32_t* iptr, const int32_t* iidx,
                   const int32_t* acolptr, const int32_t* arowidx, const double* avals,
                   const int32_t* tcolptr, const int32_t* trowidx, const double* tvals,
                   double* coef, double* resid, int32_t* flags, int32_t* msize,
                   const int32_t* jptr, int32_t* jidx, void* ws, size_t ws_bytes, void* st) {
  if (mode > 3) {
    set_error("pmp_ls_columns: bad arguments (modes 4 / 5 need pmp_ls_columns_planned)");
    return PMP_ERR_ARG;
  }
  return ls_columns(mode, team, use_global, lcap, mcap, ncap, ncols, cols, n, iptr, iidx, acolptr,
                    arowidx, avals, tcolptr, trowidx, tvals, coef, resid, flags, msize, jptr, jidx,
                    nullptr, nullptr, ws, ws_bytes, st);
}

int pmp_ls_columns_planned(int mode, int team, int use_global, int lcap, int mcap, int ncap,
                           int ncols, const int32_t* cols, int n, const int32_t* iptr,
                           const int32_t* iidx, const int32_t* acolptr, const int32_t* arowidx,
                           const double* avals, const int32_t* tcolptr, const int32_t* trowidx,
                           const double* tvals, double* coef, double* resid, int32_t* flags,
                           int32_t* plan, const int32_t* plan_ptr, void* ws, size_t ws_bytes,
                           void* st) {
  if (mode != 4 && mode != 5) {
    set_error("pmp_ls_columns_planned: mode must be 4 (record) or 5 (replay)");
    return PMP_ERR_ARG;
  }
  return ls_columns(mode, team, use_global, lcap, mcap, ncap, ncols, cols, n, iptr, iidx, acolptr,
                    arowidx, avals, tcolptr, trowidx, tvals, coef, resid, flags, nullptr, nullptr,
                    nullptr, plan, plan_ptr, ws, ws_bytes, st);
}

int pmp_ls_columns_multi(int mode, int team, int use_global, int lcap, int mcap, int ncap,
                         int ncols, const int32_t* cols, int n, const int32_t* iptr,
                         const int32_t* iidx, const int32_t* acolptr, const int32_t* arowidx,
                         int nsys, const double* const* h_avals, const int32_t* tcolptr,
                         const int32_t* trowidx, const double* tvals, double* const* h_coef,
                         double* const* h_resid, int32_t* const* h_flags, int32_t* plan,
                         const int32_t* plan_ptr, void* ws, size_t ws_bytes, void* st) {
  if ((mode != 4 && mode != 5) || nsys < 0 || (nsys > 0 && (!h_avals || !h_coef || !h_resid ||
                                                            !h_flags))) {
    set_error("pmp_ls_columns_multi: bad arguments (mode=%d nsys=%d)", mode, nsys);
    return PMP_ERR_ARG;
  }
  if (nsys == 0 || ncols == 0) return PMP_OK;
  int first = 0;
  if (mode == 4 || !seg_eligible(mode, team, use_global, mcap, ncap)) {
    // record on the first system (or no segmented tier): one system per call
    const int rc = ls_columns(mode, team, use_global, lcap, mcap, ncap, ncols, cols, n, iptr,
                              iidx, acolptr, arowidx, h_avals[0], tcolptr, trowidx, tvals,
                              h_coef[0], h_resid[0], h_flags[0], nullptr, nullptr, nullptr, plan,
                              plan_ptr, ws, ws_bytes, st);
    if (rc != PMP_OK) return rc;
    first = 1;
    if (!seg_eligible(5, team, use_global, mcap, ncap)) {
      for (int q = 1; q < nsys; ++q) {
        const int r2 = ls_columns(5, team, use_global, lcap, mcap, ncap, ncols, cols, n, iptr,
                                  iidx, acolptr, arowidx, h_avals[q], tcolptr, trowidx, tvals,
                                  h_coef[q], h_resid[q], h_flags[q], nullptr, nullptr, nullptr,
                                  plan, plan_ptr, ws, ws_bytes, st);
        if (r2 != PMP_OK) return r2;
      }
      return PMP_OK;
    }
  }
  // the replays: segmented tier, up to PMP_LS_MAX_SYSTEMS systems per launch
  LsParams P;
  P.plan = plan;
  P.plan_ptr = plan_ptr;
  P.mode = 5;
  P.ncols = ncols;
  P.cols = cols;
  P.n = n;
  P.iptr = iptr;
  P.iidx = iidx;
  P.acolptr = acolptr;
  P.arowidx = arowidx;
  P.avals = nullptr;
  P.tcolptr = tcolptr;
  P.trowidx = trowidx;
  P.tvals = tvals;
  P.coef = nullptr;
  P.resid = nullptr;
  P.flags = nullptr;
  P.msize = nullptr;
  P.jptr = nullptr;
  P.jidx = nullptr;
  P.lcap = lcap;
  P.mcap = mcap;
  P.ncap = ncap;
  P.team_bytes = 0;
  P.gws = nullptr;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(st);
  for (int q0 = first; q0 < nsys; q0 += kLsMaxSys) {
    LsMulti S;
    S.nsys = nsys - q0 < kLsMaxSys ? nsys - q0 : kLsMaxSys;
    for (int q = 0; q < S.nsys; ++q) {
      S.avals[q] = h_avals[q0 + q];
      S.coef[q] = h_coef[q0 + q];
      S.resid[q] = h_resid[q0 + q];
      S.flags[q] = h_flags[q0 + q];
    }
    if (S.nsys == 1) {
      P.avals = S.avals[0];
      P.coef = S.coef[0];
      P.resid = S.resid[0];
      P.flags = S.flags[0];
    }
    const int rc = launch_ls_seg(P, S, mcap, ncap, s);
    if (rc != PMP_OK) return rc;
  }
  return PMP_OK;
}

size_t pmp_augment_team_bytes(int lcap) { return aug_team_bytes(lcap); }

int pmp_augment(int mode, int lcap, int use_global, int ncols, const int32_t* cols, int max_fill,
                const int32_t* iptr, const int32_t* iidx, const int32_t* acolptr,
                const int32_t* arowidx, const double* avals, int32_t* newsize,
                const int32_t* newptr, int32_t* newidx, void* ws, size_t ws_bytes, void* st) {
  if ((mode != 0 && mode != 1) || lcap < 1 || (lcap & (lcap - 1))) {
    set_error("pmp_augment: bad arguments");
    return PMP_ERR_ARG;
  }
  if (ncols <= 0) return PMP_OK;
  AugParams P;
  P.mode = mode;
  P.ncols = ncols;
  P.cols = cols;
  P.max_fill = max_fill;
  P.iptr = iptr;
  P.iidx = iidx;
  P.acolptr = acolptr;
  P.arowidx = arowidx;
  P.avals = avals;
  P.newsize = newsize;
  P.newptr = newptr;
  P.newidx = newidx;
  P.lcap = lcap;
  P.team_bytes = aug_team_bytes(lcap);
  P.gws = (char*)ws;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(st);
  if (use_global) return launch_aug<256, true>(P, s, ws_bytes);
  if (lcap <= 2048) return launch_aug<32, false>(P, s, ws_bytes);
  return launch_aug<256, false>(P, s, ws_bytes);
}

}  // extern "C"
