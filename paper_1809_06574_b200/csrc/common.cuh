// Shared device helpers for libpmorb200 (sm_100a).
//
// "Team" = the group of threads that cooperates on one least-squares column
// (one warp, or a whole CTA).  All reductions are fixed-order (shfl_xor
// butterflies + in-order smem sums), so every kernel in the library is
// bitwise deterministic run to run.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pmorb200.h"

namespace pmp {

void set_error(const char* fmt, ...);
int cuda_status(const char* where);

constexpr int kIntMax = 0x7fffffff;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int T>
struct Team {
  int tid;
  double* red;  // >= T/32 + 1 doubles of team scratch

  __device__ __forceinline__ void sync() const {
    if (T == 32)
      __syncwarp();
    else
      __syncthreads();
  }

  // Sum of one value per thread; result broadcast to every team thread.
  __device__ __forceinline__ double sum(double v) const {
    v = warp_sum(v);
    if (T == 32) return v;
    const int w = tid >> 5;
    if ((tid & 31) == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < T / 32; ++i) s += red[i];
    __syncthreads();
    return s;
  }

  // out[c] = sum_{i in [r0, r1)} f(c, i) for c in [0, ncols), parallel over
  // columns AND rows: G lanes (a power of two dividing 32) per column,
  // reduced with a fixed shfl_xor butterfly.  Caller syncs afterwards.
  template <class F>
  __device__ __forceinline__ void colsum(int ncols, int r0, int r1, F f, double* out) const {
    if (ncols <= 0) return;
    int g = 32;
    while (g > 1 && g * ncols > T) g >>= 1;
    const int groups = T / g;
    const int gid = tid / g, lig = tid % g;
    // every thread of a warp must take part in the shuffles: iterate the
    // same number of rounds in all lanes
    const int rounds = (ncols + groups - 1) / groups;
    for (int rd = 0; rd < rounds; ++rd) {
      const int c = rd * groups + gid;
      double s = 0.0;
      if (c < ncols)
        for (int i = r0 + lig; i < r1; i += g) s += f(c, i);
      for (int o = g >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (c < ncols && lig == 0) out[c] = s;
    }
  }
};

__device__ __forceinline__ int lower_bound_i(const int* a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// pmp_orth_step with an optional zero-copy mirror of its small outputs
// (orth.cu); used by the native block-step driver (gcro_host.cu)
int orth_step_mirrored(int n, const double* C, int ldc, int k, double* V, int ldv, int total,
                       int npass, double* W, int ldw, int sb, int qout, double* outB,
                       double* outH1, double* outH2, double* outR, double* outFlag, void* ws,
                       size_t ws_bytes, void* stream, const double* dbase, double* mbase);

// Raise a kernel's dynamic shared-memory limit (only ever upwards, so any
// smaller launch stays valid) and return how many blocks of `threads` fit
// per SM.  Both are cached: the CUDA attribute / occupancy queries cost
// microseconds of host time, and the block-Krylov loop launches these
// kernels tens of thousands of times.  One device per process.
inline int prepare_smem(const void* fn, size_t smem, int threads) {
  struct Lim {
    const void* fn;
    size_t max_smem;
  };
  struct Occ {
    const void* fn;
    size_t smem;
    int threads, bps;
  };
  static Lim lim[64];
  static int nlim = 0;
  static Occ occ[256];
  static int nocc = 0;
  for (int i = 0; i < nocc; ++i)
    if (occ[i].fn == fn && occ[i].smem == smem && occ[i].threads == threads) return occ[i].bps;
  int li = -1;
  for (int i = 0; i < nlim; ++i)
    if (lim[i].fn == fn) li = i;
  if (li < 0 && nlim < 64) {
    li = nlim++;
    lim[li] = {fn, 0};
  }
  if (li < 0 || lim[li].max_smem < smem) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (li >= 0) lim[li].max_smem = smem;
  }
  int bps = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, threads, smem);
  if (nocc < 256) occ[nocc++] = {fn, smem, threads, bps};
  return bps;
}

inline int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace pmp
