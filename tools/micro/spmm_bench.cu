// Micro-benchmark of the block-row SpMM used inside the persistent solve
// (cycle_dev.cuh spmm_rows), in the solve kernel's execution geometry:
// 2 x 148 blocks of 256 threads, 128 registers, ~84 KB of dynamic shared
// memory per block, `groups` independent systems sharing the GPU (each block
// owns a contiguous row range of one system's 7-point-stencil matrix).
// Diagnostic only (DESIGN.md SpMM section quotes its numbers).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -o tools/micro/spmm_bench tools/micro/spmm_bench.cu
//   tools/micro/spmm_bench [N=128] [groups=6] [reps=5]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

constexpr int kT = 256;

struct Sys {
  const int32_t* rp;
  const int32_t* ci;
  const double* va;
  const double* X;
  double* Y;
};

struct Args {
  Sys sys[8];
  int n, gsz, rows_per_block, ring_doubles;
};

// ---- variant 0 / 1: the production loop (ld.cg or ld.ca gathers) -------------
template <int NY, bool CA>
__device__ __noinline__ void spmm_rows(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                       const double* __restrict__ va, const double* X, int ldx,
                                       int sb, double* Y, int ldy, int r0, int nr) {
  constexpr int PER = kT / NY, RPT = 2, CH = 8;
  const int c = threadIdx.x % NY, slot = threadIdx.x / NY;
  const bool col_ok = c < sb;
  for (int base = 0; base < nr; base += RPT * PER) {
    int lo[RPT], hi[RPT];
    double a0[RPT], a1[RPT];
    int len = 0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int r = base + slot + u * PER;
      lo[u] = hi[u] = 0;
      a0[u] = a1[u] = 0.0;
      if (r < nr) {
        lo[u] = __ldg(rp + r0 + r);
        hi[u] = __ldg(rp + r0 + r + 1);
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
        for (int q = 0; q < CH; ++q) {
          const double* p = X + (size_t)j[u][q] * ldx + c;
          x[u][q] = (j[u][q] >= 0 && col_ok) ? (CA ? __ldca(p) : __ldcg(p)) : 0.0;
        }
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

// ---- variant 2: asynchronous staging ---------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Tiles of TR = RPT * 256 / NY rows.  Per tile the index / value segment of
// the tile (contiguous in CSR) is copied into shared memory two tiles ahead,
// the gathered X rows (16-byte pieces) one tile ahead; the products read
// shared memory only.  Same per-row summation order as spmm_rows.
template <int NY, int RPT>
__device__ __noinline__ void spmm_rows_async(const int32_t* __restrict__ rp,
                                             const int32_t* __restrict__ ci,
                                             const double* __restrict__ va, const double* X,
                                             int ldx, double* Y, int ldy, int r0, int nr,
                                             double* ring, int ring_doubles) {
  constexpr int PER = kT / NY, TR = RPT * PER, S = 3, PC = NY / 2;
  const int c = threadIdx.x % NY, slot = threadIdx.x / NY;
  // stage = xg [EMAX * NY] | va_s [EMAX] | ci_s [EMAX ints]
  const int stage = (ring_doubles / S) & ~1;
  const int EMAX = ((stage * 8) / (NY * 8 + 8 + 4)) & ~3;
  auto xg = [&](int st) { return ring + (size_t)st * stage; };
  auto vs = [&](int st) { return ring + (size_t)st * stage + (size_t)EMAX * NY; };
  auto cs = [&](int st) { return reinterpret_cast<int*>(ring + (size_t)st * stage + (size_t)EMAX * (NY + 1)); };
  const int ntiles = (nr + TR - 1) / TR;
  const int32_t* rpb = rp + r0;
  auto bound = [&](int t) { return __ldg(rpb + min(t * TR, nr)); };
  auto issue_cv = [&](int t, int e_lo, int cnt) {
    if (cnt > EMAX) __trap();
    const int st = t % S;
    int* cd = cs(st);
    double* vd = vs(st);
    for (int q = threadIdx.x; q < cnt; q += kT) {
      cp_async4(cd + q, ci + e_lo + q);
      cp_async8(vd + q, va + e_lo + q);
    }
  };
  auto issue_x = [&](int t, int cnt) {
    const int st = t % S;
    const int* cd = cs(st);
    double* xd = xg(st);
    for (int q = threadIdx.x; q < cnt * PC; q += kT) {
      const int e = q / PC, ch = q % PC;
      cp_async16(xd + (size_t)e * NY + 2 * ch, X + (size_t)cd[e] * ldx + 2 * ch);
    }
  };
  __syncthreads();
  // prologue: cv(0), cv(1); X(0)
  int b0 = bound(0), b1 = bound(1), b2 = bound(2), b3 = bound(3);
  issue_cv(0, b0, b1 - b0);
  cp_async_commit();
  cp_async_wait0();
  __syncthreads();
  issue_x(0, b1 - b0);
  if (ntiles > 1) issue_cv(1, b1, b2 - b1);
  cp_async_commit();
  int lo[RPT], hi[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int r = slot + u * PER;
    lo[u] = hi[u] = 0;
    if (r < nr) {
      lo[u] = __ldg(rpb + r);
      hi[u] = __ldg(rpb + r + 1);
    }
  }
  for (int t = 0; t < ntiles; ++t) {
    cp_async_wait0();  // X(t), cv(t + 1)
    __syncthreads();
    if (t + 1 < ntiles) issue_x(t + 1, b2 - b1);
    const int b4 = bound(t + 4);
    if (t + 2 < ntiles) issue_cv(t + 2, b2, b3 - b2);
    cp_async_commit();
    // next tile's row extents (used one iteration from now)
    int nlo[RPT], nhi[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int r = (t + 1) * TR + slot + u * PER;
      nlo[u] = nhi[u] = 0;
      if (r < nr) {
        nlo[u] = __ldg(rpb + r);
        nhi[u] = __ldg(rpb + r + 1);
      }
    }
    const int st = t % S;
    const double* xd = xg(st);
    const double* vd = vs(st);
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int r = t * TR + slot + u * PER;
      if (r < nr) {
        double a0 = 0.0, a1 = 0.0;
        int e = lo[u] - b0;
        const int eh = hi[u] - b0;
        for (; e + 1 < eh; e += 2) {
          a0 += vd[e] * xd[(size_t)e * NY + c];
          a1 += vd[e + 1] * xd[(size_t)(e + 1) * NY + c];
        }
        if (e < eh) a0 += vd[e] * xd[(size_t)e * NY + c];
        Y[(size_t)r * ldy + c] = a0 + a1;
      }
      lo[u] = nlo[u];
      hi[u] = nhi[u];
    }
    b0 = b1;
    b1 = b2;
    b2 = b3;
    b3 = b4;
  }
  __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(kT, 2) k_bench(Args A) {
  extern __shared__ __align__(16) double sh[];
  const int grp = blockIdx.x / A.gsz, lb = blockIdx.x % A.gsz;
  const Sys S = A.sys[grp];
  const int r0 = lb * A.rows_per_block;
  const int nr = max(0, min(A.n, r0 + A.rows_per_block) - r0);
  if (nr == 0) return;
  if (V == 0) spmm_rows<8, false>(S.rp, S.ci, S.va, S.X, 8, 8, S.Y + (size_t)r0 * 8, 8, r0, nr);
  if (V == 1) spmm_rows<8, true>(S.rp, S.ci, S.va, S.X, 8, 8, S.Y + (size_t)r0 * 8, 8, r0, nr);
  if (V == 2)
    spmm_rows_async<8, 1>(S.rp, S.ci, S.va, S.X, 8, S.Y + (size_t)r0 * 8, 8, r0, nr, sh, A.ring_doubles);
  if (V == 3)
    spmm_rows_async<8, 2>(S.rp, S.ci, S.va, S.X, 8, S.Y + (size_t)r0 * 8, 8, r0, nr, sh, A.ring_doubles);
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 128;
  const int groups = argc > 2 ? atoi(argv[2]) : 6;
  const int reps = argc > 3 ? atoi(argv[3]) : 5;
  const int smem_kb = argc > 4 ? atoi(argv[4]) : 84;
  const int n = N * N * N;
  std::vector<int32_t> rp(n + 1), ci;
  std::vector<double> va;
  ci.reserve((size_t)7 * n);
  va.reserve((size_t)7 * n);
  uint64_t seed = 12345;
  auto rnd = [&]() {
    seed = seed * 6364136223846793005ULL + 1442695040888963407ULL;
    return (double)(seed >> 11) / 9007199254740992.0;
  };
  for (int i = 0; i < n; ++i) {
    rp[i] = (int)ci.size();
    const int x = i % N, y = (i / N) % N, z = i / (N * N);
    if (z > 0) ci.push_back(i - N * N), va.push_back(-rnd());
    if (y > 0) ci.push_back(i - N), va.push_back(-rnd());
    if (x > 0) ci.push_back(i - 1), va.push_back(-rnd());
    ci.push_back(i), va.push_back(6.0 + rnd());
    if (x < N - 1) ci.push_back(i + 1), va.push_back(-rnd());
    if (y < N - 1) ci.push_back(i + N), va.push_back(-rnd());
    if (z < N - 1) ci.push_back(i + N * N), va.push_back(-rnd());
  }
  rp[n] = (int)ci.size();
  const size_t nnz = ci.size();
  std::vector<double> X((size_t)n * 8);
  for (auto& v : X) v = rnd() - 0.5;
  int dev_sms = 0;
  CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, 0));
  Args A;
  memset(&A, 0, sizeof(A));
  A.n = n;
  A.gsz = 2 * dev_sms / groups;
  A.rows_per_block = (n + A.gsz - 1) / A.gsz;
  A.ring_doubles = smem_kb * 1024 / 8;
  std::vector<double*> Ys;
  for (int g = 0; g < groups; ++g) {
    int32_t *drp, *dci;
    double *dva, *dX, *dY;
    CK(cudaMalloc(&drp, (n + 1) * 4));
    CK(cudaMalloc(&dci, nnz * 4));
    CK(cudaMalloc(&dva, nnz * 8));
    CK(cudaMalloc(&dX, (size_t)n * 64));
    CK(cudaMalloc(&dY, (size_t)n * 64));
    CK(cudaMemcpy(drp, rp.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dva, va.data(), nnz * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dX, X.data(), (size_t)n * 64, cudaMemcpyHostToDevice));
    A.sys[g] = Sys{drp, dci, dva, dX, dY};
    Ys.push_back(dY);
  }
  const size_t smem = (size_t)smem_kb * 1024;
  void (*fns[4])(Args) = {k_bench<0>, k_bench<1>, k_bench<2>, k_bench<3>};
  const char* names[4] = {"ld.cg gathers (production)", "ld.ca gathers", "async staged, 32-row tiles",
                          "async staged, 64-row tiles"};
  std::vector<double> ref((size_t)n * 8), out((size_t)n * 8);
  const double alg = (double)groups * (12.0 * nnz + 4.0 * (n + 1) + 16.0 * n * 8);
  const double l2 = (double)groups * (12.0 * nnz + 4.0 * (n + 1) + 8.0 * nnz * 8 + 8.0 * n * 8);
  printf("n = %d (N = %d), nnz = %zu, groups = %d, blocks/group = %d, rows/block = %d, smem %d KB\n", n,
         N, nnz, groups, A.gsz, A.rows_per_block, smem_kb);
  printf("algorithmic bytes per pass %.1f MB, gather-level bytes %.1f MB\n", alg / 1e6, l2 / 1e6);
  for (int v = 0; v < 4; ++v) {
    CK(cudaFuncSetAttribute(fns[v], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int g = 0; g < groups; ++g) CK(cudaMemset(Ys[g], 0, (size_t)n * 64));
    fns[v]<<<A.gsz * groups, kT, smem>>>(A);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) fns[v]<<<A.gsz * groups, kT, smem>>>(A);
    CK(cudaEventRecord(e1));
    CK(cudaDeviceSynchronize());
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    CK(cudaMemcpy(out.data(), Ys[groups - 1], (size_t)n * 64, cudaMemcpyDeviceToHost));
    if (v == 0) ref = out;
    size_t bad = 0;
    for (size_t i = 0; i < out.size(); ++i) bad += memcmp(&out[i], &ref[i], 8) != 0;
    printf("variant %d %-30s %8.3f ms  alg %7.1f GB/s  gather-level %7.1f GB/s  mismatches vs v0 %zu\n", v,
           names[v], ms, alg / ms / 1e6, l2 / ms / 1e6, bad);
  }
  return 0;
}
