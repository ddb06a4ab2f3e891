// Micro-benchmark (diagnostic): cost of the small serial pieces of the
// persistent cycle kernel, run in isolation.
#include <cstdio>
#include "../../paper_1809_06574_b200/csrc/orth_dev.cuh"

namespace pmp {
void set_error(const char*, ...) {}
int cuda_status(const char*) { return 0; }
cudaError_t coop_launch(const void*, int, void**, size_t, cudaStream_t) { return cudaSuccess; }
int orth_max_grid() { return 296; }
}
using namespace pmp;

__device__ __noinline__ bool chol_generic(double* A, int m, double* R, int* piv) {
  return warp_cholesky_smem(A, m, R, piv, true, 1e-5);
}

__global__ void k_bench(int m, int reps, long long* out, int mode, const double* Gin) {
  extern __shared__ double dyn[];
  double* G = dyn;
  double* A = dyn + 256;
  double* R = dyn + 512;
  int* piv = reinterpret_cast<int*>(dyn + 768);
  const int t = threadIdx.x;
  for (int q = t; q < m * m; q += blockDim.x) {
    const int i = q / m, j = q % m;
    G[q] = Gin ? Gin[q] : (i == j ? m + 1.0 : 0.0) + 1.0 / (1.0 + i + j);
  }
  __syncthreads();
  long long best = 1LL << 60;
  for (int r = 0; r < reps; ++r) {
    for (int q = t; q < m * m; q += blockDim.x) A[q] = G[q];
    __syncthreads();
    if (t < 32) {
      const long long c0 = clock64();
      bool ok = mode == 0 ? warp_cholesky_smem(A, m, R, piv, true, 1e-5) : chol_generic(A, m, R, piv);
      const long long c1 = clock64();
      if (t == 0 && ok && c1 - c0 < best) best = c1 - c0;
    }
    __syncthreads();
  }
  if (t == 0) out[blockIdx.x] = best;
}

int main(int argc, char** argv) {
  double* gin = nullptr;
  if (argc > 1) {
    double h[64];
    FILE* f = fopen(argv[1], "rb");
    if (f && fread(h, 8, 64, f) == 64) {
      cudaMalloc(&gin, 512);
      cudaMemcpy(gin, h, 512, cudaMemcpyHostToDevice);
    }
    if (f) fclose(f);
  }
  long long* d;
  cudaMalloc(&d, 8 * 1024);
  long long h[1024];
  cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int blocks : {1, 148, 296}) {
      for (size_t sm : {(size_t)8 * 1024, (size_t)100 * 1024}) {
        k_bench<<<blocks, 256, sm>>>(8, 5, d, mode, gin);
        cudaMemcpy(h, d, 8 * blocks, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int b = 0; b < blocks; ++b) mx = h[b] > mx ? h[b] : mx;
        printf("mode %d blocks %d smem %zuKB: chol %lld cycles (block 0), max %lld\n", mode,
               blocks, sm / 1024, h[0], mx);
      }
    }
  return 0;
}
