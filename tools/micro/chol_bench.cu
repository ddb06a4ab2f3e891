// Micro-benchmark (diagnostic): cost of the small serial pieces of the
// persistent cycle kernel, run in isolation on one block.
#include <cstdio>
#include "../../paper_1809_06574_b200/csrc/orth_dev.cuh"

namespace pmp {
void set_error(const char*, ...) {}
int cuda_status(const char*) { return 0; }
cudaError_t coop_launch(const void*, int, void**, size_t, cudaStream_t) { return cudaSuccess; }
int orth_max_grid() { return 296; }
}
using namespace pmp;

__global__ void k_bench(int m, int reps, long long* out) {
  __shared__ double G[256], A[256], R[256];
  __shared__ int piv[32];
  const int t = threadIdx.x;
  for (int q = t; q < m * m; q += blockDim.x) {
    const int i = q / m, j = q % m;
    G[q] = (i == j ? m + 1.0 : 0.0) + 1.0 / (1.0 + i + j);
  }
  __syncthreads();
  long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
  for (int r = 0; r < reps; ++r) {
    for (int q = t; q < m * m; q += blockDim.x) A[q] = G[q];
    __syncthreads();
    if (r == reps - 1) t0 = clock64();
    if (t < 32) warp_cholesky_smem(A, m, R, piv, true, 1e-5);
    __syncthreads();
    if (r == reps - 1) t1 = clock64();
    if (t < 32) warp_cholesky_reg<8>(G, m, R, piv, true, 1e-5);
    __syncthreads();
    if (r == reps - 1) t2 = clock64();
    __syncthreads();
    if (r == reps - 1) t3 = clock64();
  }
  if (t == 0) {
    out[0] = t1 - t0;
    out[1] = t2 - t1;
    out[2] = t3 - t2;
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  long long h[8];
  for (int reps : {1, 2, 10}) {
    k_bench<<<1, 256>>>(8, reps, d);
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("reps %d: chol_smem %lld cycles, chol_reg %lld cycles, syncthreads %lld cycles\n", reps,
           h[0], h[1], h[2]);
  }
  return 0;
}
