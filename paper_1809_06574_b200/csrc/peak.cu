// FP64 pipe peaks of this B200, measured live (the LS roofline
// must be quoted against a MEASURED DFMA / DMMA peak, not the nominal one).
//
//   kind 0: DFMA  -- every thread runs 8 independent fma chains
//   kind 1: DMMA  -- every warp runs 4 independent mma.sync m8n8k4 f64 chains
//
// One launch of 4 x #SMs blocks x 256 threads, timed with CUDA events on the
// caller's stream (after one warm-up launch); returns TFLOP/s.
#include <cuda_runtime.h>

#include "common.cuh"

namespace pmp {

__global__ void __launch_bounds__(256) k_peak_dfma(int iters, double seed, double* out) {
  double a[8];
  const double b = 1.0 + 1e-12 * threadIdx.x, c = 1e-9;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + i;
  for (int t = 0; t < iters; ++t) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[blockIdx.x] = s;  // keeps the chains alive
}

__global__ void __launch_bounds__(256) k_peak_dmma(int iters, double seed, double* out) {
  double a = seed + threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-6;
  double d[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i][0] = d[i][1] = 0.0;
  for (int t = 0; t < iters; ++t) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile(
            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
            : "+d"(d[i][0]), "+d"(d[i][1])
            : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.678) out[blockIdx.x] = s;
}

}  // namespace pmp

using namespace pmp;

extern "C" int pmp_fp64_peak(int kind, int iters, double* tflops, void* stream) {
  if ((kind != 0 && kind != 1) || iters <= 0 || !tflops) { set_error("pmp_fp64_peak: bad arguments"); return PMP_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = 4 * sms, threads = 256;
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double) * blocks) != cudaSuccess) return cuda_status("pmp_fp64_peak malloc");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0.f;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0, st);
    if (kind == 0)
      k_peak_dfma<<<blocks, threads, 0, st>>>(iters, 1.0, out);
    else
      k_peak_dmma<<<blocks, threads, 0, st>>>(iters, 1.0, out);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const int rc = cuda_status("pmp_fp64_peak");
  if (rc) return rc;
  double flops;
  if (kind == 0)
    flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  else
    flops = 2.0 * 8 * 8 * 4 * 4 * 8 * (double)iters * blocks * (threads / 32);
  *tflops = flops / (ms * 1e-3) / 1e12;
  return 0;
}
