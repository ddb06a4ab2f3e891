// Sparse-structure kernels: scans, CSR<->CSC transposes, the level-0 SPAI
// pattern gather (spai.py:182-207), zero compaction (sparsecore.py:43) and
// small list helpers.  Integer work; HBM/L2-bound.
#include <stdarg.h>
#include <stdio.h>

#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace pmp {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", where, cudaGetErrorString(e));
    return PMP_ERR_CUDA;
  }
  return PMP_OK;
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// scan
// ---------------------------------------------------------------------------

static size_t scan_bytes(int n) {
  size_t b = 0;
  cub::DeviceScan::InclusiveSum(nullptr, b, (const int*)nullptr, (int*)nullptr, n > 0 ? n : 1);
  return b + 256;
}

// exclusive scan of n counts into n + 1 outputs: out[0] = 0 and an
// inclusive scan into out + 1 (out[n] = total)
static int scan_impl(int n, const int* in, int* out, void* ws, size_t bytes, cudaStream_t st) {
  size_t need = scan_bytes(n);
  if (bytes < need) {
    set_error("scan: workspace %zu < %zu", bytes, need);
    return PMP_ERR_WORKSPACE;
  }
  cudaMemsetAsync(out, 0, sizeof(int), st);
  if (n == 0) return PMP_OK;
  size_t b = need - 256;
  cudaError_t e = cub::DeviceScan::InclusiveSum(ws, b, in, out + 1, n, st);
  if (e != cudaSuccess) {
    set_error("scan: %s", cudaGetErrorString(e));
    return PMP_ERR_CUDA;
  }
  return PMP_OK;
}

// ---------------------------------------------------------------------------
// transpose
// ---------------------------------------------------------------------------

__global__ void k_count_cols(int n, const int* ptr, const int* idx, const double* vals,
                             int drop, int* cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int e = ptr[i]; e < ptr[i + 1]; ++e) {
    if (drop && vals[e] == 0.0) continue;
    atomicAdd(&cnt[idx[e]], 1);
  }
}

__global__ void k_fill_cols(int n, const int* ptr, const int* idx, const double* vals, int drop,
                            const int* out_ptr, int* cursor, int* out_idx, int* src_e) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int e = ptr[i]; e < ptr[i + 1]; ++e) {
    if (drop && vals[e] == 0.0) continue;
    int j = idx[e];
    int pos = out_ptr[j] + atomicAdd(&cursor[j], 1);
    out_idx[pos] = i;
    src_e[pos] = e;
  }
}

// sort each output segment by index (insertion sort: segments are short),
// then emit the permutation and the transposed values
__global__ void k_sort_segments(int n, const int* out_ptr, int* out_idx, int* src_e,
                                const double* vals, double* out_vals, int* perm) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  int lo = out_ptr[j], hi = out_ptr[j + 1];
  for (int a = lo + 1; a < hi; ++a) {
    int key = out_idx[a], se = src_e[a];
    int b = a - 1;
    while (b >= lo && out_idx[b] > key) {
      out_idx[b + 1] = out_idx[b];
      src_e[b + 1] = src_e[b];
      --b;
    }
    out_idx[b + 1] = key;
    src_e[b + 1] = se;
  }
  for (int a = lo; a < hi; ++a) {
    int e = src_e[a];
    if (perm) perm[e] = a;
    if (out_vals) out_vals[a] = vals[e];
  }
}

__global__ void k_fill_int(int n, int* p, int v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_permute(int nnz, const int* perm, const double* src, double* dst) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  int p = perm[e];
  if (p >= 0) dst[p] = src[e];
}

// k value arrays through one permutation (a window of factors sharing one
// pattern): blockIdx.y selects the array; perm stays L2-resident across y.
__global__ void k_permute_batch(int nnz, const int* perm, const double* src, long long sstride,
                                double* dst, long long dstride) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  int p = perm[e];
  if (p >= 0) dst[blockIdx.y * dstride + p] = src[blockIdx.y * sstride + e];
}

// ---------------------------------------------------------------------------
// level-0 pattern: I_j = rows(A(:, j)) U {j}
// ---------------------------------------------------------------------------

__global__ void k_pattern_l0_size(int n, const int* colptr, const int* rowidx, int* size) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  int lo = colptr[j], hi = colptr[j + 1];
  int pos = lo + lower_bound_i(rowidx + lo, hi - lo, j);
  size[j] = (hi - lo) + ((pos < hi && rowidx[pos] == j) ? 0 : 1);
}

__global__ void k_pattern_l0_fill(int n, const int* colptr, const int* rowidx, const int* iptr,
                                  int* iidx) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  int lo = colptr[j], hi = colptr[j + 1];
  int o = iptr[j];
  bool placed = false;
  for (int e = lo; e < hi; ++e) {
    int r = rowidx[e];
    if (!placed && r >= j) {
      if (r != j) iidx[o++] = j;
      placed = true;
    }
    iidx[o++] = r;
  }
  if (!placed) iidx[o++] = j;
}

// ---------------------------------------------------------------------------
// zero compaction
// ---------------------------------------------------------------------------

__global__ void k_count_nz_rows(int n, const int* ptr, const double* vals, int* cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = 0;
  for (int e = ptr[i]; e < ptr[i + 1]; ++e) c += (vals[e] != 0.0);
  cnt[i] = c;
}

__global__ void k_compact_rows(int n, const int* ptr, const int* idx, const double* vals,
                               const int* optr, int* oidx, double* ovals) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int o = optr[i];
  for (int e = ptr[i]; e < ptr[i + 1]; ++e) {
    double v = vals[e];
    if (v != 0.0) {
      oidx[o] = idx[e];
      ovals[o] = v;
      ++o;
    }
  }
}

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------

__global__ void k_copy_cols(int n, int nc, const double* src, int lds, const int* sc,
                            double* dst, int ldd, const int* dc) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)n * nc) return;
  int i = (int)(t / nc), c = (int)(t % nc);
  int a = sc ? sc[c] : c, b = dc ? dc[c] : c;
  dst[(size_t)i * ldd + b] = src[(size_t)i * lds + a];
}

__global__ void k_axpby_cols(int n, int nc, double alpha, const double* src, int lds,
                             const int* sc, double beta, double* dst, int ldd, const int* dc) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)n * nc) return;
  int i = (int)(t / nc), c = (int)(t % nc);
  int a = sc ? sc[c] : c, b = dc ? dc[c] : c;
  double* d = dst + (size_t)i * ldd + b;
  double v = alpha * src[(size_t)i * lds + a];
  if (beta != 0.0) v += beta * (*d);
  *d = v;
}

__global__ void k_count_flags(int n, const int* flags, int mask, int* count) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  int v = (j < n) && (flags[j] & mask);
  unsigned b = __ballot_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(count, __popc(b));
}

__global__ void k_flag_gt(int ncols, const int* cols, const double* resid, double ep,
                          int* flag) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  int j = cols ? cols[c] : c;
  flag[c] = resid[j] > ep ? 1 : 0;
}

__global__ void k_scatter_sel(int ncols, const int* cols, const int* flag, const int* pos,
                              int* out, int* count) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  if (flag[c]) out[pos[c]] = cols ? cols[c] : c;
  if (c == ncols - 1) *count = pos[c] + flag[c];
}

// final column layout after the level-1 pass: column j takes its augmented
// support when it has one (|aug_j| > 0), its base support otherwise
__global__ void k_merge_sizes(int n, const int* bptr, const int* aptr, int* size) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  int na = aptr[j + 1] - aptr[j];
  size[j] = na > 0 ? na : bptr[j + 1] - bptr[j];
}

__global__ void k_merge(int n, const int* bptr, const int* bidx, const double* bcoef,
                        const int* aptr, const int* aidx, const double* acoef, const int* optr,
                        int* oidx, double* ocoef) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int* idx;
  const double* cf;
  int lo = aptr[j], hi = aptr[j + 1];
  if (hi > lo) {
    idx = aidx, cf = acoef;
  } else {
    lo = bptr[j], hi = bptr[j + 1], idx = bidx, cf = bcoef;
  }
  int o = optr[j];
  for (int e = lo; e < hi; ++e, ++o) {
    oidx[o] = idx[e];
    ocoef[o] = cf[e];
  }
}

}  // namespace pmp

using namespace pmp;

extern "C" {

const char* pmp_last_error(void) { return g_err; }
int pmp_version(void) { return 1; }

size_t pmp_scan_workspace(int n) { return scan_bytes(n); }

int pmp_scan(int n, const int32_t* in, int32_t* out, void* ws, size_t bytes, void* st) {
  if (n < 0) return PMP_ERR_ARG;
  return scan_impl(n, in, out, ws, bytes, S(st));
}

size_t pmp_transpose_workspace(int n, int nnz) {
  return 256 + sizeof(int) * ((size_t)n + 1) * 2 + sizeof(int) * (size_t)nnz + scan_bytes(n) +
         1024;
}

int pmp_transpose(int n, int nnz, const int32_t* ptr, const int32_t* idx, const double* vals,
                  int drop, int32_t* out_ptr, int32_t* out_idx, double* out_vals, int32_t* perm,
                  void* ws, size_t bytes, void* st) {
  if (n < 0 || nnz < 0 || (drop && !vals)) {
    set_error("pmp_transpose: bad arguments");
    return PMP_ERR_ARG;
  }
  if (bytes < pmp_transpose_workspace(n, nnz)) {
    set_error("pmp_transpose: workspace too small");
    return PMP_ERR_WORKSPACE;
  }
  cudaStream_t s = S(st);
  char* w = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  int* cnt = (int*)w;
  w += sizeof(int) * ((size_t)n + 1);
  int* cursor = (int*)w;
  w += sizeof(int) * ((size_t)n + 1);
  int* src_e = (int*)w;
  w += sizeof(int) * (size_t)nnz;
  w = (char*)(((uintptr_t)w + 255) & ~(uintptr_t)255);
  const int B = 256;
  cudaMemsetAsync(cnt, 0, sizeof(int) * ((size_t)n + 1) * 2, s);
  if (perm && drop) k_fill_int<<<ceil_div(nnz, B), B, 0, s>>>(nnz, perm, -1);
  if (n > 0) k_count_cols<<<ceil_div(n, B), B, 0, s>>>(n, ptr, idx, vals, drop, cnt);
  int rc = scan_impl(n, cnt, out_ptr, w, scan_bytes(n), s);
  if (rc) return rc;
  if (n > 0) {
    k_fill_cols<<<ceil_div(n, B), B, 0, s>>>(n, ptr, idx, vals, drop, out_ptr, cursor, out_idx,
                                             src_e);
    k_sort_segments<<<ceil_div(n, B), B, 0, s>>>(n, out_ptr, out_idx, src_e, vals, out_vals,
                                                 perm);
  }
  return cuda_status("pmp_transpose");
}

int pmp_permute(int nnz, const int32_t* perm, const double* src, double* dst, void* st) {
  if (nnz <= 0) return PMP_OK;
  k_permute<<<ceil_div(nnz, 256), 256, 0, S(st)>>>(nnz, perm, src, dst);
  return cuda_status("pmp_permute");
}

int pmp_permute_batch(int nnz, const int32_t* perm, int k, const double* src, long long sstride,
                      double* dst, long long dstride, void* st) {
  if (nnz < 0 || k < 0 || k > 65535) {
    set_error("pmp_permute_batch: bad nnz / k");
    return PMP_ERR_ARG;
  }
  if (nnz == 0 || k == 0) return PMP_OK;
  dim3 grid(ceil_div(nnz, 256), k);
  k_permute_batch<<<grid, 256, 0, S(st)>>>(nnz, perm, src, sstride, dst, dstride);
  return cuda_status("pmp_permute_batch");
}

size_t pmp_pattern_l0_workspace(int n) {
  return 512 + sizeof(int) * ((size_t)n + 1) + scan_bytes(n);
}

int pmp_pattern_l0_ptr(int n, const int32_t* colptr, const int32_t* rowidx, int32_t* iptr,
                       void* ws, size_t bytes, void* st) {
  if (n < 0) return PMP_ERR_ARG;
  if (bytes < pmp_pattern_l0_workspace(n)) {
    set_error("pmp_pattern_l0: workspace too small");
    return PMP_ERR_WORKSPACE;
  }
  cudaStream_t s = S(st);
  char* w = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  int* size = (int*)w;
  w += sizeof(int) * ((size_t)n + 1);
  w = (char*)(((uintptr_t)w + 255) & ~(uintptr_t)255);
  if (n > 0) k_pattern_l0_size<<<ceil_div(n, 256), 256, 0, s>>>(n, colptr, rowidx, size);
  int rc = scan_impl(n, size, iptr, w, scan_bytes(n), s);
  if (rc) return rc;
  return cuda_status("pmp_pattern_l0_ptr");
}

int pmp_pattern_l0(int n, const int32_t* colptr, const int32_t* rowidx, int32_t* iptr,
                   int32_t* iidx, void* ws, size_t bytes, void* st) {
  int rc = pmp_pattern_l0_ptr(n, colptr, rowidx, iptr, ws, bytes, st);
  if (rc) return rc;
  if (n > 0) k_pattern_l0_fill<<<ceil_div(n, 256), 256, 0, S(st)>>>(n, colptr, rowidx, iptr, iidx);
  return cuda_status("pmp_pattern_l0");
}

size_t pmp_compact_workspace(int n) { return 512 + sizeof(int) * ((size_t)n + 1) + scan_bytes(n); }

int pmp_compact_zeros(int n, const int32_t* ptr, const int32_t* idx, const double* vals,
                      int32_t* optr, int32_t* oidx, double* ovals, void* ws, size_t bytes,
                      void* st) {
  if (bytes < pmp_compact_workspace(n)) {
    set_error("pmp_compact_zeros: workspace too small");
    return PMP_ERR_WORKSPACE;
  }
  cudaStream_t s = S(st);
  char* w = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  int* cnt = (int*)w;
  w += sizeof(int) * ((size_t)n + 1);
  w = (char*)(((uintptr_t)w + 255) & ~(uintptr_t)255);
  if (n > 0) k_count_nz_rows<<<ceil_div(n, 256), 256, 0, s>>>(n, ptr, vals, cnt);
  int rc = scan_impl(n, cnt, optr, w, scan_bytes(n), s);
  if (rc) return rc;
  if (n > 0) k_compact_rows<<<ceil_div(n, 256), 256, 0, s>>>(n, ptr, idx, vals, optr, oidx, ovals);
  return cuda_status("pmp_compact_zeros");
}

int pmp_copy_cols(int n, int nc, const double* src, int lds, const int32_t* sc, double* dst,
                  int ldd, const int32_t* dc, void* st) {
  long long tot = (long long)n * nc;
  if (tot <= 0) return PMP_OK;
  k_copy_cols<<<ceil_div(tot, 256), 256, 0, S(st)>>>(n, nc, src, lds, sc, dst, ldd, dc);
  return cuda_status("pmp_copy_cols");
}

int pmp_axpby_cols(int n, int nc, double alpha, const double* src, int lds, const int32_t* sc,
                   double beta, double* dst, int ldd, const int32_t* dc, void* st) {
  long long tot = (long long)n * nc;
  if (tot <= 0) return PMP_OK;
  k_axpby_cols<<<ceil_div(tot, 256), 256, 0, S(st)>>>(n, nc, alpha, src, lds, sc, beta, dst, ldd, dc);
  return cuda_status("pmp_axpby_cols");
}

int pmp_count_flags(int n, const int32_t* flags, int mask, int32_t* count, void* st) {
  if (n <= 0) return PMP_OK;
  k_count_flags<<<ceil_div(n, 256), 256, 0, S(st)>>>(n, flags, mask, count);
  return cuda_status("pmp_count_flags");
}

size_t pmp_select_workspace(int ncols) {
  return 512 + sizeof(int) * ((size_t)ncols + 1) * 2 + scan_bytes(ncols);
}

int pmp_select_gt(int ncols, const int32_t* cols, const double* resid, double ep, int32_t* out,
                  int32_t* count, void* ws, size_t bytes, void* st) {
  if (bytes < pmp_select_workspace(ncols)) {
    set_error("pmp_select_gt: workspace too small");
    return PMP_ERR_WORKSPACE;
  }
  if (ncols <= 0) return PMP_OK;
  cudaStream_t s = S(st);
  char* w = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  int* flag = (int*)w;
  w += sizeof(int) * ((size_t)ncols + 1);
  int* pos = (int*)w;
  w += sizeof(int) * ((size_t)ncols + 1);
  w = (char*)(((uintptr_t)w + 255) & ~(uintptr_t)255);
  k_flag_gt<<<ceil_div(ncols, 256), 256, 0, s>>>(ncols, cols, resid, ep, flag);
  int rc = scan_impl(ncols, flag, pos, w, scan_bytes(ncols), s);
  if (rc) return rc;
  k_scatter_sel<<<ceil_div(ncols, 256), 256, 0, s>>>(ncols, cols, flag, pos, out, count);
  return cuda_status("pmp_select_gt");
}

int pmp_merge_sizes(int n, const int32_t* bptr, const int32_t* aptr, int32_t* size, void* st) {
  if (n <= 0) return PMP_OK;
  k_merge_sizes<<<ceil_div(n, 256), 256, 0, S(st)>>>(n, bptr, aptr, size);
  return cuda_status("pmp_merge_sizes");
}

int pmp_merge_columns(int n, const int32_t* bptr, const int32_t* bidx, const double* bcoef,
                      const int32_t* aptr, const int32_t* aidx, const double* acoef,
                      const int32_t* optr, int32_t* oidx, double* ocoef, void* st) {
  if (n <= 0) return PMP_OK;
  k_merge<<<ceil_div(n, 256), 256, 0, S(st)>>>(n, bptr, bidx, bcoef, aptr, aidx, acoef, optr, oidx,
                                               ocoef);
  return cuda_status("pmp_merge_columns");
}

}  // extern "C"
