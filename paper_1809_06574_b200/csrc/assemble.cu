// Kernel 1: A(sigma, p) = (s^2 M(p) + s D(p)) + K(p) over a fixed union
// pattern (SecondOrderModel.assemble, rpmor.py:92-107 / _eval_terms :41-49),
// or the affine sum A0 + sum_j c_j A_j (AffineFamily.evaluate,
// affine.py:118-134).  One thread per stored entry, streaming and
// HBM-bound: every term value is read once, the result written once (plus
// once more, permuted, when a transposed copy is requested).
//
// Bit-exactness: scipy evaluates each entry as
//   acc = T0; acc = acc + c_i * T_i (c_i != 0, term order)        per group
//   val = ((s*s) * m + s * d) + 1.0 * k                            groups
// with every product and sum rounded separately (complex arithmetic with a
// zero imaginary part degenerates to exactly these real operations).  The
// __dmul_rn / __dadd_rn intrinsics forbid FMA contraction so the device
// reproduces that rounding sequence bit for bit.
#include "common.cuh"

namespace pmp {

struct AsmRecipe {
  int nterms;
  int mode;  // 0 MDK, 1 affine
  int any_diag;
  double s, s2;
  const double* vals[PMP_MAX_TERMS];
  int kind[PMP_MAX_TERMS];
  int group[PMP_MAX_TERMS];
  int first[PMP_MAX_TERMS];
  double coef[PMP_MAX_TERMS];
};

__device__ __forceinline__ double term_value(const AsmRecipe& R, int t, int e, bool diag, int row) {
  if (R.kind[t] == 0) return __ldg(R.vals[t] + e);
  return diag ? __ldg(R.vals[t] + row) : 0.0;
}

// The three group accumulators (mass / damping / stiffness parts) live in
// registers: indexing a small array with the term's group put it in local
// memory (ncu on k_assemble_multi at c4: 0.8 of 32 bytes used per local
// sector, the kernel at 0.87 TB/s instead of HBM speed).  Same operations in
// the same order as the array form: bit-exact.
struct Groups {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  bool p0 = false, p1 = false, p2 = false;
  __device__ __forceinline__ void open(int g, double v) {
    if (g == 0) { a0 = v; p0 = true; }
    else if (g == 1) { a1 = v; p1 = true; }
    else { a2 = v; p2 = true; }
  }
  __device__ __forceinline__ void add(int g, double c, double v) {
    const double t = __dmul_rn(c, v);
    if (g == 0) a0 = __dadd_rn(a0, t);
    else if (g == 1) a1 = __dadd_rn(a1, t);
    else a2 = __dadd_rn(a2, t);
  }
  // (s2 * mass + s * damping) + stiffness over the groups present
  __device__ __forceinline__ double mdk(double s2, double s) const {
    bool have = false;
    double val = 0.0;
    if (p0) { val = __dmul_rn(s2, a0); have = true; }
    if (p1) { const double part = __dmul_rn(s, a1); val = have ? __dadd_rn(val, part) : part; have = true; }
    if (p2) { const double part = __dmul_rn(1.0, a2); val = have ? __dadd_rn(val, part) : part; }
    return val;
  }
};

__global__ void __launch_bounds__(256) k_assemble(AsmRecipe R, int nnz, const int* __restrict__ rowid,
                                                  const int* __restrict__ colidx,
                                                  double* __restrict__ out, const int* __restrict__ perm,
                                                  double* __restrict__ out_perm, int* zero_count) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  bool zero = false;
  if (e < nnz) {
    bool diag = false;
    int row = 0;
    if (R.any_diag) {
      row = __ldg(rowid + e);
      diag = (__ldg(colidx + e) == row);
    }
    Groups G;
#pragma unroll 1
    for (int t = 0; t < R.nterms; ++t) {
      const int g = R.group[t];
      const double v = term_value(R, t, e, diag, row);
      if (R.first[t])
        G.open(g, v);
      else
        G.add(g, R.coef[t], v);
    }
    double val;
    if (R.mode == 0) {
      val = G.mdk(R.s2, R.s);
      if (val == 0.0) val = 0.0;  // canonical +0 for dropped entries
    } else {
      val = G.a0;
      if (fabs(val) < 1e-300) val = 0.0;
    }
    zero = (val == 0.0);
    out[e] = val;
    if (perm) out_perm[perm[e]] = val;
  }
  unsigned b = __ballot_sync(0xffffffffu, zero);
  if ((threadIdx.x & 31) == 0 && b && zero_count) atomicAdd(zero_count, __popc(b));
}

// Several systems of one recipe shape (same terms, groups and opening
// terms; coefficients and shifts differ -- a parameter sweep): one thread
// per stored entry loads every term value ONCE and writes the entry of each
// system.  Per system the arithmetic is k_assemble's exactly (bit-exact).
constexpr int kAsmMaxSys = 16;
struct AsmMulti {
  int nsys;
  double s[kAsmMaxSys], s2[kAsmMaxSys];
  double coef[kAsmMaxSys][PMP_MAX_TERMS];
  double* out[kAsmMaxSys];
  double* out_perm[kAsmMaxSys];
};

// NT: the recipe's term count when it is small (the loops over the terms are
// then exactly NT long: at 16 predicated iterations per system the kernel was
// issue-bound, ncu: 88 % of issue slots), 16 = any count.
template <int NT>
__global__ void __launch_bounds__(256) k_assemble_multi(AsmRecipe R, AsmMulti S, int nnz,
                                                        const int* __restrict__ rowid,
                                                        const int* __restrict__ colidx,
                                                        const int* __restrict__ perm,
                                                        int* zero_count) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  double tv[NT];
  bool diag = false;
  int row = 0, pe = 0;
  if (e < nnz) {
    if (R.any_diag) {
      row = __ldg(rowid + e);
      diag = (__ldg(colidx + e) == row);
    }
#pragma unroll
    for (int t = 0; t < NT; ++t)
      tv[t] = (NT < PMP_MAX_TERMS || t < R.nterms) ? term_value(R, t, e, diag, row) : 0.0;
    if (perm) pe = __ldg(perm + e);
  }
  for (int q = 0; q < S.nsys; ++q) {
    bool zero = false;
    if (e < nnz) {
      Groups G;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if (NT < PMP_MAX_TERMS || t < R.nterms) {
          const int g = R.group[t];
          if (R.first[t])
            G.open(g, tv[t]);
          else
            G.add(g, S.coef[q][t], tv[t]);
        }
      }
      double val;
      if (R.mode == 0) {
        val = G.mdk(S.s2[q], S.s[q]);
        if (val == 0.0) val = 0.0;
      } else {
        val = G.a0;
        if (fabs(val) < 1e-300) val = 0.0;
      }
      zero = (val == 0.0);
      S.out[q][e] = val;
      if (perm) S.out_perm[q][pe] = val;
    }
    const unsigned b = __ballot_sync(0xffffffffu, zero);
    if (lane == 0 && b && zero_count) atomicAdd(zero_count + q, __popc(b));
  }
}

}  // namespace pmp

using namespace pmp;

extern "C" int pmp_assemble_multi(int nnz, int nterms, const double* const* h_term_vals,
                                  const int32_t* h_kind, const int32_t* h_group,
                                  const int32_t* h_first, int nsys, const double* h_coef,
                                  const double* h_s, int mode, const int32_t* d_rowid,
                                  const int32_t* d_colidx, double* const* h_out,
                                  const int32_t* d_perm, double* const* h_out_perm,
                                  int32_t* d_zero_counts, void* stream) {
  if (nterms < 1 || nterms > PMP_MAX_TERMS || nnz < 0 || (mode != 0 && mode != 1) || nsys < 0 ||
      (nsys > 0 && (!h_coef || !h_s || !h_out || (d_perm && !h_out_perm)))) {
    set_error("pmp_assemble_multi: bad arguments (nterms=%d, nnz=%d, mode=%d, nsys=%d)", nterms,
              nnz, mode, nsys);
    return PMP_ERR_ARG;
  }
  AsmRecipe R;
  R.nterms = nterms;
  R.mode = mode;
  R.s = R.s2 = 0.0;
  R.any_diag = 0;
  for (int t = 0; t < nterms; ++t) {
    R.vals[t] = h_term_vals[t];
    R.kind[t] = h_kind[t];
    R.group[t] = h_group[t];
    R.first[t] = h_first[t];
    R.coef[t] = 0.0;
    if (h_group[t] < 0 || h_group[t] > 2 || (mode == 1 && h_group[t] != 0)) {
      set_error("pmp_assemble_multi: bad group %d for term %d", h_group[t], t);
      return PMP_ERR_ARG;
    }
    if (h_kind[t] == 1) R.any_diag = 1;
  }
  if (R.any_diag && !d_rowid) {
    set_error("pmp_assemble_multi: diagonal terms need d_rowid");
    return PMP_ERR_ARG;
  }
  if (nnz == 0 || nsys == 0) return PMP_OK;
  for (int q0 = 0; q0 < nsys; q0 += kAsmMaxSys) {
    AsmMulti S;
    S.nsys = nsys - q0 < kAsmMaxSys ? nsys - q0 : kAsmMaxSys;
    for (int q = 0; q < S.nsys; ++q) {
      const double sv = h_s[q0 + q];
      S.s[q] = sv;
      S.s2[q] = sv * sv;  // host double multiply: numpy's s*s
      for (int t = 0; t < nterms; ++t) S.coef[q][t] = h_coef[(size_t)(q0 + q) * nterms + t];
      S.out[q] = h_out[q0 + q];
      S.out_perm[q] = d_perm ? h_out_perm[q0 + q] : nullptr;
    }
    int* zc = d_zero_counts ? d_zero_counts + q0 : nullptr;
    const dim3 grid(ceil_div(nnz, 256));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
#define PMP_ASM_CASE(N)                                                                  \
  case N:                                                                                \
    k_assemble_multi<N><<<grid, 256, 0, st>>>(R, S, nnz, d_rowid, d_colidx, d_perm, zc); \
    break;
    switch (nterms <= 8 ? nterms : 16) {
      PMP_ASM_CASE(1) PMP_ASM_CASE(2) PMP_ASM_CASE(3) PMP_ASM_CASE(4) PMP_ASM_CASE(5)
      PMP_ASM_CASE(6) PMP_ASM_CASE(7) PMP_ASM_CASE(8)
      default:
        k_assemble_multi<16><<<grid, 256, 0, st>>>(R, S, nnz, d_rowid, d_colidx, d_perm, zc);
    }
#undef PMP_ASM_CASE
    const int rc = cuda_status("pmp_assemble_multi");
    if (rc != PMP_OK) return rc;
  }
  return PMP_OK;
}

extern "C" int pmp_assemble(int nnz, int nterms, const double* const* h_term_vals,
                            const int32_t* h_kind, const int32_t* h_group, const int32_t* h_first,
                            const double* h_coef, int mode, double s, const int32_t* d_rowid,
                            const int32_t* d_colidx, double* d_out, const int32_t* d_perm,
                            double* d_out_perm, int32_t* d_zero_count, void* stream) {
  if (nterms < 1 || nterms > PMP_MAX_TERMS || nnz < 0 || (mode != 0 && mode != 1)) {
    set_error("pmp_assemble: bad arguments (nterms=%d, nnz=%d, mode=%d)", nterms, nnz, mode);
    return PMP_ERR_ARG;
  }
  AsmRecipe R;
  R.nterms = nterms;
  R.mode = mode;
  R.s = s;
  R.s2 = s * s;  // host double multiply: same rounding as numpy's s*s
  R.any_diag = 0;
  for (int t = 0; t < nterms; ++t) {
    R.vals[t] = h_term_vals[t];
    R.kind[t] = h_kind[t];
    R.group[t] = h_group[t];
    R.first[t] = h_first[t];
    R.coef[t] = h_coef[t];
    if (h_group[t] < 0 || h_group[t] > 2 || (mode == 1 && h_group[t] != 0)) {
      set_error("pmp_assemble: bad group %d for term %d", h_group[t], t);
      return PMP_ERR_ARG;
    }
    if (h_kind[t] == 1) R.any_diag = 1;
  }
  if (R.any_diag && !d_rowid) {
    set_error("pmp_assemble: diagonal terms need d_rowid");
    return PMP_ERR_ARG;
  }
  if (nnz == 0) return PMP_OK;
  k_assemble<<<ceil_div(nnz, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      R, nnz, d_rowid, d_colidx, d_out, d_perm, d_out_perm, d_zero_count);
  return cuda_status("pmp_assemble");
}
