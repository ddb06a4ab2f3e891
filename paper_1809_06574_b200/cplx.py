"""Complex128 on the B200 path (the reference computes in
complex128 throughout, sparsecore.py:8-10), through the real form.

A complex n x n matrix A = Ar + i Ai lives in HBM as R(A), the 2n x 2n real
matrix whose entry (r, c) block is [[Ar, -Ai], [Ai, Ar]] (every structural
entry a full 2 x 2 block, every row holding its diagonal block; built on
the device by pmp_realify).  A complex vector x is R(x) = (xr_0, xi_0,
xr_1, xi_1, ...).  Because R(A) R(x) = R(A x):

* SPAI / update columns (spai.py:229-292): the complex least-squares
  problem over a support I with target t is exactly the real one over the
  columns {2k, 2k+1 : k in I} of R(A) with target R(t); the real level-0
  support of column 2j is that set for I = rows(A(:, j)) U {j}.  Solving
  every real column gives R(M) itself (column 2j+1 is R(i M(:, j)));
  exported factors take the even columns.  Level-1 augmentation ranks by
  the complex moduli |A| (spai.py:212) on the complex structure and is
  realified afterwards.
* Block GCRO (krylov.py:105-275): span_C{B, AB, ...} realified is the real
  block Krylov space of [R(b_0), R(i b_0), R(b_1), R(i b_1), ...]; the real
  solver on that 2s-column block, with the restart length and outer-space
  dimension doubled (they count real columns), takes the same block steps
  and decisions (deflation ranks pair up, partner columns have equal
  residuals, the fold keeps pairs) -- iterations equal, X = the even
  columns.

Every kernel runs in FP64 on the device; the host only canonicalises the
user's scipy input (as_csr semantics) and converts results back.
"""

import numpy as np
import scipy.sparse as sp
import torch

from . import _abi
from .device import DeviceCSR, DevicePattern, Structure, _dev, f64, i32


def is_complex_host(A):
    """scipy / numpy input with a non-zero imaginary part."""
    if sp.issparse(A):
        return np.iscomplexobj(A.data) and A.nnz > 0 and bool(np.any(A.data.imag != 0))
    if isinstance(A, np.ndarray) or np.isscalar(A) or isinstance(A, (list, tuple)):
        arr = np.asarray(A)
        return np.iscomplexobj(arr) and bool(np.any(arr.imag != 0))
    return False


def is_complex(A):
    return isinstance(A, DeviceCSR) and A.cplx or (not isinstance(A, DeviceCSR)
                                                   and is_complex_host(A))


def canon_complex(A):
    """as_csr (sparsecore.py:26-44): complex128, duplicates summed, sorted,
    explicit zeros removed."""
    M = sp.csr_matrix(A, dtype=np.complex128, copy=True)
    M.sum_duplicates()
    M.sort_indices()
    M.eliminate_zeros()
    return M


def realify_csr(A):
    """Complex scipy matrix -> device real form R(A) (a DeviceCSR flagged
    ``cplx``).  The diagonal enters the structure (explicit zero blocks when
    absent) so the real level-0 supports are the complex ones realified."""
    M = canon_complex(A)
    n, m = M.shape
    if n != m:
        raise ValueError("expected a square matrix, got %s" % (M.shape,))
    coo = M.tocoo()
    rows = np.concatenate([coo.row, np.arange(n)])
    cols = np.concatenate([coo.col, np.arange(n)])
    vals = np.concatenate([coo.data, np.zeros(n, dtype=np.complex128)])
    S = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
    S.sum_duplicates()      # keeps the explicit zero diagonal (no pruning)
    S.sort_indices()
    rp, ci = i32(S.indptr), i32(S.indices)
    re, im = f64(S.data.real), f64(S.data.imag)
    nnz = S.nnz
    dev = _dev()
    rp2 = torch.empty(2 * n + 1, dtype=torch.int32, device=dev)
    ci2 = torch.empty(max(4 * nnz, 1), dtype=torch.int32, device=dev)
    v2 = torch.empty(max(4 * nnz, 1), dtype=torch.float64, device=dev)
    _abi.call("pmp_realify", n, _abi.ptr(rp), _abi.ptr(ci), _abi.ptr(re), _abi.ptr(im),
              _abi.ptr(rp2), _abi.ptr(ci2), _abi.ptr(v2), _abi.stream())
    herm = (M - M.conj().T).nnz == 0 or not np.any((M - M.conj().T).data)
    Pn = sp.csr_matrix((np.ones(S.nnz), S.indices, S.indptr), shape=S.shape)
    sym_pat = (Pn - Pn.T).nnz == 0
    st = Structure(2 * n, rp2, ci2[:4 * nnz], symmetric_pattern=bool(sym_pat) or None)
    R = DeviceCSR(st, v2[:4 * nnz], symmetric=bool(herm))   # R(A)^T = R(A^H)
    R.cplx = True
    R.cplx_struct = Structure(n, rp, ci)
    R.cplx_re, R.cplx_im = re, im
    return R


def to_complex_scipy(R, drop_zeros=True):
    """Real form (device) -> complex scipy CSR: A(r, c) = R(2r, 2c) + i R(2r+1, 2c)."""
    M = R.to_scipy_real(drop_zeros=False).tocsr()
    n = M.shape[0] // 2
    re = M[0::2, :][:, 0::2]
    im = M[1::2, :][:, 0::2]
    out = (re.astype(np.complex128) + 1j * im).tocsr()
    out.sum_duplicates()
    out.sort_indices()
    if drop_zeros:
        out.eliminate_zeros()
    assert out.shape == (n, n)
    return out


def block_to_real(V, pairs=True):
    """n x s complex block (numpy or CUDA complex tensor) -> device real
    2n x 2s block [R(v_0), R(i v_0), ...] (pairs) -- or 2n x s [R(v_c)]."""
    if torch.is_tensor(V):
        Vc = V.to(device=_dev())
        if not torch.is_complex(Vc):
            Vc = Vc.to(torch.complex128)
        arr_re = Vc.real.to(torch.float64).contiguous()
        arr_im = Vc.imag.to(torch.float64).contiguous()
    else:
        a = np.asarray(V, dtype=np.complex128)
        arr_re, arr_im = f64(np.ascontiguousarray(a.real)), f64(np.ascontiguousarray(a.imag))
    if arr_re.dim() == 1:
        arr_re, arr_im = arr_re[:, None], arr_im[:, None]
    n, s = arr_re.shape
    Y = torch.empty(2 * n, 2 * s, dtype=torch.float64, device=_dev())
    _abi.call("pmp_realify_block", n, s, _abi.ptr(arr_re), _abi.ptr(arr_im), s, _abi.ptr(Y),
              2 * s, _abi.stream())
    if pairs:
        return Y
    out = torch.empty(2 * n, s, dtype=torch.float64, device=_dev())
    # the R(v_c) columns only: strided copy through the library
    _abi.call("pmp_copy_cols", 2 * n, s, _abi.ptr(Y), 2 * s,
              _abi.ptr(torch.arange(0, 2 * s, 2, dtype=torch.int32, device=_dev())),
              _abi.ptr(out), s, None, _abi.stream())
    return out


def block_from_real(Y, stride):
    """2n x k real block -> n x s complex CUDA tensor from columns 0, stride, ..."""
    n2, k = Y.shape
    n = n2 // 2
    s = (k + stride - 1) // stride
    re = torch.empty(n, s, dtype=torch.float64, device=_dev())
    im = torch.empty(n, s, dtype=torch.float64, device=_dev())
    Yc = Y.contiguous()
    _abi.call("pmp_derealify_block", n, s, _abi.ptr(Yc), k, stride, _abi.ptr(re), _abi.ptr(im),
              s, _abi.stream())
    return torch.complex(re, im)


def modulus_csr(R):
    """|A| on the complex structure (level-1 weights, spai.py:212)."""
    st = R.cplx_struct
    out = torch.empty(max(st.nnz, 1), dtype=torch.float64, device=_dev())[:st.nnz]
    _abi.call("pmp_modulus", st.nnz, _abi.ptr(R.cplx_re), _abi.ptr(R.cplx_im), _abi.ptr(out),
              _abi.stream())
    M = DeviceCSR(st, out, symmetric=False)
    return M


def realify_pattern(pat):
    """Complex supports (n columns) -> real-form supports (2n columns)."""
    n = pat.n
    optr = torch.empty(2 * n + 1, dtype=torch.int32, device=_dev())
    oidx = torch.empty(max(4 * pat.nnz, 1), dtype=torch.int32, device=_dev())
    _abi.call("pmp_pattern_realify", n, _abi.ptr(pat.iptr), _abi.ptr(pat.iidx), _abi.ptr(optr),
              _abi.ptr(oidx), _abi.stream())
    return DevicePattern(2 * n, optr, oidx, 4 * pat.nnz)
