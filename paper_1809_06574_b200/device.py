"""Device-resident sparse matrices, patterns and scratch for the B200 path.

HBM layout:
  * a matrix is CSR: ``rowptr`` int32[n+1], ``colidx`` int32[nnz] (sorted
    within rows), ``vals`` float64[nnz];
  * its column view (needed by the per-column SPAI/update solves,
    ``A.tocsc()`` at spai.py:320) is either the CSR itself -- when the
    matrix is known to be exactly symmetric, as every MDK system assembled
    from symmetric terms is -- or a transposed copy obtained by permuting
    ``vals`` through a permutation cached on the shared structure;
  * matrices assembled from one model share one :class:`Structure` (union
    pattern), so patterns, transposes and least-squares plans are computed
    once per sequence and reused by every (sigma, p) system.

PyTorch provides the allocations and the current stream only; all compute
goes through libpmorb200 (``_abi``).
"""

import itertools

import numpy as np
import scipy.sparse as sp
import torch

from . import _abi

_ids = itertools.count(1)


_CUDA_OK = False


def _dev():
    # (the availability probe goes through NVML on every call -- ~5 us, a
    # few hundred times per sequence step -- so it is done once)
    global _CUDA_OK
    if not _CUDA_OK:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1809_06574_b200 needs a CUDA device (B200); no CPU fallback")
        _CUDA_OK = True
    return torch.device("cuda", torch.cuda.current_device())


def i32(a, device=None):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=device or _dev())


def f64(a, device=None):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=device or _dev())


class Scratch:
    """Grow-only named scratch buffers (the library never allocates).
    Buffers requested with ``zero=True`` are zero-filled once at allocation
    (the reduction tickets of pmp_gram / pmp_tsqr_r rely on it and reset
    themselves after every use)."""

    def __init__(self):
        self._bufs = {}

    def get(self, name, nbytes, zero=False):
        nbytes = max(int(nbytes), 16)
        b = self._bufs.get(name)
        if b is None or b.numel() < nbytes:
            cap = max(nbytes, 2 * (b.numel() if b is not None else 0))
            b = (torch.zeros if zero else torch.empty)(cap, dtype=torch.uint8, device=_dev())
            self._bufs[name] = b
        return b


_scratch = {}


def scratch():
    """Scratch of the current (device, stream): concurrent workers on their
    own streams never share a workspace."""
    key = (torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream)
    s = _scratch.get(key)
    if s is None:
        s = _scratch[key] = Scratch()
    return s


class Structure:
    """Sparsity structure shared by every matrix assembled from one model."""

    def __init__(self, n, rowptr, colidx, symmetric_pattern=None):
        self.key = next(_ids)
        self.n = int(n)
        self.rowptr = rowptr
        self.colidx = colidx
        self.nnz = int(colidx.numel())
        self._csc = None
        self._rowid = None
        self.cache = {}
        self.symmetric_pattern = symmetric_pattern

    def rowid(self):
        """COO row index of every stored entry (for diagonal terms)."""
        if self._rowid is None:
            rp = self.rowptr.cpu().numpy()
            self._rowid = i32(np.repeat(np.arange(self.n, dtype=np.int32), np.diff(rp)))
        return self._rowid

    def csc(self):
        """(colptr, rowidx, perm) of the transposed structure; perm maps a
        CSR slot to its CSC slot."""
        if self._csc is None:
            n, nnz = self.n, self.nnz
            colptr = torch.empty(n + 1, dtype=torch.int32, device=_dev())
            rowidx = torch.empty(max(nnz, 1), dtype=torch.int32, device=_dev())
            perm = torch.empty(max(nnz, 1), dtype=torch.int32, device=_dev())
            ws = scratch().get("transpose", _abi.lib().pmp_transpose_workspace(n, nnz))
            _abi.call("pmp_transpose", n, nnz, _abi.ptr(self.rowptr), _abi.ptr(self.colidx), None,
                      0, _abi.ptr(colptr), _abi.ptr(rowidx), None, _abi.ptr(perm), _abi.ptr(ws),
                      ws.numel(), _abi.stream())
            self._csc = (colptr, rowidx[:nnz], perm[:nnz])
        return self._csc


class DeviceCSR:
    """n x n CSR matrix in HBM (float64 values, int32 indices).

    ``symmetric`` asserts A == A^T bitwise, so the CSR arrays double as the
    CSC view.
    """

    def __init__(self, structure, vals, symmetric=False):
        self.structure = structure
        self.vals = vals
        self.symmetric = bool(symmetric)
        self._csc_vals = None
        # complex matrices are stored as their real form R(A) (cplx.py):
        # shape / n are then the REAL dimensions (2n), complex_n the complex
        self.cplx = False

    # -- construction / export --------------------------------------------
    @classmethod
    def from_scipy(cls, A, structure=None, check_symmetric=True):
        if isinstance(A, DeviceCSR):
            return A
        A = sp.csr_matrix(A)
        if np.iscomplexobj(A.data):
            if A.nnz and np.abs(A.data.imag).max() != 0:
                raise NotImplementedError("complex-valued systems are not supported by the B200 "
                                          "path yet (real FP64 only)")
            A = sp.csr_matrix((A.data.real, A.indices, A.indptr), shape=A.shape)
        A = sp.csr_matrix(A, dtype=np.float64, copy=True)
        A.sum_duplicates()
        A.sort_indices()
        A.eliminate_zeros()
        if A.shape[0] != A.shape[1]:
            raise ValueError("expected a square matrix, got %s" % (A.shape,))
        sym = False
        if check_symmetric:
            D = A - A.T
            sym = D.nnz == 0 or not np.any(D.data)
        if structure is None:
            structure = Structure(A.shape[0], i32(A.indptr), i32(A.indices),
                                  symmetric_pattern=sym or None)
        return cls(structure, f64(A.data), symmetric=sym)

    @property
    def complex_n(self):
        return self.structure.n // 2 if self.cplx else self.structure.n

    def to_scipy(self, drop_zeros=True):
        """Host CSR (complex128 for a complex matrix's real form)."""
        if self.cplx:
            from .cplx import to_complex_scipy
            return to_complex_scipy(self, drop_zeros)
        return self.to_scipy_real(drop_zeros)

    def to_scipy_real(self, drop_zeros=True):
        s = self.structure
        M = sp.csr_matrix((self.vals.cpu().numpy(), s.colidx.cpu().numpy(), s.rowptr.cpu().numpy()),
                          shape=(s.n, s.n))
        if drop_zeros:
            M.eliminate_zeros()
        return M

    @property
    def shape(self):
        return (self.structure.n, self.structure.n)

    @property
    def n(self):
        return self.structure.n

    @property
    def nnz(self):
        return self.structure.nnz

    def csc(self):
        """(colptr, rowidx, vals) column view."""
        s = self.structure
        if self.symmetric:
            return s.rowptr, s.colidx, self.vals
        colptr, rowidx, perm = s.csc()
        if self._csc_vals is None:
            cv = torch.empty_like(self.vals)
            _abi.call("pmp_permute", s.nnz, _abi.ptr(perm), _abi.ptr(self.vals), _abi.ptr(cv),
                      _abi.stream())
            self._csc_vals = cv
        return colptr, rowidx, self._csc_vals

    def csc_structure(self):
        s = self.structure
        if self.symmetric or s.symmetric_pattern:
            return s.rowptr, s.colidx
        return s.csc()[:2]

    def spmm(self, X, ldx, s, Y, ldy, alpha=1.0, beta=0.0, Y0=None, ldy0=0):
        """Y = alpha A X + beta Y0 on raw device pointers (row-major blocks)."""
        st = self.structure
        _abi.call("pmp_spmm", st.n, _abi.ptr(st.rowptr), _abi.ptr(st.colidx), _abi.ptr(self.vals),
                  int(s), X, int(ldx), float(alpha), float(beta), Y0, int(ldy0), Y, int(ldy),
                  _abi.stream())


class DevicePattern:
    """Per-column supports I_j in CSC-like form (iptr int32[n+1], iidx)."""

    def __init__(self, n, iptr, iidx, nnz=None):
        self.key = next(_ids)
        self.n = int(n)
        self.iptr = iptr
        self.iidx = iidx
        self.nnz = int(iidx.numel()) if nnz is None else int(nnz)
        self.cache = {}

    def columns(self):
        ptr = self.iptr.cpu().numpy()
        idx = self.iidx.cpu().numpy()
        return [idx[ptr[j]:ptr[j + 1]].astype(np.int64) for j in range(self.n)]

    @classmethod
    def from_columns(cls, n, cols):
        ptr = np.zeros(n + 1, dtype=np.int64)
        ptr[1:] = np.cumsum([len(c) for c in cols])
        idx = np.concatenate([np.asarray(c, dtype=np.int64) for c in cols]) if cols else np.zeros(0)
        return cls(n, i32(ptr), i32(idx) if idx.size else torch.zeros(1, dtype=torch.int32,
                                                                         device=_dev()),
                   nnz=int(ptr[-1]))


def level0_pattern(structure_or_csr):
    """Level-0 SPAI pattern I_j = rows(A(:, j)) U {j} (spai.py:182-207),
    cached on the structure."""
    A = structure_or_csr
    st = A.structure if isinstance(A, DeviceCSR) else A
    pat = st.cache.get("pattern_l0")
    if pat is not None:
        return pat
    if isinstance(A, DeviceCSR):
        colptr, rowidx = A.csc_structure()
    else:
        colptr, rowidx = (st.rowptr, st.colidx) if st.symmetric_pattern else st.csc()[:2]
    n = st.n
    iptr = torch.empty(n + 1, dtype=torch.int32, device=_dev())
    ws = scratch().get("pattern", _abi.lib().pmp_pattern_l0_workspace(n))
    _abi.call("pmp_pattern_l0_ptr", n, _abi.ptr(colptr), _abi.ptr(rowidx), _abi.ptr(iptr),
              _abi.ptr(ws), ws.numel(), _abi.stream())
    nnz = int(iptr[n].item())
    iidx = torch.empty(max(nnz, 1), dtype=torch.int32, device=_dev())
    _abi.call("pmp_pattern_l0", n, _abi.ptr(colptr), _abi.ptr(rowidx), _abi.ptr(iptr),
              _abi.ptr(iidx), _abi.ptr(ws), ws.numel(), _abi.stream())
    pat = DevicePattern(n, iptr, iidx, nnz)
    st.cache["pattern_l0"] = pat
    return pat
