"""Matrix Market interchange with the reference (sparsecore.py:243-285).

Files are written the way the reference's ``write_matrix_market`` writes
them: canonical CSR (``as_csr``: duplicates summed, indices sorted, explicit
zeros removed) printed by ``scipy.io.mmwrite(field="complex", precision=17,
symmetry="general")``, so both sides read each other's files bit-exactly.
The B200 path computes in real FP64 and writes +0 imaginary parts (the
reference's complex arithmetic sometimes prints -0; the values read back
are the same).  Reading accepts
any Matrix Market file the reference accepts; complex data with a non-zero
imaginary part raises ``NotImplementedError`` (complex128 is the first
"next" row of SURVEY.md 8(f)).

Host-side only: persistence is file I/O around the device path.
"""

import numpy as np
import scipy.io
import scipy.sparse as sp

MM_PRECISION = 17  # sparsecore.py:247 -- bit-exact text round trips


def canonical_csr(A):
    """The reference's ``as_csr`` (sparsecore.py:26-44) restricted to real
    data: float64 CSR, duplicates summed, sorted indices, no explicit zeros."""
    A = sp.csr_matrix(A)
    if np.iscomplexobj(A.data):
        if A.nnz and np.abs(A.data.imag).max() != 0:
            raise NotImplementedError("complex-valued matrices are not supported by the B200 "
                                      "path yet (real FP64 only)")
        A = sp.csr_matrix((A.data.real, A.indices, A.indptr), shape=A.shape)
    A = sp.csr_matrix(A, dtype=np.float64, copy=True)
    A.sum_duplicates()
    A.sort_indices()
    A.eliminate_zeros()
    return A


def write_matrix_market(A, path):
    """sparsecore.py:250-259: coordinate format, complex field, 17 digits."""
    A = canonical_csr(A)
    Ac = sp.csr_matrix((A.data.astype(np.complex128), A.indices, A.indptr), shape=A.shape)
    scipy.io.mmwrite(str(path), Ac.tocoo(), field="complex", precision=MM_PRECISION,
                     symmetry="general")


def read_matrix_market(path):
    """sparsecore.py:262-272: symmetric / skew / hermitian files expanded to
    general storage; malformed files raise ValueError (from the parser)."""
    M = scipy.io.mmread(str(path), spmatrix=False)
    if not sp.issparse(M):
        M = sp.csr_matrix(np.atleast_2d(M))
    return canonical_csr(M)


def write_dense_matrix_market(X, path):
    """sparsecore.py:275-278: array format, complex field, 17 digits."""
    X = np.asarray(X)
    if X.ndim == 1:
        X = X[:, None]
    scipy.io.mmwrite(str(path), X.astype(np.complex128), field="complex",
                     precision=MM_PRECISION)


def read_dense_matrix_market(path):
    """sparsecore.py:281-285, returned as a real float64 block."""
    M = scipy.io.mmread(str(path), spmatrix=False)
    if sp.issparse(M):
        M = M.toarray()
    M = np.atleast_2d(np.asarray(M))
    if np.iscomplexobj(M):
        if np.abs(M.imag).max(initial=0.0) != 0:
            raise NotImplementedError("complex-valued blocks are not supported by the B200 "
                                      "path yet (real FP64 only)")
        M = M.real
    return np.ascontiguousarray(M, dtype=np.float64)
