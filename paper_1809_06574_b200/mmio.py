"""Matrix Market interchange with the reference (sparsecore.py:243-285).

Files are written the way the reference's ``write_matrix_market`` writes
them: canonical CSR (``as_csr``: duplicates summed, indices sorted, explicit
zeros removed) printed by ``scipy.io.mmwrite(field="complex", precision=17,
symmetry="general")``, so both sides read each other's files bit-exactly.
Real systems are written with +0 imaginary parts (the reference's complex
arithmetic sometimes prints -0; the values read back are the same).  Reading
accepts any Matrix Market file the reference accepts and returns float64
data when every imaginary part is zero, complex128 otherwise (complex
systems run through their real form on the device, cplx.py).

Host-side only: persistence is file I/O around the device path.
"""

import numpy as np
import scipy.io
import scipy.sparse as sp

MM_PRECISION = 17  # sparsecore.py:247 -- bit-exact text round trips


def canonical_csr(A):
    """The reference's ``as_csr`` (sparsecore.py:26-44): CSR, duplicates
    summed, sorted indices, no explicit zeros; float64 when the data is real
    (or complex with all-zero imaginary parts), complex128 otherwise."""
    A = sp.csr_matrix(A)
    cx = np.iscomplexobj(A.data) and A.nnz and np.abs(A.data.imag).max() != 0
    if np.iscomplexobj(A.data) and not cx:
        A = sp.csr_matrix((A.data.real, A.indices, A.indptr), shape=A.shape)
    A = sp.csr_matrix(A, dtype=np.complex128 if cx else np.float64, copy=True)
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
    """sparsecore.py:281-285; float64 when every imaginary part is zero,
    complex128 otherwise."""
    M = scipy.io.mmread(str(path), spmatrix=False)
    if sp.issparse(M):
        M = M.toarray()
    M = np.atleast_2d(np.asarray(M))
    if np.iscomplexobj(M):
        if np.abs(M.imag).max(initial=0.0) != 0:
            return np.ascontiguousarray(M, dtype=np.complex128)
        M = M.real
    return np.ascontiguousarray(M, dtype=np.float64)
