"""Loader for the committed golden fixtures (tests/golden/*.npz), produced
by tests/golden/make_golden.py from the real reference."""

import os

import numpy as np
import scipy.sparse as sp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["rand40", "tridiag9", "degenerate2", "c1s24", "c2s8", "c3s6", "c5n500"]
WORKLOAD_CASES = {"c1s24": (1, 24), "c2s8": (2, 8), "c3s6": (3, 6), "c5n500": (5, 500)}


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def csr(g, prefix):
    shape = tuple(int(v) for v in g[prefix + "_shape"])
    return sp.csr_matrix((g[prefix + "_data"], g[prefix + "_indices"], g[prefix + "_indptr"]),
                         shape=shape)


def pattern(g, prefix):
    ptr, idx = g[prefix + "_ptr"], g[prefix + "_idx"]
    return [idx[ptr[j]:ptr[j + 1]] for j in range(ptr.size - 1)]


def has(g, prefix):
    return any(k.startswith(prefix + "_") for k in g)


def compare_factor(M, ref, tol=1e-10, zero_tol=1e-14):
    """stored structure equal modulo entries that one side
    rounds to exactly 0.0 (as_csr drops them); values within ``tol``
    relative Frobenius.  Returns (relative error, #one-sided entries)."""
    M = sp.csc_matrix(M)
    ref = sp.csc_matrix(ref)
    assert M.shape == ref.shape
    D = (M - ref).tocsc()
    err = sp.linalg.norm(D) / max(sp.linalg.norm(ref), 1e-300)
    assert err <= tol, err
    onesided = 0
    colnorm = np.sqrt(np.asarray(ref.multiply(ref).sum(axis=0)).ravel())
    for j in range(M.shape[1]):
        a = set(M.indices[M.indptr[j]:M.indptr[j + 1]].tolist())
        b = set(ref.indices[ref.indptr[j]:ref.indptr[j + 1]].tolist())
        for r in a ^ b:
            v = M[r, j] if r in a else ref[r, j]
            assert abs(v) <= zero_tol * max(colnorm[j], 1e-300), (j, r, v)
            onesided += 1
    return err, onesided
