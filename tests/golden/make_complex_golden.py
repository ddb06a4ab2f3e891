"""Complex128 goldens from the REAL reference ``pmorprec``
(importable only in the build container, /root/reference/pkg/src):

* ``cx_rand40``: the reference unit tests' complex generator
  (pkg/tests/conftest.py:13-24: random_sparse(..., complex_values=True),
  well_conditioned shift 4) -- SPAI at levels 0 / 1, update_first /
  update_second, block GCRO with a complex right-hand side block;
* ``cx_gyro``: the gyroscope analog family (zoo.py:154-186) at a small
  n -- its four expansion points have imaginary shifts, so every assembled
  system is genuinely complex -- assembled matrices, a SPAI at point 1,
  update_first at point 2 and the block solve there;
* ``cx_mdk``: a real second-order model (the c1 stencil at n = 144)
  assembled at an imaginary shift s = 2j and a complex parameter.

    OPENBLAS_NUM_THREADS=1 PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_complex_golden.py
"""

import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import pmorprec as ref                                   # noqa: E402
from pmorprec.spai import SpaiConfig                     # noqa: E402
from pmorprec.update import UpdateConfig                 # noqa: E402
from pmorprec.krylov import SolverConfig                 # noqa: E402
from pmorprec.rpmor import SecondOrderModel              # noqa: E402
from pmorprec import zoo                                 # noqa: E402

from paper_1809_06574_b200.workloads import make_config  # noqa: E402


def random_sparse(n, density=0.1, seed=0, shift=0.0):
    """pkg/tests/conftest.py:13-24 with complex_values=True."""
    rs = np.random.RandomState(seed)
    A = sp.random(n, n, density=density, random_state=rs, format="csr")
    A = A.astype(np.complex128) + 1j * sp.random(
        n, n, density=density, random_state=np.random.RandomState(seed + 1), format="csr")
    if shift:
        A = A + shift * sp.identity(n)
    return ref.as_csr(A)


def csr(prefix, M, out):
    M = ref.as_csr(M)
    out[prefix + "_indptr"] = M.indptr.astype(np.int64)
    out[prefix + "_indices"] = M.indices.astype(np.int64)
    out[prefix + "_data"] = M.data.copy()
    out[prefix + "_shape"] = np.array(M.shape)


def stats(prefix, st, out):
    out[prefix + "_resid"] = np.asarray(st.residuals, dtype=float)
    out[prefix + "_aug"] = np.array(st.augmented_columns)
    out[prefix + "_def"] = np.array(st.rank_deficient_columns)


def solve(prefix, A, B, P, out, cfg=None):
    X, rep = ref.block_gcro_solve(A, B, P=P, cfg=cfg or SolverConfig(tol=1e-8))
    out[prefix + "_X"] = X
    out[prefix + "_iters"] = np.array(rep.iterations)
    out[prefix + "_conv"] = np.array(rep.converged)
    out[prefix + "_hist"] = np.array([np.asarray(h, dtype=float) for h in rep.residual_history])
    out[prefix + "_matvec"] = np.array(rep.matvec_count)
    out[prefix + "_papply"] = np.array(rep.precond_apply_count)


def rand_case():
    out = {}
    A = random_sparse(40, density=0.08, seed=3, shift=4.0)
    E = random_sparse(40, density=0.05, seed=11)
    A2 = ref.as_csr(A + 1e-2 * E)
    A3 = ref.as_csr(A + 2e-2 * E)
    csr("A1", A, out)
    csr("A2", A2, out)
    csr("A3", A3, out)
    B = (np.random.default_rng(5).standard_normal((40, 3))
         + 1j * np.random.default_rng(6).standard_normal((40, 3)))
    out["B"] = B
    for lvl, fill in ((0, 80), (1, 12)):
        P, st = ref.spai_build(A, SpaiConfig(pattern_level=lvl, max_fill_per_column=fill))
        csr("P%d" % lvl, P.matrix, out)
        stats("P%d" % lvl, st, out)
        Q, stq = ref.update_first(A, A2, P, UpdateConfig(pattern_level=lvl,
                                                          max_fill_per_column=fill))
        csr("Q%d" % lvl, Q.q, out)
        stats("Q%d" % lvl, stq, out)
        solve("s%d" % lvl, A2, B, Q, out)
        # second approach: Q2 against A2 on top of the first update
        Q2, st2 = ref.update_second(A2, A3, Q, UpdateConfig(approach="second", pattern_level=lvl,
                                                             max_fill_per_column=fill))
        csr("R%d" % lvl, Q2.q, out)
        stats("R%d" % lvl, st2, out)
        solve("t%d" % lvl, A3, B, Q2, out)
    solve("nop", A2, B, None, out)
    np.savez_compressed(os.path.join(HERE, "cx_rand40.npz"), **out)
    print("wrote cx_rand40")


def gyro_case():
    out = {}
    spec = zoo.GyroAnalogSpec(n=300, seed=7)
    model, points = zoo.gen_gyro_analog(spec)
    fam = model.family
    for j, T in enumerate(fam.terms):
        csr("T%d" % j, T, out)
    out["rhs"] = np.asarray(fam.rhs)
    for i, pt in enumerate(points):
        out["pt%d" % i] = np.asarray(pt.values, dtype=np.complex128)
        csr("A%d" % i, fam.evaluate(pt), out)
    A1, A2 = fam.evaluate(points[0]), fam.evaluate(points[1])
    P, st = ref.spai_build(A1, SpaiConfig(pattern_level=0))
    csr("P0", P.matrix, out)
    stats("P0", st, out)
    Q, stq = ref.update_first(A1, A2, P, UpdateConfig(pattern_level=0))
    csr("Q0", Q.q, out)
    stats("Q0", stq, out)
    B = np.asarray(fam.rhs, dtype=np.complex128)
    solve("s1", A1, B, P, out)
    solve("s2", A2, B, Q, out)
    np.savez_compressed(os.path.join(HERE, "cx_gyro.npz"), **out)
    print("wrote cx_gyro", A1.shape, A1.nnz)


def mdk_case():
    out = {}
    W = make_config(1, scale=12)
    m = SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms, rhs=W.rhs)
    pts = [(2.0j, [0.5]), (0.3 + 1.5j, [0.75 - 0.25j]), (1.0, [0.5j])]
    for i, (s, p) in enumerate(pts):
        csr("A%d" % i, m.assemble(s, p), out)
        out["s%d" % i] = np.array(complex(s))
        out["p%d" % i] = np.asarray(p, dtype=np.complex128)
    np.savez_compressed(os.path.join(HERE, "cx_mdk.npz"), **out)
    print("wrote cx_mdk")


def affine_case():
    """Genuinely complex terms x complex coefficients: pins the rounding of
    numpy's complex multiply (scalar * data in affine.py:129, data * scalar
    through scipy in rpmor.py:47 / :104)."""
    from pmorprec.affine import AffineFamily
    out = {}
    terms = [random_sparse(36, density=0.12, seed=31 + 2 * j, shift=3.0 if j == 0 else 0.0)
             for j in range(4)]
    for j, T in enumerate(terms):
        csr("T%d" % j, T, out)
    fam = AffineFamily(terms)
    pts = [np.array([0.5 - 0.25j, 1.5 + 2.0j, -0.3 + 0.7j]),
           np.array([1.0 / 3.0 + 1j / 7.0, 0.0, 2.5j])]
    for i, pt in enumerate(pts):
        out["pt%d" % i] = pt
        csr("A%d" % i, fam.evaluate(pt), out)
    # complex terms through the second-order form as well
    m = SecondOrderModel.from_mdk([terms[1], terms[2]], [terms[3]], [terms[0], terms[2]])
    mp = [(0.3 + 1.5j, [0.75 - 0.25j]), (1.25, [0.5j])]
    for i, (s, p) in enumerate(mp):
        out["ms%d" % i] = np.array(complex(s))
        out["mp%d" % i] = np.asarray(p, dtype=np.complex128)
        csr("M%d" % i, m.assemble(s, p), out)
    np.savez_compressed(os.path.join(HERE, "cx_affine.npz"), **out)
    print("wrote cx_affine")


if __name__ == "__main__":
    rand_case()
    gyro_case()
    mdk_case()
    affine_case()
