"""Complex128 on the device against the REAL reference
(tests/golden/cx_*.npz, tests/golden/make_complex_golden.py) and the
reference's own unit-test assertions re-run on complex inputs
(pkg/tests/test_spai.py / test_update.py / test_krylov.py, whose generator
defaults to complex values, conftest.py:13-24).

Bars: assembly bit-exact (real terms, complex shifts /
parameters); supports bit-exact; factors <= 1e-10 relative Frobenius;
residuals <= 1e-12; solves: iterations +-2, true residual <= 1e-8.
"""

import numpy as np
import pytest
import scipy.sparse as sp

import goldens as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1809_06574_b200 as pm
    return pm


def ccsr(g, prefix):
    shape = tuple(int(v) for v in g[prefix + "_shape"])
    return sp.csr_matrix((g[prefix + "_data"], g[prefix + "_indices"], g[prefix + "_indptr"]),
                         shape=shape)


def random_sparse(n, density=0.1, seed=0, shift=0.0):
    """pkg/tests/conftest.py:13-24 (complex_values=True)."""
    rs = np.random.RandomState(seed)
    A = sp.random(n, n, density=density, random_state=rs, format="csr")
    A = A.astype(np.complex128) + 1j * sp.random(
        n, n, density=density, random_state=np.random.RandomState(seed + 1), format="csr")
    if shift:
        A = A + shift * sp.identity(n)
    A = sp.csr_matrix(A)
    A.eliminate_zeros()
    return A


def fro_rel(M, R):
    return sp.linalg.norm(sp.csr_matrix(M) - R) / sp.linalg.norm(R)


def same_supports(M, R):
    M, R = sp.csc_matrix(M), sp.csc_matrix(R)
    M.eliminate_zeros()
    R.eliminate_zeros()
    return (np.array_equal(M.indptr, R.indptr) and np.array_equal(M.indices, R.indices))


def check_solve(A, B, X, rep, g, prefix, tol=1e-8):
    rel = np.linalg.norm(B - A @ X, axis=0) / np.linalg.norm(B, axis=0)
    assert rep.converged == bool(g[prefix + "_conv"])
    assert np.all(rel <= tol), rel
    assert abs(rep.iterations - int(g[prefix + "_iters"])) <= 2, (rep.iterations,
                                                                 int(g[prefix + "_iters"]))
    Xr = g[prefix + "_X"]
    assert np.linalg.norm(X - Xr) / np.linalg.norm(Xr) <= 1e-6


@pytest.mark.parametrize("lvl", [0, 1])
def test_complex_spai_update_solve_vs_reference(pm, lvl):
    g = G.load("cx_rand40")
    A1, A2, A3, B = ccsr(g, "A1"), ccsr(g, "A2"), ccsr(g, "A3"), g["B"]
    fill = 80 if lvl == 0 else 12
    P, st = pm.spai_build(A1, pm.SpaiConfig(pattern_level=lvl, max_fill_per_column=fill))
    Pm = P.matrix.to_scipy()
    Pr = ccsr(g, "P%d" % lvl)
    assert Pm.dtype == np.complex128
    assert same_supports(Pm, Pr)
    assert fro_rel(Pm, Pr) <= 1e-10
    assert np.max(np.abs(st.residuals - g["P%d_resid" % lvl])) <= 1e-12
    assert st.augmented_columns == int(g["P%d_aug" % lvl])
    assert st.rank_deficient_columns == int(g["P%d_def" % lvl])
    ucfg = pm.UpdateConfig(pattern_level=lvl, max_fill_per_column=fill)
    Q, stq = pm.update_first(A1, A2, P, ucfg)
    assert fro_rel(Q.q.to_scipy(), ccsr(g, "Q%d" % lvl)) <= 1e-10
    assert np.max(np.abs(stq.residuals - g["Q%d_resid" % lvl])) <= 1e-12
    assert stq.augmented_columns == int(g["Q%d_aug" % lvl])
    X, rep = pm.block_gcro_solve(A2, B, P=Q, cfg=pm.SolverConfig(tol=1e-8))
    assert X.dtype == np.complex128
    check_solve(A2, B, X, rep, g, "s%d" % lvl)
    # the second approach: chain of depth 3
    R, str_ = pm.update_second(A2, A3, Q, pm.UpdateConfig(approach="second", pattern_level=lvl,
                                                          max_fill_per_column=fill))
    assert R.depth == 3
    assert fro_rel(R.q.to_scipy(), ccsr(g, "R%d" % lvl)) <= 1e-10
    X3, rep3 = pm.block_gcro_solve(A3, B, P=R, cfg=pm.SolverConfig(tol=1e-8))
    check_solve(A3, B, X3, rep3, g, "t%d" % lvl)


def test_complex_unpreconditioned_solve(pm):
    g = G.load("cx_rand40")
    A2, B = ccsr(g, "A2"), g["B"]
    X, rep = pm.block_gcro_solve(A2, B, cfg=pm.SolverConfig(tol=1e-8))
    check_solve(A2, B, X, rep, g, "nop")
    assert rep.matvec_count == int(g["nop_matvec"])


def test_gyroscope_family_assembly_and_solve(pm):
    """The paper's own workload shape: the gyroscope analog (imaginary
    shifts, zoo.py:154-186) -- affine assembly bit-exact, SPAI / update /
    solve against the reference."""
    g = G.load("cx_gyro")
    terms = [ccsr(g, "T%d" % j) for j in range(7)]
    fam = pm.AffineFamily(terms, rhs=g["rhs"])
    for i in range(4):
        A = fam.evaluate(g["pt%d" % i])
        Ah = A.to_scipy()
        Ar = ccsr(g, "A%d" % i)
        assert np.array_equal(Ah.indptr, Ar.indptr) and np.array_equal(Ah.indices, Ar.indices)
        assert np.array_equal(Ah.data, Ar.data), i          # bit-exact
    A1, A2 = fam.evaluate(g["pt0"]), fam.evaluate(g["pt1"])
    P, st = pm.spai_build(A1, pm.SpaiConfig(pattern_level=0))
    assert fro_rel(P.matrix.to_scipy(), ccsr(g, "P0")) <= 1e-10
    Q, _ = pm.update_first(A1, A2, P, pm.UpdateConfig(pattern_level=0))
    assert fro_rel(Q.q.to_scipy(), ccsr(g, "Q0")) <= 1e-10
    B = np.asarray(g["rhs"], dtype=np.complex128)
    X1, r1 = pm.block_gcro_solve(A1, B, P=P, cfg=pm.SolverConfig(tol=1e-8))
    check_solve(ccsr(g, "A0"), B, X1, r1, g, "s1")
    X2, r2 = pm.block_gcro_solve(A2, B, P=Q, cfg=pm.SolverConfig(tol=1e-8))
    check_solve(ccsr(g, "A1"), B, X2, r2, g, "s2")


def test_mdk_complex_shift_assembly_bit_exact(pm):
    from paper_1809_06574_b200.workloads import make_config
    g = G.load("cx_mdk")
    W = make_config(1, scale=12)
    m = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                     rhs=W.rhs)
    for i in range(3):
        A = m.assemble(complex(g["s%d" % i]), g["p%d" % i]).to_scipy()
        Ar = ccsr(g, "A%d" % i)
        assert np.array_equal(A.indptr, Ar.indptr) and np.array_equal(A.indices, Ar.indices)
        assert np.array_equal(A.data, Ar.data), i


def test_complex_terms_times_complex_coefficients_bit_exact(pm):
    """numpy's complex multiply is not symmetric in its operands (one product
    of each part is fused): affine.py:129 is scalar * data, scipy's
    scalar * matrix (rpmor.py:47, :104) is data * scalar."""
    g = G.load("cx_affine")
    terms = [ccsr(g, "T%d" % j) for j in range(4)]
    fam = pm.AffineFamily(terms)
    for i in range(2):
        A = fam.evaluate(g["pt%d" % i]).to_scipy()
        Ar = ccsr(g, "A%d" % i)
        assert np.array_equal(A.indptr, Ar.indptr) and np.array_equal(A.indices, Ar.indices)
        assert np.array_equal(A.data, Ar.data), i
    m = pm.SecondOrderModel.from_mdk([terms[1], terms[2]], [terms[3]], [terms[0], terms[2]])
    for i in range(2):
        A = m.assemble(complex(g["ms%d" % i]), g["mp%d" % i]).to_scipy()
        Ar = ccsr(g, "M%d" % i)
        assert np.array_equal(A.indptr, Ar.indptr) and np.array_equal(A.indices, Ar.indices)
        assert np.array_equal(A.data, Ar.data), i


# ---- the reference's unit-test assertions on complex inputs -------------------

def test_spai_column_full_pattern_matches_dense_inverse(pm):
    """test_spai.py:58-63."""
    A = random_sparse(12, density=0.3, seed=2, shift=3.0)
    Ainv = np.linalg.inv(A.toarray())
    for i in (0, 5, 11):
        sup, coef, resid, dfc = pm.spai_column(A, i, np.arange(12))
        assert np.allclose(coef, Ainv[:, i], atol=1e-12)
        assert resid <= 1e-12 and not dfc


def test_full_pattern_build_reproduces_inverse(pm):
    """test_spai.py:100-105."""
    A = random_sparse(15, density=0.3, seed=4, shift=3.0)
    full = [np.arange(15)] * 15
    P, _ = pm.spai_build(A, pattern=full)
    assert np.allclose(P.matrix.to_scipy().toarray(), np.linalg.inv(A.toarray()), atol=1e-10)


def test_update_identity_and_scaled(pm):
    """test_update.py:25-39: Q = I for the same matrix, I / 2 for 2 A."""
    A = random_sparse(30, density=0.1, seed=8, shift=4.0)
    P, _ = pm.spai_build(A, pm.SpaiConfig(pattern_level=0))
    Q, _ = pm.update_first(A, A, P, pm.UpdateConfig(pattern_level=0))
    assert np.allclose(Q.q.to_scipy().toarray(), np.eye(30), atol=1e-10)
    Q2, _ = pm.update_first(A, 2 * A, P, pm.UpdateConfig(pattern_level=0))
    assert np.allclose(Q2.q.to_scipy().toarray(), 0.5 * np.eye(30), atol=1e-10)


def test_krylov_dense_lu_and_block_vs_singles(pm):
    """test_krylov.py:29-36 and :106-119."""
    A = random_sparse(60, density=0.08, seed=13, shift=4.0)
    rng = np.random.default_rng(1)
    B = rng.standard_normal((60, 3)) + 1j * rng.standard_normal((60, 3))
    X, rep = pm.block_gcro_solve(A, B, cfg=pm.SolverConfig(tol=1e-10))
    Xd = np.linalg.solve(A.toarray(), B)
    assert np.linalg.norm(X - Xd) / np.linalg.norm(Xd) <= 1e-8
    its = []
    for c in range(3):
        x, r = pm.gcro_solve(A, B[:, c], cfg=pm.SolverConfig(tol=1e-10))
        assert np.linalg.norm(x - Xd[:, c]) / np.linalg.norm(Xd[:, c]) <= 1e-8
        its.append(r.iterations)
    assert rep.iterations <= max(its)


def test_complex_preconditioner_apply_and_quality(pm):
    A = random_sparse(25, density=0.15, seed=21, shift=4.0)
    P, _ = pm.spai_build(A, pm.SpaiConfig(pattern_level=0))
    Pm = P.matrix.to_scipy()
    V = np.random.default_rng(3).standard_normal((25, 2)) + 1j
    assert np.allclose(P.apply(V), Pm @ V, atol=1e-13)
    q = pm.quality(A, P)
    qr = np.linalg.norm(np.eye(25) - (A @ Pm).toarray())
    assert abs(q - qr) <= 1e-10 * max(qr, 1.0)


def test_complex_preconditioner_save_load_round_trip(pm, tmp_path):
    """spai.py:103-128 on a complex chain: the saved Matrix Market factors
    (complex field, 17 digits) load back onto the device and apply the same."""
    A = random_sparse(30, density=0.12, seed=41, shift=4.0)
    A2 = sp.csr_matrix(A + 1e-2 * random_sparse(30, density=0.05, seed=43))
    P, _ = pm.spai_build(A, pm.SpaiConfig(pattern_level=0))
    Q, _ = pm.update_first(A, A2, P, pm.UpdateConfig(pattern_level=0))
    Q.save(tmp_path / "chain")
    L = pm.Preconditioner.load(tmp_path / "chain")
    assert L.depth == Q.depth == 2 and L.cplx
    V = (np.random.default_rng(9).standard_normal((30, 3))
         + 1j * np.random.default_rng(10).standard_normal((30, 3)))
    assert np.allclose(L.apply(V), Q.apply(V), rtol=0, atol=1e-14)
    for a, b in zip(L.factors(), Q.factors()):
        assert np.array_equal(a.to_scipy().toarray(), b.to_scipy().toarray())
