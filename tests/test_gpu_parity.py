"""Device parity: the B200 path against the golden outputs of the real
reference (tests/golden/) and the CPU oracle, through the C-ABI library.

Bars: assembly and patterns bit-exact; SPAI / update
factors within 1e-10 relative Frobenius (structure equal modulo exact
zeros); residuals within 1e-12; solves to the 1e-8 relative residual with
iteration counts within +-2.
"""

import os
import sys

import numpy as np
import pytest
import scipy.sparse as sp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import goldens as G  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "oracle"))
import pmor_oracle as orc  # noqa: E402


@pytest.fixture(scope="module")
def pm():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1809_06574_b200 as pm
    from paper_1809_06574_b200 import _abi
    _abi.load()
    return pm


def _mf(name):
    return 12 if name == "rand40" else (50 if name == "tridiag9" else 80)


# ---------------------------------------------------------------------------
# assembly (kernel 1): bit-exact
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", list(G.WORKLOAD_CASES))
def test_assembly_bit_exact(pm, name):
    from paper_1809_06574_b200.workloads import make_config
    g = G.load(name + "_assemble")
    cfg, scale = G.WORKLOAD_CASES[name]
    W = make_config(cfg, scale=scale)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    i = 0
    while "asm%d_point" % i in g:
        pt = g["asm%d_point" % i]
        A = model.assemble(pt[0], pt[1:]).to_scipy()
        ref = G.csr(g, "asm%d" % i)
        assert np.array_equal(A.indptr, ref.indptr)
        assert np.array_equal(A.indices, ref.indices)
        assert np.array_equal(A.data, ref.data)
        i += 1


def test_affine_evaluate_bit_exact(pm):
    rs = np.random.RandomState(3)
    terms = [sp.random(60, 60, density=0.1, random_state=rs, format="csr") + 3 * sp.identity(60)]
    terms += [sp.random(60, 60, density=0.05, random_state=rs, format="csr") for _ in range(3)]
    coeffs = [0.3, 0.0, -1.7]
    ref = orc.affine_evaluate(terms, coeffs)
    got = pm.AffineFamily(terms).evaluate(coeffs).to_scipy()
    assert np.array_equal(got.indptr, ref.indptr)
    assert np.array_equal(got.indices, ref.indices)
    assert np.array_equal(got.data, ref.data)


def test_assembly_drops_exact_zeros(pm):
    # K0 and K1 cancel exactly on the off-diagonal at p = -1
    n = 20
    K0 = sp.diags([np.ones(n - 1), 4 * np.ones(n), np.ones(n - 1)], (-1, 0, 1)).tocsr()
    K1 = sp.diags([np.ones(n - 1), np.ones(n - 1)], (-1, 1)).tocsr()
    M = sp.identity(n, format="csr")
    model = pm.SecondOrderModel.from_mdk([M], None, [K0, K1], rhs=np.ones((n, 1)))
    A = model.assemble(0.0, [-1.0]).to_scipy(drop_zeros=False)
    ref = orc.assemble_mdk([M], None, [K0, K1], 0.0, [-1.0])
    assert np.array_equal(A.indptr, ref.indptr) and np.array_equal(A.data, ref.data)


# ---------------------------------------------------------------------------
# patterns (kernel 2 + augmentation): bit-exact
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", G.CASES)
def test_patterns_bit_exact(pm, name):
    g = G.load(name)
    A1 = G.csr(g, "A1")
    p0 = pm.spai_pattern(A1, level=0)
    for a, b in zip(p0.columns, G.pattern(g, "pat0")):
        assert np.array_equal(a, b)
    if G.has(g, "pat1"):
        p1 = pm.spai_pattern(A1, level=1, max_fill_per_column=_mf(name))
        for j, (a, b) in enumerate(zip(p1.columns, G.pattern(g, "pat1"))):
            assert np.array_equal(a, b), j


@pytest.mark.parametrize("name", G.CASES)
def test_touched_rows_bit_exact(pm, name):
    """J_j exported by the least-squares kernel (mode 2) == spai.py:237-240."""
    import torch as th
    from paper_1809_06574_b200 import _abi
    from paper_1809_06574_b200.device import DeviceCSR, level0_pattern
    from paper_1809_06574_b200.spai import _get_tiers, _run_tiers
    g = G.load(name)
    for Akey, Tkey, Jkey in (("A1", None, "J0"), ("Al", "A1", "J0u")):
        if not G.has(g, Jkey):
            continue
        A = DeviceCSR.from_scipy(G.csr(g, Akey))
        T = DeviceCSR.from_scipy(G.csr(g, Tkey)) if Tkey else None
        pat = level0_pattern(A)
        Jref = G.pattern(g, Jkey)
        jptr = np.zeros(len(Jref) + 1, dtype=np.int64)
        jptr[1:] = np.cumsum([len(c) for c in Jref])
        jptr_d = th.as_tensor(jptr.astype(np.int32), device="cuda")
        jidx = th.full((max(int(jptr[-1]), 1),), -1, dtype=th.int32, device="cuda")
        tiers = _get_tiers(pat, A, T)
        n = A.n
        coef = th.empty(max(pat.nnz, 1), dtype=th.float64, device="cuda")
        resid = th.empty(n, dtype=th.float64, device="cuda")
        flags = th.zeros(n, dtype=th.int32, device="cuda")
        _run_tiers(tiers, pat, A.csc(), T.csc() if T else None, coef, resid, flags, mode=2,
                   jptr=jptr_d, jidx=jidx)
        got = jidx.cpu().numpy()
        for j in range(n):
            assert np.array_equal(got[jptr[j]:jptr[j + 1]], Jref[j]), (Jkey, j)


# ---------------------------------------------------------------------------
# SPAI and update values (kernels 3/4)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", G.CASES)
def test_spai_and_update_vs_reference(pm, name):
    g = G.load(name)
    A1, Al = G.csr(g, "A1"), G.csr(g, "Al")
    for lvl in (0, 1):
        if not G.has(g, "P%d" % lvl):
            continue
        cfg = pm.SpaiConfig(pattern_level=lvl, max_fill_per_column=_mf(name))
        # the first build records the symbolic plan, the second replays it
        # (register warp tier for small columns): both against the reference
        for rep in range(2):
            P, st = pm.spai_build(A1, cfg)
            G.compare_factor(P.matrix.to_scipy(), G.csr(g, "P%d" % lvl))
            assert np.allclose(st.residuals, g["P%d_resid" % lvl], rtol=0, atol=1e-12)
            assert st.augmented_columns == int(g["P%d_aug" % lvl])
            assert st.rank_deficient_columns == int(g["P%d_def" % lvl])
        if not G.has(g, "Q%d" % lvl):
            continue
        ucfg = pm.UpdateConfig(pattern_level=lvl, max_fill_per_column=_mf(name))
        for rep in range(2):
            Pu, su = pm.update_first(A1, Al, P, ucfg)
            assert Pu.kind == "factored" and Pu.depth == 2
            G.compare_factor(Pu.q.to_scipy(), G.csr(g, "Q%d" % lvl))
            assert np.allclose(su.residuals, g["Q%d_resid" % lvl], rtol=0, atol=1e-12)
            assert su.augmented_columns == int(g["Q%d_aug" % lvl])
            assert su.rank_deficient_columns == int(g["Q%d_def" % lvl])


def test_build_deterministic(pm):
    g = G.load("c3s6")
    A1 = G.csr(g, "A1")
    a, _ = pm.spai_build(A1, pm.SpaiConfig(pattern_level=1))
    b, _ = pm.spai_build(A1, pm.SpaiConfig(pattern_level=1))
    assert np.array_equal(a.matrix.vals.cpu().numpy(), b.matrix.vals.cpu().numpy())


# ---------------------------------------------------------------------------
# reference unit-test assertions on real inputs (test_spai.py, test_update.py)
# ---------------------------------------------------------------------------

def test_known_answers(pm):
    P, st = pm.spai_build(sp.identity(6, format="csr"))
    assert np.allclose(P.matrix.to_scipy().toarray(), np.eye(6), atol=1e-15)
    assert st.residuals.max() <= 1e-14
    d = np.array([2.0, 5.0, 0.5, 8.0])
    P, _ = pm.spai_build(sp.diags(d).tocsr())
    assert np.allclose(P.matrix.to_scipy().diagonal(), 1 / d, rtol=0, atol=1e-15)
    sup, vals, resid, dfc = pm.spai_column(sp.diags([2.0, 4.0]).tocsr(), 1, [1])
    assert abs(vals[0] - 0.25) <= 1e-15 and resid <= 1e-15 and not dfc
    # degenerate column flagged, not fatal (test_spai.py:170-174)
    _, st = pm.spai_build(sp.csr_matrix(np.array([[1.0, 0.0], [0.0, 0.0]])),
                          pm.SpaiConfig(pattern_level=0))
    assert st.rank_deficient_columns >= 1


def test_full_pattern_inverse(pm):
    rs = np.random.RandomState(17)
    A = sp.random(50, 50, density=0.08, random_state=rs, format="csr") + 4 * sp.identity(50)
    P, _ = pm.spai_build(A, pattern=[np.arange(50)] * 50)
    inv = np.linalg.inv(A.toarray())
    assert np.linalg.norm(P.matrix.to_scipy().toarray() - inv) <= 1e-10 * np.linalg.norm(inv)


def test_update_identity_and_scaling(pm):
    rs = np.random.RandomState(1)
    A1 = (sp.random(30, 30, density=0.08, random_state=rs, format="csr")
          + 4 * sp.identity(30)).tocsr()
    P1, _ = pm.spai_build(A1)
    P, st = pm.update_first(A1, A1, P1)
    assert np.linalg.norm(P.q.to_scipy().toarray() - np.eye(30)) <= 1e-10
    assert st.residuals.max() <= 1e-10
    P, _ = pm.update_first(A1, 2.0 * A1, P1)
    assert np.linalg.norm(P.q.to_scipy().toarray() - 0.5 * np.eye(30)) <= 1e-10
    V = np.random.default_rng(7).standard_normal((30, 2))
    direct = P.materialize() @ V
    assert np.linalg.norm(P.apply(V) - direct) <= 1e-13 * np.linalg.norm(direct)
    P3, _ = pm.update_second(A1, A1, P)
    assert P3.depth == 3


# ---------------------------------------------------------------------------
# block GCRO (kernel 5)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["rand40", "tridiag9", "c1s24", "c2s8", "c3s6", "c5n500"])
def test_block_gcro_vs_reference(pm, name):
    g = G.load(name)
    A1, Al, B = G.csr(g, "A1"), G.csr(g, "Al"), g["B"]
    P0, _ = pm.spai_build(A1, pm.SpaiConfig(pattern_level=0))
    Pu, _ = pm.update_first(A1, Al, P0, pm.UpdateConfig(pattern_level=0))
    for tag, A, P in (("s1", A1, P0), ("s2", Al, Pu), ("nop", Al, None)):
        X, rep = pm.block_gcro_solve(A, B, P=P, cfg=pm.SolverConfig(tol=1e-8))
        assert rep.converged == bool(g[tag + "_conv"])
        assert abs(rep.iterations - int(g[tag + "_iters"])) <= 2, (tag, rep.iterations,
                                                                   int(g[tag + "_iters"]))
        rel = np.linalg.norm(B - A @ X, axis=0) / np.linalg.norm(B, axis=0)
        assert np.all(rel <= 1e-8), rel
        assert abs(float(np.max(rep.final_residuals)) - rel.max()) <= 1e-9


def test_gcro_known_answers(pm):
    I5 = sp.identity(5, format="csr")
    x, rep = pm.gcro_solve(I5, np.arange(1.0, 6.0))
    assert rep.converged and rep.iterations <= 1 and np.linalg.norm(x - np.arange(1.0, 6.0)) < 1e-12
    A = sp.diags(np.arange(1.0, 11.0)).tocsr()
    x, rep = pm.gcro_solve(A, np.ones(10))
    assert rep.converged and np.linalg.norm(x - 1 / np.arange(1.0, 11.0)) <= 1e-10
    with pytest.raises(pm.SolverBreakdown):
        pm.gcro_solve(sp.diags([1.0, 0.0, 0.0]).tocsr(), np.array([1.0, 1.0, 1.0]))
    with pytest.raises(ValueError):
        pm.gcro_solve(sp.identity(4, format="csr"), np.ones(5))
    with pytest.raises(TypeError):
        pm.apply_preconditioner(np.eye(3), np.ones((3, 1)))


def test_block_special_cases(pm):
    rs = np.random.RandomState(27)
    A = (sp.random(50, 50, density=0.08, random_state=rs, format="csr")
         + 4 * sp.identity(50)).tocsr()
    rng = np.random.default_rng(28)
    b1, b2 = rng.standard_normal(50), rng.standard_normal(50)
    X, rep = pm.block_gcro_solve(A, np.column_stack([b1, b2, b1 + b2]))   # rank 2 block
    assert rep.converged and np.linalg.norm(X[:, 2] - X[:, 0] - X[:, 1]) <= 1e-9
    X, rep = pm.block_gcro_solve(A, np.column_stack([b1, np.zeros(50)]))  # zero column
    assert rep.converged and np.all(X[:, 1] == 0) and rep.final_residuals[1] == 0.0
    Bm = rng.standard_normal((50, 4))
    Bm[:, 2] *= 1e-6
    X, rep = pm.block_gcro_solve(A, Bm)                                    # column scales
    rel = np.linalg.norm(Bm - A @ X, axis=0) / np.linalg.norm(Bm, axis=0)
    assert rep.converged and np.all(rel <= 1e-10)
    x, rep = pm.gcro_solve(A, b1, cfg=pm.SolverConfig(max_iters=3))       # not converged
    assert not rep.converged and rep.iterations == 3 and np.all(np.isfinite(x))
    x, rep = pm.gcro_solve(A, b1, cfg=pm.SolverConfig(inner_restart=8, outer_space_dim=5))
    assert rep.converged                                                   # restarts + fold
    assert np.linalg.norm(b1 - A @ x) / np.linalg.norm(b1) <= 1e-10


def test_restart_matches_oracle(pm):
    """Restarted cycles with outer-space recycling follow the oracle."""
    rs = np.random.RandomState(9)
    A = (sp.random(150, 150, density=0.12, random_state=rs, format="csr")
         + 4 * sp.identity(150)).tocsr()
    B = np.random.default_rng(10).standard_normal((150, 3))
    cfg = dict(inner_restart=4, outer_space_dim=5, tol=1e-10)
    X, rep = pm.block_gcro_solve(A, B, cfg=pm.SolverConfig(**cfg))
    Xr, info = orc.block_gcro(A, B, None, **cfg)
    assert rep.converged and info["converged"]
    assert abs(rep.iterations - info["iterations"]) <= 2, (rep.iterations, info["iterations"])


# ---------------------------------------------------------------------------
# full sequences (driver) vs the oracle
# ---------------------------------------------------------------------------

def test_c1_sequence_vs_oracle(pm):
    from paper_1809_06574_b200.workloads import make_config
    W = make_config(1)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=0),
                           update=pm.UpdateConfig(pattern_level=0))
    recs, info = pm.run_sequence(model, W.s_grid, W.p_grid, pol, keep_solutions=True)
    ref = orc.run_sequence(W, level=0, tol=1e-8)
    pts = W.points()
    for r, (idx, Xr, inf, _) in zip(recs, ref):
        assert r["index"] == idx
        assert r["converged"] and inf["converged"]
        assert abs(r["iterations"] - inf["iterations"]) <= 2, (idx, r["iterations"],
                                                               inf["iterations"])
        A = orc.assemble_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms, *pts[idx])
        X = r["X"].cpu().numpy()
        rel = np.linalg.norm(W.rhs - A @ X, axis=0) / np.linalg.norm(W.rhs, axis=0)
        assert np.all(rel <= 1e-8)


def test_concurrent_workers_bitwise_identical(pm):
    """Systems driven by 3 host threads on their own streams (grid-barrier
    kernels serialised on a shared stream) give bitwise the same solutions
    and iteration counts as the single-stream run."""
    from paper_1809_06574_b200.workloads import make_config
    W = make_config(1, scale=32)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=0),
                           update=pm.UpdateConfig(pattern_level=0))
    r1, _ = pm.run_sequence(model, W.s_grid, W.p_grid, pol, keep_solutions=True, workers=1,
                            batch=1)
    r3, _ = pm.run_sequence(model, W.s_grid, W.p_grid, pol, keep_solutions=True, workers=3,
                            batch=1)
    assert [r["index"] for r in r1] == [r["index"] for r in r3]
    for a, b in zip(r1, r3):
        assert a["iterations"] == b["iterations"]
        assert torch.equal(a["X"], b["X"])


@pytest.mark.parametrize("cfg,level", [(2, 0), (3, 0), (3, 1), (4, 0)])
def test_full_size_sampled_columns(pm, cfg, level):
    """Full-size configs: every column built on the device, a deterministic
    sample checked against the oracle (supports bit-exact, values 1e-10)."""
    from paper_1809_06574_b200.workloads import make_config
    W = make_config(cfg)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pts = W.points()
    A1 = model.assemble(*pts[0])
    A2 = model.assemble(*pts[1])
    P1, st = pm.spai_build(A1, pm.SpaiConfig(pattern_level=level))
    Pu, su = pm.update_first(A1, A2, P1, pm.UpdateConfig(pattern_level=level))
    A1h, A2h = A1.to_scipy(), A2.to_scipy()
    cols = np.sort(np.random.default_rng(7).permutation(A1.n)[:300])
    for F, res, stats in ((P1.matrix, orc.spai_build(A1h, pattern_level=level, columns=cols), st),
                          (Pu.q, orc.update_factor(A1h, A2h, pattern_level=level, columns=cols),
                           su)):
        Fc = F.to_scipy(drop_zeros=False).tocsc()
        for (j, sup, coef, r, dfc, aug) in res:
            lo, hi = Fc.indptr[j], Fc.indptr[j + 1]
            assert np.array_equal(Fc.indices[lo:hi], sup), j
            err = np.linalg.norm(Fc.data[lo:hi] - coef) / max(np.linalg.norm(coef), 1e-300)
            assert err <= 1e-10, (j, err)
            assert abs(stats.residuals[j] - r) <= 1e-12


def test_c5_large_columns_semi_normal(pm):
    """c5 (power-law rows) at n = 2^16: most columns exceed shared memory and
    go through the semi-normal-equations kernel; sampled columns must match
    the oracle's gelsy solution (supports bit-exact, values 1e-10)."""
    from paper_1809_06574_b200.workloads import make_config
    W = make_config(5, scale=1 << 16)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pts = W.points()
    A1 = model.assemble(*pts[0])
    A2 = model.assemble(*pts[1])
    P1, st = pm.spai_build(A1, pm.SpaiConfig(pattern_level=0))
    Pu, su = pm.update_first(A1, A2, P1, pm.UpdateConfig(pattern_level=0))
    A1h, A2h = A1.to_scipy(), A2.to_scipy()
    cols = np.sort(np.random.default_rng(11).permutation(A1.n)[:120])
    for F, res, stats in ((P1.matrix, orc.spai_build(A1h, pattern_level=0, columns=cols), st),
                          (Pu.q, orc.update_factor(A1h, A2h, pattern_level=0, columns=cols),
                           su)):
        Fc = F.to_scipy(drop_zeros=False).tocsc()
        for (j, sup, coef, r, dfc, aug) in res:
            lo, hi = Fc.indptr[j], Fc.indptr[j + 1]
            assert np.array_equal(Fc.indices[lo:hi], sup), j
            err = np.linalg.norm(Fc.data[lo:hi] - coef) / max(np.linalg.norm(coef), 1e-300)
            assert err <= 1e-10, (j, err)
            assert abs(stats.residuals[j] - r) <= 1e-12


def test_c2_sequence_property(pm):
    """c2 at full size: every system's true residual <= 1e-8 (recomputed on
    the host from X) and the first two systems' iterations match the oracle."""
    from paper_1809_06574_b200.workloads import make_config
    W = make_config(2)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=0),
                           update=pm.UpdateConfig(pattern_level=0))
    s_grid = W.s_grid[:2]
    recs, info = pm.run_sequence(model, s_grid, W.p_grid[:3], pol, keep_solutions=True)
    ref = orc.run_sequence(W, level=0, tol=1e-8, systems={0, 1})
    for r, (idx, Xr, inf, _) in zip(recs[:2], ref):
        assert abs(r["iterations"] - inf["iterations"]) <= 2
    pts = [(s, np.atleast_1d(p)) for s in s_grid for p in W.p_grid[:3]]
    for r in recs:
        A = orc.assemble_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms, *pts[r["index"]])
        X = r["X"].cpu().numpy()
        rel = np.linalg.norm(W.rhs - A @ X, axis=0) / np.linalg.norm(W.rhs, axis=0)
        assert r["converged"] and np.all(rel <= 1e-8)


@pytest.mark.parametrize("name", ["rand40", "c1s24", "c2s8", "c3s6", "c5n500"])
def test_device_cycle_matches_host_loop(pm, name):
    """The persistent device cycle (pmp_gcro_cycle_dev) against the
    host-driven native loop (pmp_gcro_inner): same convergence, iteration
    counts within 2 (preconditioned), solutions within the solve tolerance;
    both geometries
    (1 and 2 blocks per SM)."""
    from paper_1809_06574_b200 import krylov
    g = G.load(name)
    A1, Al, B = G.csr(g, "A1"), G.csr(g, "Al"), g["B"]
    P0, _ = pm.spai_build(A1, pm.SpaiConfig(pattern_level=0))
    Pu, _ = pm.update_first(A1, Al, P0, pm.UpdateConfig(pattern_level=0))
    cfg = pm.SolverConfig(tol=1e-10, inner_restart=12, outer_space_dim=4)
    saved = krylov.DEVICE_CYCLE, krylov._CYCLE_BPS
    try:
        for A, P in ((A1, P0), (Al, Pu), (Al, None)):
            krylov.DEVICE_CYCLE = False
            Xh, rh = pm.block_gcro_solve(A, B, P=P, cfg=cfg)
            for bps in (1, 2):
                krylov.DEVICE_CYCLE, krylov._CYCLE_BPS = True, bps
                Xd, rd = pm.block_gcro_solve(A, B, P=P, cfg=cfg)
                assert rd.converged == rh.converged
                if P is not None:
                    # (unpreconditioned, the small c3s6 case deflates at most
                    # steps and is rounding-chaotic: convergence only)
                    assert abs(rd.iterations - rh.iterations) <= 2, (rd.iterations,
                                                                     rh.iterations)
                assert rd.matvec_count > 0
                rel = np.linalg.norm(B - A @ Xd, axis=0) / np.linalg.norm(B, axis=0)
                assert np.all(rel <= 1e-10), rel
                assert len(rd.residual_history) >= rd.iterations
    finally:
        krylov.DEVICE_CYCLE, krylov._CYCLE_BPS = saved


@pytest.mark.parametrize("name", ["c1s24", "c2s8", "c3s6", "c5n500"])
def test_solve_batch_matches_single(pm, name):
    """Whole solves on the device, several systems per launch
    (block_gcro_solve_batch): every system's residual <= tol (recomputed on
    the host), iterations within 2 of the single-system path, histories
    end at the true residual."""
    import torch
    g = G.load(name)
    A1, Al, B = G.csr(g, "A1"), G.csr(g, "Al"), g["B"]
    P0, _ = pm.spai_build(A1, pm.SpaiConfig(pattern_level=0))
    Pu, _ = pm.update_first(A1, Al, P0, pm.UpdateConfig(pattern_level=0))
    cfg = pm.SolverConfig(tol=1e-8)
    Bd = torch.as_tensor(B, device="cuda")
    for systems in ([(A1, P0), (Al, P0)], [(Al, Pu), (A1, Pu), (Al, Pu)],
                    [(A1, P0), (Al, Pu), (Al, None)]):    # mixed chain lengths
        for groups in (1, 2, 3):
            res = pm.block_gcro_solve_batch(systems, Bd, cfg=cfg, groups=groups)
            for (A, P), (X, rep) in zip(systems, res):
                Xh, rh = pm.block_gcro_solve(A, B, P=P, cfg=cfg)
                assert rep.converged == rh.converged
                assert abs(rep.iterations - rh.iterations) <= 2, (rep.iterations, rh.iterations)
                Xn = X.cpu().numpy()
                rel = np.linalg.norm(B - A @ Xn, axis=0) / np.linalg.norm(B, axis=0)
                assert np.all(rel <= 1e-8), rel
                assert abs(float(np.max(rep.final_residuals)) - rel.max()) <= 1e-9


def test_ls_plan_replay(pm):
    """SPAI / update columns solved from a recorded symbolic plan (second and
    later builds on the same structures; small columns go through the
    register warp tier, whose reductions run in a different order) agree with
    the unplanned solve to rounding, and replays are bitwise reproducible."""
    from paper_1809_06574_b200 import spai
    from paper_1809_06574_b200.workloads import make_config
    W = make_config(2, scale=12)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pts = W.points()
    A1 = model.assemble(*pts[0])
    P1, _ = pm.spai_build(A1, pm.SpaiConfig(pattern_level=0))        # records
    P1b, _ = pm.spai_build(A1, pm.SpaiConfig(pattern_level=0))       # replays
    P1c, _ = pm.spai_build(A1, pm.SpaiConfig(pattern_level=0))       # replays
    assert torch.equal(P1b.matrix.vals, P1c.matrix.vals)
    d = (P1.matrix.vals - P1b.matrix.vals).norm() / P1.matrix.vals.norm()
    assert float(d) <= 1e-13
    outs = []
    for pt in pts[1:4]:
        A = model.assemble(*pt)
        Pu, su = pm.update_first(A1, A, P1, pm.UpdateConfig(pattern_level=0))
        saved = spai.USE_LS_PLANS
        spai.USE_LS_PLANS = False
        try:
            Pr, sr = pm.update_first(A1, A, P1, pm.UpdateConfig(pattern_level=0))
        finally:
            spai.USE_LS_PLANS = saved
        d = (Pu.q.vals - Pr.q.vals).norm() / Pr.q.vals.norm()
        assert float(d) <= 1e-13, float(d)
        assert np.allclose(np.asarray(su.residuals), np.asarray(sr.residuals), rtol=0,
                           atol=1e-14)
        assert su.rank_deficient_columns == sr.rank_deficient_columns
        outs.append(Pu)


def test_update_first_many_bitwise(pm):
    """Updates of a sweep built together (one multi-system least-squares
    launch for the small-column tier) == one at a time, bitwise, and within
    the parity bar of the oracle on sampled columns."""
    from paper_1809_06574_b200.workloads import make_config
    W = make_config(2, scale=12)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pts = W.points()
    A1 = model.assemble(*pts[0])
    P1, _ = pm.spai_build(A1, pm.SpaiConfig(pattern_level=0))
    As = model.assemble_many(pts[1:7])
    cfg = pm.UpdateConfig(pattern_level=0)
    many = pm.update_first_many(A1, As, P1, cfg)
    for A, (Pm, sm) in zip(As, many):
        P, s = pm.update_first(A1, A, P1, cfg)
        assert torch.equal(Pm.q.vals, P.q.vals)
        assert np.array_equal(np.asarray(sm.residuals), np.asarray(s.residuals))
        assert sm.rank_deficient_columns == s.rank_deficient_columns
    A1h = A1.to_scipy()
    for A, (Pm, sm) in list(zip(As, many))[::3]:
        Q, res = orc.update_factor(A1h, A.to_scipy(), pattern_level=0)[:2]
        G.compare_factor(Pm.q.to_scipy(), Q)


def test_permute_batch_matches_single(pm):
    """pmp_permute_batch (a window's factors in one launch) == pmp_permute
    per array, bitwise, with strided rows; k = 0 / nnz = 0 are no-ops."""
    from paper_1809_06574_b200 import _abi
    g = torch.Generator().manual_seed(7)
    nnz, k, stride = 1237, 5, 1300
    perm = torch.randperm(nnz, generator=g).to(torch.int32).cuda()
    src = torch.randn(k, stride, generator=g, dtype=torch.float64).cuda()
    dst = torch.full((k, stride), -1.0, dtype=torch.float64, device="cuda")
    _abi.call("pmp_permute_batch", nnz, _abi.ptr(perm), k, _abi.ptr(src), stride,
              _abi.ptr(dst), stride, _abi.stream())
    for q in range(k):
        ref = torch.empty(nnz, dtype=torch.float64, device="cuda")
        _abi.call("pmp_permute", nnz, _abi.ptr(perm), _abi.ptr(src[q]), _abi.ptr(ref),
                  _abi.stream())
        assert torch.equal(dst[q, :nnz], ref)
        assert torch.all(dst[q, nnz:] == -1.0)
    _abi.call("pmp_permute_batch", nnz, _abi.ptr(perm), 0, _abi.ptr(src), stride,
              _abi.ptr(dst), stride, _abi.stream())
    _abi.call("pmp_permute_batch", 0, _abi.ptr(perm), k, _abi.ptr(src), stride,
              _abi.ptr(dst), stride, _abi.stream())
    torch.cuda.synchronize()


def test_assemble_many_bit_exact(pm):
    """A window assembled in multi-system launches == one system at a time,
    bitwise (symmetric and unsymmetric terms; a zero parameter changes the
    recipe shape mid-window)."""
    from paper_1809_06574_b200.workloads import make_config
    W = make_config(1, scale=16)
    rng = np.random.default_rng(5)
    n = W.mass_terms[0].shape[0]
    K1 = sp.random(n, n, density=4.0 / n, random_state=rng, format="csr")
    for stiff in (W.stiffness_terms, [W.stiffness_terms[0], K1]):
        model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, stiff, rhs=W.rhs)
        pts = list(W.points()) + [(0.7, np.array([0.0])), (2.0, np.array([0.3]))]
        many = model.assemble_many(pts)
        for (s, p), Am in zip(pts, many):
            A = model.assemble(s, p)
            assert torch.equal(Am.vals, A.vals)
            assert np.array_equal(Am.to_scipy().toarray(), A.to_scipy().toarray())


def test_large_n_rows_beyond_shared_memory(pm):
    """n large enough that a block's W rows no longer fit in shared memory
    (c3 at full size, n = 262,144, s = 16): the persistent solve switches to
    W rows in global memory; every solution reaches the 1e-8 true residual."""
    from paper_1809_06574_b200.workloads import make_config
    W = make_config(3)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=0),
                           update=pm.UpdateConfig(pattern_level=0))
    recs, _ = pm.run_sequence(model, W.s_grid[:1], W.p_grid[:2], pol,
                              pm.SolverConfig(tol=1e-8), keep_solutions=True)
    pts = [(W.s_grid[0], np.atleast_1d(p)) for p in W.p_grid[:2]]
    for r in recs:
        A = model.assemble(*pts[r["index"]]).to_scipy()
        X = r["X"].cpu().numpy()
        rel = np.linalg.norm(W.rhs - A @ X, axis=0) / np.linalg.norm(W.rhs, axis=0)
        assert r["converged"] and rel.max() <= 1e-8, (r["index"], rel.max())


# ---------------------------------------------------------------------------
# persistence: load the chain the reference saved, apply
# it on the device; save ours and load it back
# ---------------------------------------------------------------------------

def test_load_reference_saved_chain(pm, tmp_path):
    d = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "precond_ref")
    P = pm.Preconditioner.load(d)
    assert P.kind == "factored" and P.depth == 2
    g = np.load(os.path.join(d, "apply.npz"))
    Y = P.apply(g["V"])
    err = np.linalg.norm(Y - g["Y"]) / np.linalg.norm(g["Y"])
    assert err <= 1e-13, err
    # ours -> files -> ours: same factors bit for bit, same apply bit for bit
    P.save(tmp_path / "p", stats_summary={"columns": int(g["n"])})
    P2 = pm.Preconditioner.load(tmp_path / "p")
    for F1, F2 in zip(P.factors(), P2.factors()):
        a, b = F1.to_scipy(), F2.to_scipy()
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
        assert np.array_equal(a.data, b.data)
    assert np.array_equal(P2.apply(g["V"]), Y)


def test_save_load_built_preconditioner(pm, tmp_path):
    from paper_1809_06574_b200.workloads import make_config
    W = make_config(1, scale=16)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pts = W.points()
    A1, A2 = model.assemble(*pts[0]), model.assemble(*pts[1])
    P1, st = pm.spai_build(A1, pm.SpaiConfig(pattern_level=0))
    P2, _ = pm.update_first(A1, A2, P1, pm.UpdateConfig(pattern_level=0))
    P2.save(tmp_path / "chain", stats_summary=st.summary())
    import json
    side = json.load(open(tmp_path / "chain" / "preconditioner.json"))
    assert side["kind"] == "factored" and len(side["factors"]) == 2
    assert side["stats"]["columns"] == W.n
    Q = pm.Preconditioner.load(tmp_path / "chain")
    V = np.random.default_rng(5).standard_normal((W.n, 4))
    assert np.array_equal(Q.apply(V), P2.apply(V))
    # the reference's reader sees the same values (scipy.io.mmread + as_csr)
    import scipy.io
    R = sp.csr_matrix(scipy.io.mmread(str(tmp_path / "chain" / "factor_01.mtx"), spmatrix=False))
    M = P1.matrix.to_scipy()
    assert np.array_equal(R.real.toarray(), M.toarray())


# ---------------------------------------------------------------------------
# moment pipeline vs the reference's rpmor_reduce
# (tests/golden/rpmor_small.npz, written by the real reference)
# ---------------------------------------------------------------------------

def _rpmor_golden(pm):
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                             "rpmor_small.npz"))
    terms = [sp.csr_matrix((g["t%d_data" % j], g["t%d_indices" % j], g["t%d_indptr" % j]))
             for j in range(3)]
    return g, pm.AffineFamily(terms, rhs=g["B"], output=g["C"])


def test_rpmor_reduce_vs_reference(pm, tmp_path):
    g, fam = _rpmor_golden(pm)
    pol = pm.PrecondPolicy(kind="spai-update-first", spai=pm.SpaiConfig(pattern_level=0),
                           update=pm.UpdateConfig(pattern_level=0))
    pts = [pm.ExpansionPoint(p, label="p%d" % i) for i, p in enumerate(g["points"])]
    red, rep = pm.rpmor_reduce(fam, pts, levels=1, solver_cfg=pm.SolverConfig(tol=1e-10),
                               policy=pol)
    assert rep.basis_size == g["basis"].shape[1]
    assert [r.n_rhs for r in rep.records] == list(g["n_rhs"])
    assert [r.level for r in rep.records] == list(g["levels"])
    it = np.array([r.iterations for r in rep.records])
    assert np.abs(it - g["iters"]).max() <= 2, (it, g["iters"])
    V = red.basis.cpu().numpy()
    assert np.linalg.norm(V - g["basis"]) <= 1e-8 * np.linalg.norm(g["basis"])
    assert np.abs(V.T @ V - np.eye(V.shape[1])).max() <= 1e-12
    for j in range(3):
        ref = g["red_t%d" % j]
        assert np.linalg.norm(red.terms[j] - ref) <= 1e-8 * np.linalg.norm(ref)
    for q, H in zip(g["queries"], g["transfer"]):
        Hq = red.transfer(q)
        assert np.linalg.norm(Hq - H) <= 1e-8 * np.linalg.norm(H)
    red.save(tmp_path / "rom")
    back = pm.ReducedModel.load(tmp_path / "rom")
    for a, b in zip(back.terms, red.terms):
        assert np.array_equal(a, b)
    assert np.array_equal(back.basis, V)


def test_moments_known_answers(pm):
    n = 12
    I = sp.identity(n, format="csr")
    Z = sp.csr_matrix((n, n))
    fam = pm.AffineFamily([I, Z], rhs=np.arange(1.0, n + 1.0)[:, None])
    X0, _ = pm.zeroth_moment(fam, [0.0])
    assert np.linalg.norm(X0[:, 0] - np.arange(1.0, n + 1.0)) <= 1e-12
    X1, _ = pm.first_moments(fam, [0.0], X0)
    assert np.all(X1 == 0)
    d = np.array([2.0, 4.0, 8.0])
    fam = pm.AffineFamily([sp.diags(d).tocsr(), sp.csr_matrix((3, 3))], rhs=np.ones((3, 1)))
    X0, _ = pm.zeroth_moment(fam, [0.0])
    assert np.allclose(X0[:, 0], 1.0 / d, rtol=0, atol=1e-12)
    # first-moment right-hand sides: one SpMM per parameter term
    g, fam = _rpmor_golden(pm)
    x0 = np.random.default_rng(1).standard_normal((fam.dim, 1))
    rhs = pm.first_moment_rhs(fam, x0)
    ref = np.hstack([T @ x0 for T in fam.terms[1:]])
    assert np.linalg.norm(rhs - ref) <= 1e-14 * np.linalg.norm(ref)
    with pytest.raises(ValueError):
        pm.rpmor_reduce(fam, [])


def test_extend_orthonormal_basis_matches_oracle(pm):
    rng = np.random.default_rng(4)
    X = rng.standard_normal((500, 6))
    X[:, 3] = X[:, 0] + 2 * X[:, 1]          # dependent: dropped
    X[:, 5] = 0.0                            # zero: skipped
    Q = pm.extend_orthonormal_basis(None, X)
    Qr = orc.extend_orthonormal_basis(None, X)
    assert Q.shape == Qr.shape == (500, 4)
    assert np.abs(Q - Qr).max() <= 1e-12
    Y = rng.standard_normal((500, 3))
    Q2 = pm.extend_orthonormal_basis(Q, Y)
    Q2r = orc.extend_orthonormal_basis(Qr, Y)
    assert np.abs(Q2 - Q2r).max() <= 1e-12


# ---------------------------------------------------------------------------
# experiment CLI vs the reference's run_experiment
# ---------------------------------------------------------------------------

def test_cli_run_matches_reference_report(pm, tmp_path, monkeypatch):
    import json
    from paper_1809_06574_b200 import cli
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    monkeypatch.chdir(root)   # the config names the family by its relative path
    ref = json.load(open(os.path.join(root, "tests", "golden", "cli_report.json")))
    code = cli.main(["run", "--config", "tests/golden/cli_config.json",
                     "--out", str(tmp_path / "run")])
    assert code == cli.EXIT_OK
    got = json.load(open(tmp_path / "run" / "report.json"))
    assert got["config_hash"] == ref["config_hash"]
    assert got["family_fingerprint"] == ref["family_fingerprint"]
    assert len(got["records"]) == len(ref["records"])
    for a, b in zip(got["records"], ref["records"]):
        for key in ("step", "point_label", "level", "call_index", "n_rhs", "converged"):
            assert a[key] == b[key], key
        assert abs(a["iterations"] - b["iterations"]) <= 2
        assert max(a["final_residuals"]) <= 1e-10
    for a, b in zip(got["steps"], ref["steps"]):
        assert a["precond_kind"] == b["precond_kind"]
        for key in ("norm_identity_minus", "norm_first_minus"):
            assert abs(a[key] - b[key]) <= 1e-12 * max(1.0, abs(b[key]))
        assert abs(a["quality_norm"] - b["quality_norm"]) <= 1e-10 * b["quality_norm"]
        assert a["build_stats"]["columns"] == b["build_stats"]["columns"]
        assert abs(a["build_stats"]["max_residual"] - b["build_stats"]["max_residual"]) <= 1e-12
    # the reference's compare accepts the pair
    d = cli.compare_reports(ref, got)
    assert len(d["steps"]) == 3
    # the family written next to the report loads back identically
    fam2, pts2 = cli.load_family(tmp_path / "run" / "family")
    assert [p.values.tolist() for p in pts2] == [[0.5, 0.2], [0.8, 0.3], [1.5, 0.7]]


# ---------------------------------------------------------------------------
# update_second chains and sequence_precondition (test_update.py:98-184 of the
# reference, real inputs)
# ---------------------------------------------------------------------------

def _rand_sparse(n, density, seed):
    rng = np.random.default_rng(seed)
    M = sp.random(n, n, density=density, random_state=rng, format="csr")
    M.data = rng.standard_normal(M.nnz)
    return M


def _well_conditioned(n, seed):
    M = _rand_sparse(n, 0.1, seed)
    d = np.asarray(abs(M).sum(axis=1)).ravel() + 1.0
    return (M + sp.diags(d)).tocsr()


def _seq_family(pm, n=30, seed=20):
    return pm.AffineFamily([_well_conditioned(n, seed), _rand_sparse(n, 0.05, seed + 1),
                            _rand_sparse(n, 0.05, seed + 2)])


def test_update_second_chains(pm):
    A = _well_conditioned(20, 10)
    P1, _ = pm.spai_build(A)
    P2, _ = pm.update_second(A, A, P1)
    assert np.linalg.norm(P2.q.to_scipy().toarray() - np.eye(20)) <= 1e-10
    P3, _ = pm.update_second(A, A, P2)
    assert P3.depth == 3
    M1 = P1.matrix.to_scipy()
    assert np.linalg.norm((P3.materialize() - M1).toarray()) <= 1e-12 * np.linalg.norm(M1.toarray())
    # three systems off one affine family: both strategies within 2x of a fresh build
    fam = pm.AffineFamily([_well_conditioned(40, 12), _rand_sparse(40, 0.05, 60),
                           _rand_sparse(40, 0.05, 61)])
    A1, A2, A3 = (fam.evaluate(p) for p in ([1e-3, 1e-3], [2e-3, 1e-3], [2e-3, 2e-3]))
    P1, _ = pm.spai_build(A1)
    fresh, _ = pm.spai_build(A3)
    first, _ = pm.update_first(A1, A3, P1)
    prev2, _ = pm.update_second(A1, A2, P1)
    second, _ = pm.update_second(A2, A3, prev2)
    qf, q1, q2 = pm.quality(A3, fresh), pm.quality(A3, first), pm.quality(A3, second)
    ref = np.linalg.norm((sp.identity(40) - A3.to_scipy() @ fresh.matrix.to_scipy()).toarray())
    assert abs(qf - ref) <= 1e-12 * ref
    assert q1 <= 2.0 * qf and q2 <= 2.0 * qf and q1 <= q2 + 0.1 * qf


def test_sequence_precondition_semantics(pm):
    fam = _seq_family(pm)
    precs, steps = pm.sequence_precondition(fam, [pm.ExpansionPoint([1e-3, 1e-3])])
    assert len(precs) == 1 and precs[0].kind == "explicit" and steps[0].kind == "initial"
    fam = _seq_family(pm, seed=22)
    pt = pm.ExpansionPoint([1e-3, -1e-3])
    precs, steps = pm.sequence_precondition(fam, [pt, pt])
    assert precs[1].kind == "factored" and steps[1].kind == "update"
    assert np.linalg.norm(precs[1].q.to_scipy().toarray() - np.eye(30)) <= 1e-10
    fam = _seq_family(pm, seed=24)
    pts = [pm.ExpansionPoint([k * 1e-3, -k * 1e-3]) for k in range(4)]
    precs, _ = pm.sequence_precondition(fam, pts, pm.UpdateConfig(approach="second"))
    assert [p.depth for p in precs] == [1, 2, 3, 4]
    precs, _ = pm.sequence_precondition(fam, pts, pm.UpdateConfig(approach="first"))
    assert [p.depth for p in precs] == [1, 2, 2, 2]
    fam = _seq_family(pm, seed=28)
    pts = [pm.ExpansionPoint([0.0, 0.0]), pm.ExpansionPoint([1e-3, 2e-3])]
    pf, _ = pm.sequence_precondition(fam, pts, pm.UpdateConfig(approach="first"))
    ps, _ = pm.sequence_precondition(fam, pts, pm.UpdateConfig(approach="second"))
    a, b = pf[1].q.to_scipy(), ps[1].q.to_scipy()
    assert np.array_equal(a.data, b.data) and np.array_equal(a.indices, b.indices)
    with pytest.raises(ValueError):
        pm.sequence_precondition(fam, [])


# ---------------------------------------------------------------------------
# affine family semantics (test_affine.py:30-90) and the quality diagnostic
# (test_spai.py:149-164) on the device path
# ---------------------------------------------------------------------------

def test_affine_family_semantics(pm):
    n = 25
    A0 = _well_conditioned(n, 40)
    T1, T2 = _rand_sparse(n, 0.1, 41), _rand_sparse(n, 0.1, 42)
    fam = pm.AffineFamily([A0, T1, T2])
    assert np.array_equal(fam.evaluate([0.0, 0.0]).to_scipy().toarray(), A0.toarray())
    got = fam.evaluate([1.0, 0.0]).to_scipy().toarray()
    assert np.abs(got - (A0 + T1).toarray()).max() <= 1e-15
    p = np.array([0.3, -1.2])
    dense = A0.toarray() + p[0] * T1.toarray() + p[1] * T2.toarray()
    assert np.abs(fam.evaluate(p).to_scipy().toarray() - dense).max() <= 1e-14
    # additivity in the point: A(p+q) - A(q) = A(p) - A(0)
    q = np.array([-0.7, 0.4])
    lhs = fam.evaluate(p + q).to_scipy() - fam.evaluate(q).to_scipy()
    rhs = fam.evaluate(p).to_scipy() - fam.evaluate([0.0, 0.0]).to_scipy()
    assert np.abs((lhs - rhs).toarray()).max() <= 1e-13
    a, b = fam.evaluate(p).to_scipy(), fam.evaluate(p).to_scipy()
    assert np.array_equal(a.data, b.data) and np.array_equal(a.indices, b.indices)
    with pytest.raises(ValueError):
        fam.evaluate([1.0])
    with pytest.raises(ValueError):
        pm.AffineFamily([A0, _rand_sparse(n + 1, 0.1, 1)])
    with pytest.raises(ValueError):
        pm.AffineFamily([A0])
    # complex coefficients give a complex128 system (real form on the device)
    Ac = fam.evaluate([1.0 + 1.0j, 0.0]).to_scipy()
    assert np.iscomplexobj(Ac.data) and np.any(Ac.data.imag != 0)


def test_quality_diagnostic(pm):
    n = 30
    A = _well_conditioned(n, 50)
    inv = sp.csr_matrix(np.linalg.inv(A.toarray()))
    assert pm.quality(A, pm.Preconditioner(matrix=inv)) <= 1e-12
    tiny = sp.csr_matrix((np.full(n, 1e-300), (np.arange(n), np.arange(n))), shape=(n, n))
    assert abs(pm.quality(A, pm.Preconditioner(matrix=tiny)) - np.sqrt(n)) <= 1e-12
    P, _ = pm.spai_build(A)
    q = pm.quality(A, P)
    ref = np.linalg.norm(np.eye(n) - A.toarray() @ P.matrix.to_scipy().toarray())
    assert abs(q - ref) <= 1e-12 * max(ref, 1.0) and q <= np.sqrt(n)
    with pytest.raises(ValueError):
        pm.quality(A, pm.Preconditioner.identity(n + 1))


def test_fold_cancellation_band_stays_on_device(pm):
    """c3 at 12^3 (27-point, 16 right-hand sides): half of the systems hit a
    fold whose Gram-based drop test is inside the cancellation band; the
    device resolves those column by column like the reference
    (krylov.py:249-265) instead of re-solving the system on the host path.
    Same iteration counts as the per-system path, residuals to 1e-8."""
    import torch
    from paper_1809_06574_b200 import krylov
    from paper_1809_06574_b200.workloads import make_config
    W = make_config(3, scale=12)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=0),
                           update=pm.UpdateConfig(pattern_level=0))
    cfg = pm.SolverConfig(tol=1e-8)
    p_grid = W.p_grid[:8]
    Bd = torch.as_tensor(W.rhs, device="cuda")
    krylov.FALLBACK_REASONS.clear()
    recs, _ = pm.run_sequence(model, W.s_grid, p_grid, pol, cfg, B=Bd, batch=6,
                              keep_solutions=True, timing=False)
    assert 4 not in krylov.FALLBACK_REASONS, krylov.FALLBACK_REASONS
    ref, _ = pm.run_sequence(model, W.s_grid, p_grid, pol, cfg, B=Bd, batch=1, timing=False)
    it = np.array([r["iterations"] for r in recs])
    it_ref = np.array([r["iterations"] for r in ref])
    assert np.abs(it - it_ref).max() <= 2, (it, it_ref)
    pts = [(s_, np.atleast_1d(p)) for s_ in W.s_grid for p in p_grid]
    for r in recs[::5]:
        A = model.assemble(*pts[r["index"]]).to_scipy()
        X = r["X"].cpu().numpy() if torch.is_tensor(r["X"]) else r["X"]
        rel = np.linalg.norm(W.rhs - A @ X, axis=0) / np.linalg.norm(W.rhs, axis=0)
        assert rel.max() <= 1e-8, rel.max()


def test_window_with_exact_zeros_matches_per_system_path(pm):
    """The batched window is enqueued without a host synchronisation and its
    exact-zero counts are checked after the solves; systems whose assembled
    values cancel exactly (the reference's as_csr drops them) must come out
    as on the per-system path, also when the cancelling system is the
    sequence's first (the SPAI base)."""
    n = 64
    K0 = sp.diags([np.ones(n - 1), 4 * np.ones(n), np.ones(n - 1)], (-1, 0, 1)).tocsr()
    K1 = sp.diags([np.ones(n - 1), np.ones(n - 1)], (-1, 1)).tocsr()
    M = sp.identity(n, format="csr")
    B = np.random.default_rng(9).standard_normal((n, 3))
    model = pm.SecondOrderModel.from_mdk([M], None, [K0, K1], rhs=B)
    pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=0),
                           update=pm.UpdateConfig(pattern_level=0))
    cfg = pm.SolverConfig(tol=1e-10)
    for p_grid in ([0.5, -1.0, 0.25], [-1.0, 0.5]):
        got, _ = pm.run_sequence(model, [0.5, 1.0], p_grid, pol, cfg, batch=6, timing=False,
                                 keep_solutions=True)
        ref, _ = pm.run_sequence(model, [0.5, 1.0], p_grid, pol, cfg, batch=1, timing=False,
                                 keep_solutions=True)
        for a, b in zip(got, ref):
            assert a["iterations"] == b["iterations"], (p_grid, a["index"])
            Xa = a["X"].cpu().numpy() if hasattr(a["X"], "cpu") else a["X"]
            Xb = b["X"].cpu().numpy() if hasattr(b["X"], "cpu") else b["X"]
            assert np.linalg.norm(Xa - Xb) <= 1e-12 * np.linalg.norm(Xb)


@pytest.mark.parametrize("n,s", [(24, 4), (40, 3)])
def test_persistent_solve_hands_back_deflating_blocks(pm, n, s):
    """A block Krylov space that fills the whole space (n < restart length)
    ends in a rank-deficient block: the persistent kernel must hand the
    system back (status 10, reason 3 -- krylov.py:79-95 deflation runs on the
    host-driven path), not write through its absent host mirror (it faulted
    there until round 2).  Same iterations as the host-driven path."""
    import torch
    from paper_1809_06574_b200 import krylov
    rs = np.random.RandomState(7)
    A = sp.csr_matrix(sp.random(n, n, density=min(1.0, 4.0 / n), random_state=rs, format="csr")
                      + 4.0 * sp.identity(n))
    B = np.random.default_rng(3).standard_normal((n, s))
    cfg = pm.SolverConfig(tol=1e-10)
    krylov.FALLBACK_REASONS.clear()
    Ad = krylov._as_dev_csr(A)
    res = krylov.block_gcro_solve_batch([(Ad, None)] * 3, torch.as_tensor(B, device="cuda"),
                                        cfg=cfg, groups=3)
    Xh, rh = pm.block_gcro_solve(A, B, cfg=cfg, _host=True)
    for X, r in res:
        X = X.cpu().numpy()
        rel = np.linalg.norm(B - A @ X, axis=0) / np.linalg.norm(B, axis=0)
        assert r.converged and rel.max() <= 1e-9
        assert abs(r.iterations - rh.iterations) <= 2
    assert krylov.FALLBACK_REASONS.get(3, 0) == 3
    krylov.FALLBACK_REASONS.clear()


def test_grouped_tier_planning_equals_per_column_planning(pm):
    """The LS size tiers decided on the distinct (capacity, |I|, |J|) triples
    (grouped on the device) are the tiers decided column by column: same
    launches, same dimensions, same column order -- on a stencil-like and on
    a power-law (c5-like) size distribution."""
    from paper_1809_06574_b200 import spai
    rng = np.random.default_rng(11)
    n = 200000
    cases = []
    nI = rng.choice([4, 5, 6, 7], size=n, p=[0.01, 0.04, 0.15, 0.8])
    m = np.minimum(nI * 4 - rng.integers(0, 4, n), 25)
    cases.append((nI.astype(np.int64), m.astype(np.int64), spai._pow2(m + nI)))
    nI = np.clip(np.floor(4.0 * rng.uniform(0, 1, n) ** (-1.0 / 0.98)), 4, 200).astype(np.int64)
    m = (nI * rng.integers(5, 40, n)).astype(np.int64)
    cases.append((nI, m, spai._pow2(m + 3 * nI)))
    cols = np.arange(n, dtype=np.int64)
    for nI, m, lcap in cases:
        a = spai._split_tiers(cols, lcap, m, nI)
        b = spai._split_tiers_direct(cols, lcap, m, nI)
        assert len(a) == len(b) and len(a) >= 1
        for x, y in zip(a, b):
            assert (x.team, x.glob, x.mode, x.lcap, x.mcap, x.ncap) == \
                   (y.team, y.glob, y.mode, y.lcap, y.mcap, y.ncap)
            assert np.array_equal(x.cols_host, y.cols_host)
            assert np.array_equal(x.cols.cpu().numpy(), y.cols.cpu().numpy())
