"""Generate the golden fixtures in tests/golden/ by running the REAL reference
``pmorprec`` (importable only in the survey/build container, from
/root/reference/pkg/src) on seeded inputs.

    OPENBLAS_NUM_THREADS=1 PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

The outputs pin both the CPU oracle (tests/test_oracle_golden.py, CPU) and
the device path (tests/test_gpu_parity.py, GPU).  Nothing on the GPU box
reads /root/reference; only these committed .npz files travel.
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
from pmorprec.spai import _column_support, SpaiConfig    # noqa: E402
from pmorprec.update import UpdateConfig                 # noqa: E402
from pmorprec.krylov import SolverConfig                 # noqa: E402
from pmorprec.rpmor import SecondOrderModel              # noqa: E402

from paper_1809_06574_b200.workloads import make_config  # noqa: E402


def csr_arrays(prefix, M, out):
    M = ref.as_csr(M)
    out[prefix + "_indptr"] = M.indptr.astype(np.int64)
    out[prefix + "_indices"] = M.indices.astype(np.int64)
    out[prefix + "_data"] = M.data.real.copy()
    out[prefix + "_imagmax"] = np.array(np.abs(M.data.imag).max() if M.nnz else 0.0)
    out[prefix + "_shape"] = np.array(M.shape)


def pattern_arrays(prefix, cols, out):
    ptr = np.zeros(len(cols) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(c) for c in cols])
    out[prefix + "_ptr"] = ptr
    out[prefix + "_idx"] = (np.concatenate(cols) if cols else np.zeros(0)).astype(np.int64)


def touched(A, supports, targets):
    """J per column via the reference's own expression (spai.py:237-240)."""
    A_csc = ref.as_csr(A).tocsc()
    T = ref.as_csr(targets).tocsc()
    cols = []
    for j, sup in enumerate(supports):
        parts = [T.indices[T.indptr[j]:T.indptr[j + 1]]]
        parts += [_column_support(A_csc, k) for k in sup]
        cols.append(np.unique(np.concatenate(parts)))
    return cols


def stats_arrays(prefix, st, out):
    out[prefix + "_resid"] = np.asarray(st.residuals, dtype=float)
    out[prefix + "_aug"] = np.array(st.augmented_columns)
    out[prefix + "_def"] = np.array(st.rank_deficient_columns)


def build_case(name, A1, Al, B=None, levels=(0, 1), max_fill=80, solve=True, update=True):
    out = {}
    A1 = ref.as_csr(A1)
    Al = ref.as_csr(Al)
    n = A1.shape[0]
    csr_arrays("A1", A1, out)
    csr_arrays("Al", Al, out)
    for lvl in levels:
        p0 = ref.spai_pattern(A1, level=lvl, max_fill_per_column=max_fill)
        pattern_arrays("pat%d" % lvl, p0.columns, out)
        P, st = ref.spai_build(A1, SpaiConfig(pattern_level=lvl, max_fill_per_column=max_fill))
        csr_arrays("P%d" % lvl, P.matrix, out)
        stats_arrays("P%d" % lvl, st, out)
        if not update:
            continue
        Pu, stu = ref.update_first(A1, Al, P, UpdateConfig(pattern_level=lvl,
                                                            max_fill_per_column=max_fill))
        csr_arrays("Q%d" % lvl, Pu.q, out)
        stats_arrays("Q%d" % lvl, stu, out)
    lvl0 = ref.spai_pattern(A1, level=0)
    pattern_arrays("J0", touched(A1, lvl0.columns, ref.sparsecore.identity_csr(n)), out)
    if not update:
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print("wrote", name, n, A1.nnz)
        return
    lvl0u = ref.spai_pattern(Al, level=0)
    pattern_arrays("J0u", touched(Al, lvl0u.columns, A1), out)
    if solve and B is not None:
        out["B"] = np.asarray(B, dtype=float)
        P0, _ = ref.spai_build(A1, SpaiConfig(pattern_level=0))
        for tag, A, P in (("s1", A1, P0),
                          ("s2", Al, ref.update_first(A1, Al, P0, UpdateConfig(pattern_level=0))[0]),
                          ("nop", Al, None)):
            X, rep = ref.block_gcro_solve(A, B, P=P, cfg=SolverConfig(tol=1e-8))
            out[tag + "_X"] = X.real.copy()
            out[tag + "_Ximag"] = np.array(np.abs(X.imag).max())
            out[tag + "_iters"] = np.array(rep.iterations)
            out[tag + "_conv"] = np.array(rep.converged)
            out[tag + "_hist"] = np.array([np.asarray(h, dtype=float) for h in rep.residual_history])
            out[tag + "_matvec"] = np.array(rep.matvec_count)
            out[tag + "_papply"] = np.array(rep.precond_apply_count)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print("wrote", name, n, A1.nnz, sum(v.nbytes for v in out.values()))


def workload_case(name, cfg, scale, n_assemble=3, systems=(0, 1)):
    W = make_config(cfg, scale=scale)
    model = SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                      rhs=W.rhs)
    pts = W.points()
    out = {}
    # assembly golden: first n_assemble systems in pmor_l_sequence order
    for i, (s, p) in enumerate(pts[:n_assemble]):
        csr_arrays("asm%d" % i, model.assemble(s, p), out)
        out["asm%d_point" % i] = np.concatenate([[s], p])
    np.savez_compressed(os.path.join(HERE, name + "_assemble.npz"), **out)
    A1 = model.assemble(*pts[systems[0]])
    Al = model.assemble(*pts[systems[1]])
    build_case(name, A1, Al, B=W.rhs, levels=(0, 1))


def unit_cases():
    # reference unit-test shapes with real values (the reference
    # tests default to complex; the assertions are reused on real inputs)
    rs = np.random.RandomState(7)
    A = sp.random(40, 40, density=0.15, random_state=rs, format="csr") + 2.0 * sp.identity(40)
    E = sp.random(40, 40, density=0.05, random_state=np.random.RandomState(57), format="csr")
    B = np.random.default_rng(8).standard_normal((40, 3))
    build_case("rand40", A, A + 1e-2 * E, B=B, levels=(0, 1), max_fill=12)
    n = 9
    T = sp.diags([np.ones(n - 1), 2 * np.ones(n), np.ones(n - 1)], offsets=(-1, 0, 1))
    build_case("tridiag9", T, 1.5 * T, B=np.ones((n, 1)), levels=(0, 1), max_fill=50)
    D = sp.csr_matrix(np.array([[1.0, 0.0], [0.0, 0.0]]))
    # update_first on this pair makes the reference itself raise (empty target
    # column and empty touched-row set: spai.py:241-242 returns 0 coefficients
    # for a 1-entry support, and the COO build at spai.py:307 rejects the
    # length mismatch) -- so only the SPAI build is pinned here.
    build_case("degenerate2", D, D, levels=(0,), solve=False, update=False)


if __name__ == "__main__":
    unit_cases()
    workload_case("c1s24", 1, 24)
    workload_case("c2s8", 2, 8)
    workload_case("c3s6", 3, 6)
    workload_case("c5n500", 5, 500)
