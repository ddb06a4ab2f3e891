"""Golden fixture for the moment pipeline: the REAL
reference ``pmorprec.rpmor.rpmor_reduce`` on a seeded real affine family
(12 x 12 grid Laplacian + parameter terms), two expansion points, one moment
level, update-first SPAI preconditioning (level-0 patterns).

    OPENBLAS_NUM_THREADS=1 PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_rpmor_golden.py

Writes tests/golden/rpmor_small.npz (family, basis, reduced model, per-call
iteration counts, transfer-function samples).  Only runs where
/root/reference exists; the .npz travels to the GPU box.
"""

import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from pmorprec.affine import AffineFamily, ExpansionPoint   # noqa: E402
from pmorprec.krylov import SolverConfig                   # noqa: E402
from pmorprec.rpmor import PrecondPolicy, rpmor_reduce     # noqa: E402
from pmorprec.spai import SpaiConfig                       # noqa: E402
from pmorprec.update import UpdateConfig                   # noqa: E402

from paper_1809_06574_b200.workloads import grid_laplacian  # noqa: E402


def family_arrays(seed=21, nx=12):
    rng = np.random.default_rng(seed)
    K0 = grid_laplacian((nx, nx), "star", rng, 0.5)
    n = K0.shape[0]
    A0 = (K0 + sp.identity(n)).tocsr()
    A1 = sp.diags(rng.uniform(0.0, 1.0, n)).tocsr()
    K1 = grid_laplacian((nx, nx), "star", rng, 0.3)
    A2 = (0.1 * K1).tocsr()
    B = rng.standard_normal((n, 2))
    C = rng.standard_normal((n, 2))
    return [A0, A1, A2], B, C


POINTS = [(0.5, 0.2), (1.5, 0.7)]
QUERIES = [(0.5, 0.2), (1.0, 0.4), (1.5, 0.7), (2.0, 1.0)]


def main():
    terms, B, C = family_arrays()
    fam = AffineFamily(terms, rhs=B, output=C)
    pol = PrecondPolicy(kind="spai-update-first", spai=SpaiConfig(pattern_level=0),
                        update=UpdateConfig(pattern_level=0))
    pts = [ExpansionPoint(np.array(p), label="p%d" % i) for i, p in enumerate(POINTS)]
    red, rep = rpmor_reduce(fam, pts, levels=1, solver_cfg=SolverConfig(tol=1e-10),
                            policy=pol)
    out = {}
    for j, T in enumerate(terms):
        T = sp.csr_matrix(T)
        out["t%d_indptr" % j], out["t%d_indices" % j], out["t%d_data" % j] = \
            T.indptr, T.indices, T.data
    out["B"], out["C"], out["points"], out["queries"] = B, C, np.array(POINTS), np.array(QUERIES)
    assert np.abs(red.basis.imag).max() == 0.0
    out["basis"] = red.basis.real
    for j, T in enumerate(red.terms):
        out["red_t%d" % j] = T.real
    out["red_rhs"], out["red_out"] = red.rhs.real, red.output.real
    out["iters"] = np.array([r.iterations for r in rep.records])
    out["n_rhs"] = np.array([r.n_rhs for r in rep.records])
    out["levels"] = np.array([r.level for r in rep.records])
    H = np.stack([red.transfer(ExpansionPoint(np.array(q))) for q in QUERIES])
    assert np.abs(H.imag).max() < 1e-12
    out["transfer"] = H.real
    # full-model transfer function (dense, reference's oracle scale)
    Hf = []
    for q in QUERIES:
        A = (terms[0] + q[0] * terms[1] + q[1] * terms[2]).toarray()
        Hf.append(C.T @ np.linalg.solve(A, B))
    out["transfer_full"] = np.stack(Hf)
    np.savez_compressed(os.path.join(HERE, "rpmor_small.npz"), **out)
    print("basis", red.basis.shape, "iters", out["iters"], "max |H_red - H_full|",
          np.abs(out["transfer"] - out["transfer_full"]).max())


if __name__ == "__main__":
    main()
