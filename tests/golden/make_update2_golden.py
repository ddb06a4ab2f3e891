"""update_second value golden (update.py:90-97, the second approach's chain
P_i = Q_i P_{i-1}) from the REAL reference on the c1 stencil at n = 576:
system 1 gets the SPAI, system 2 update_first, system 3 update_second
against system 2 (chain depth 3), and the block solve of system 3.

    OPENBLAS_NUM_THREADS=1 PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_update2_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import pmorprec as ref                                   # noqa: E402
from pmorprec.spai import SpaiConfig                     # noqa: E402
from pmorprec.update import UpdateConfig                 # noqa: E402
from pmorprec.krylov import SolverConfig                 # noqa: E402
from pmorprec.rpmor import SecondOrderModel              # noqa: E402

from paper_1809_06574_b200.workloads import make_config  # noqa: E402


def csr(prefix, M, out):
    M = ref.as_csr(M)
    out[prefix + "_indptr"] = M.indptr.astype(np.int64)
    out[prefix + "_indices"] = M.indices.astype(np.int64)
    out[prefix + "_data"] = M.data.real.copy()
    out[prefix + "_imagmax"] = np.array(np.abs(M.data.imag).max() if M.nnz else 0.0)
    out[prefix + "_shape"] = np.array(M.shape)


def main():
    W = make_config(1, scale=24)
    m = SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms, rhs=W.rhs)
    pts = W.points()
    A = [ref.as_csr(m.assemble(*pts[i])) for i in range(3)]
    out = {}
    for lvl in (0, 1):
        P1, _ = ref.spai_build(A[0], SpaiConfig(pattern_level=lvl))
        P2, _ = ref.update_first(A[0], A[1], P1, UpdateConfig(pattern_level=lvl))
        P3, st = ref.update_second(A[1], A[2], P2, UpdateConfig(approach="second",
                                                                 pattern_level=lvl))
        csr("Q%d" % lvl, P3.q, out)
        out["Q%d_resid" % lvl] = np.asarray(st.residuals)
        out["Q%d_aug" % lvl] = np.array(st.augmented_columns)
        X, rep = ref.block_gcro_solve(A[2], W.rhs, P=P3, cfg=SolverConfig(tol=1e-8))
        out["s%d_iters" % lvl] = np.array(rep.iterations)
        out["s%d_X" % lvl] = X.real.copy()
        out["depth%d" % lvl] = np.array(P3.depth)
    np.savez_compressed(os.path.join(HERE, "update2_c1s24.npz"), **out)
    print("wrote update2_c1s24", {k: out[k] for k in out if k.endswith("iters") or
                                   k.startswith("depth")})


if __name__ == "__main__":
    main()
