"""Golden persistence fixture: the REAL reference ``pmorprec`` builds a SPAI at
the first c1 system (16 x 16 grid) and an update-first factor for the second,
then saves the chain with its own ``Preconditioner.save`` (spai.py:103-117)
into tests/golden/precond_ref/.  Also stores the block the reference applied
the chain to and the result (``apply.npz``), so the device path can check
``Preconditioner.load`` + ``apply`` against the reference's own numbers.

    OPENBLAS_NUM_THREADS=1 PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_precond_golden.py

Only runs where /root/reference exists (the build container); the outputs
are committed and travel to the GPU box.
"""

import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import pmorprec as ref                                   # noqa: E402
from pmorprec.spai import SpaiConfig                     # noqa: E402
from pmorprec.update import UpdateConfig                 # noqa: E402
from pmorprec.rpmor import SecondOrderModel              # noqa: E402

from paper_1809_06574_b200.workloads import make_config  # noqa: E402


def main():
    W = make_config(1, scale=16)
    model = SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                      rhs=W.rhs)
    pts = W.points()
    A1 = model.assemble(*pts[0])
    A2 = model.assemble(*pts[1])
    P1, _ = ref.spai_build(A1, SpaiConfig(pattern_level=0))
    P2, st = ref.update_first(A1, A2, P1, UpdateConfig(pattern_level=0))
    out = os.path.join(HERE, "precond_ref")
    shutil.rmtree(out, ignore_errors=True)
    P2.save(out)
    V = np.random.default_rng(11).standard_normal((W.n, 3))
    Y = P2.apply(V)
    assert np.abs(Y.imag).max() == 0.0
    np.savez_compressed(os.path.join(out, "apply.npz"), V=V, Y=Y.real, n=W.n)
    print("wrote", out, sorted(os.listdir(out)))


if __name__ == "__main__":
    main()
