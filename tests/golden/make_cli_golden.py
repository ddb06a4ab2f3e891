"""Golden fixture for the experiment CLI: the REAL
reference saves a real affine family (the rpmor_small terms, three points)
with its own ``save_family`` into tests/golden/cli_family/ and runs its own
``run_experiment`` on it (block GCRO, update-first SPAI, one moment level);
the report is committed as tests/golden/cli_report.json.

    OPENBLAS_NUM_THREADS=1 PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_cli_golden.py

(run from the repo root: the config names the family directory by its
relative path, which enters the config hash and family fingerprint.)
"""

import json
import os
import shutil
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from pmorprec.affine import AffineFamily, ExpansionPoint, save_family   # noqa: E402
from pmorprec.cli import run_experiment                                # noqa: E402

CONFIG = {
    "model": {"family_dir": "tests/golden/cli_family"},
    "levels": 1,
    "solver": "block-gcro",
    "precond": "spai-update-first",
    "spai_config": {"pattern_level": 0},
    "update_config": {"pattern_level": 0},
    "solver_config": {"tol": 1e-10},
}


def main():
    g = np.load(os.path.join(HERE, "rpmor_small.npz"))
    terms = [sp.csr_matrix((g["t%d_data" % j], g["t%d_indices" % j], g["t%d_indptr" % j]))
             for j in range(3)]
    fam = AffineFamily(terms, rhs=g["B"], output=g["C"])
    pts = [ExpansionPoint(np.array(p), label="pt%d" % i)
           for i, p in enumerate([(0.5, 0.2), (0.8, 0.3), (1.5, 0.7)])]
    out = os.path.join(HERE, "cli_family")
    shutil.rmtree(out, ignore_errors=True)
    save_family(fam, out, points=pts)
    report, code, _, _ = run_experiment(CONFIG)
    assert code == 0
    with open(os.path.join(HERE, "cli_config.json"), "w") as fh:
        json.dump(CONFIG, fh, indent=2, sort_keys=True)
    with open(os.path.join(HERE, "cli_report.json"), "w") as fh:
        json.dump(report, fh, indent=2, sort_keys=True, default=float)
    print("records", len(report["records"]), "iterations",
          [r["iterations"] for r in report["records"]])


if __name__ == "__main__":
    main()
