"""Per-system solve goldens for the BENCHMARKED sequences, produced by the
REAL reference ``pmorprec`` (importable only in the build container, from
/root/reference/pkg/src) on the seeded BASELINE generators.

    OPENBLAS_NUM_THREADS=1 PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_sequence_golden.py c2 [--procs 6] [--systems 0,1,2]

For every requested system of the config's pmor_l_sequence order
(zoo.py:268-284) it records what the reference's sequence driver
(rpmor.py:199-218, first approach: system 0 gets spai_build, every other
system update_first against (A_0, P_0)) and ``block_gcro_solve(A, B, P,
SolverConfig(tol=1e-8))`` (krylov.py:105-275) return: iterations,
converged, per-column final residuals, matvec / precond-apply counts, the
update's residual statistics, and per-column norms of X.

Parallelism only splits work the reference itself treats as independent:
the factor columns are built by the reference's own ``_build_columns``
(spai.py:273-292) over contiguous column chunks in forked processes and
assembled by its ``_assemble_and_stats`` (spai.py:295-315) -- the per-column
results are deterministic, so this is bit-identical to ``spai_build`` /
``update_first`` with threads=1 -- and each system's solve runs in its own
process with one BLAS thread.

Output: tests/golden/seq_<cfg>.json (scalars only; small).  Nothing on the
GPU box reads /root/reference; only the JSON travels.
"""

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import pmorprec as ref                                               # noqa: E402
from pmorprec.spai import (SpaiConfig, Preconditioner, spai_pattern,   # noqa: E402
                           _build_columns, _assemble_and_stats)
from pmorprec.sparsecore import identity_csr                         # noqa: E402
from pmorprec.update import UpdateConfig                             # noqa: E402
from pmorprec.krylov import SolverConfig                             # noqa: E402
from pmorprec.rpmor import SecondOrderModel                          # noqa: E402

from paper_1809_06574_b200.workloads import make_config              # noqa: E402

G = {}          # fork-inherited state


def _cols_chunk(cols):
    A_csc, T_csc, pattern, cfg = G["job"]
    return _build_columns(A_csc, T_csc, pattern, cfg, None, cols)


def build_factor(pool, system, targets, procs):
    """spai_build(system) (targets = I) or _solve_factor(targets, system)
    at pattern level 0, column chunks over the pool (spai.py:318-338)."""
    system = ref.as_csr(system)
    n = system.shape[0]
    pattern = spai_pattern(system, level=0)
    cfg = SpaiConfig(pattern_level=0)
    G["job"] = (system.tocsc(), ref.as_csr(targets).tocsc(), pattern, cfg)
    t0 = time.perf_counter()
    chunks = np.array_split(np.arange(n), procs * 4)
    with mp.get_context("fork").Pool(procs) as p:
        parts = p.map(_cols_chunk, chunks)
    results = [r for part in parts for r in part]
    results.sort(key=lambda r: r[0])
    return _assemble_and_stats(n, results, t0)


def _solve_one(i):
    A, P = G["systems"][i]
    B = G["B"]
    t0 = time.perf_counter()
    X, rep = ref.block_gcro_solve(A, B, P=P, cfg=SolverConfig(tol=1e-8))
    R = B - A @ X
    rel = np.linalg.norm(R, axis=0) / np.linalg.norm(B, axis=0)
    return {"index": int(i), "iterations": int(rep.iterations),
            "converged": bool(rep.converged),
            "final_residuals": [float(v) for v in rep.final_residuals],
            "true_rel_residuals": [float(v) for v in rel],
            "matvec_count": int(rep.matvec_count),
            "precond_apply_count": int(rep.precond_apply_count),
            "x_col_norms": [float(v) for v in np.linalg.norm(X, axis=0)],
            "x_imag_max": float(np.abs(X.imag).max()),
            "solve_s": time.perf_counter() - t0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--procs", type=int, default=6)
    ap.add_argument("--systems", default="all",
                    help="comma list of sequence indices, 'all', or 'stride:K'")
    ap.add_argument("--scale", type=int, default=0,
                    help="make_config's scale (a shrunken generator: grid side, or n for c5); "
                         "the golden is then seq_<cfg>s<scale>.json")
    args = ap.parse_args()
    cfgno = int(args.config[1])
    W = make_config(cfgno, scale=args.scale or None)
    pts = W.points()
    if args.systems == "all":
        idx = list(range(len(pts)))
    elif args.systems.startswith("stride:"):
        k = int(args.systems.split(":")[1])
        idx = list(range(0, len(pts), k))
    else:
        idx = [int(v) for v in args.systems.split(",")]
    if 0 not in idx:
        idx = [0] + idx
    model = SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                      rhs=W.rhs)
    t0 = time.perf_counter()
    A1 = ref.as_csr(model.assemble(*pts[0]))
    P1m, st1 = build_factor(None, A1, identity_csr(W.n), args.procs)
    P1 = Preconditioner(matrix=P1m)
    print("P1 built %.1f s nnz %d" % (time.perf_counter() - t0, P1m.nnz), flush=True)
    systems = {0: (A1, P1)}
    upd = {}
    for i in idx:
        if i == 0:
            continue
        t1 = time.perf_counter()
        A = ref.as_csr(model.assemble(*pts[i]))
        Q, stq = build_factor(None, A, A1, args.procs)
        systems[i] = (A, Preconditioner(q=Q, base=P1))
        r = np.asarray(stq.residuals)
        upd[i] = {"q_nnz": int(Q.nnz), "resid_sum": float(r.sum()), "resid_max": float(r.max()),
                  "augmented": int(stq.augmented_columns),
                  "deficient": int(stq.rank_deficient_columns),
                  "q_fro": float(sp.linalg.norm(Q))}
        print("update %d built %.1f s" % (i, time.perf_counter() - t1), flush=True)
    G["systems"] = systems
    G["B"] = np.asarray(W.rhs, dtype=np.complex128)
    with mp.get_context("fork").Pool(args.procs) as p:
        recs = p.map(_solve_one, idx, chunksize=1)
    for r in recs:
        r.update(upd.get(r["index"], {}))
        r["sigma"] = float(pts[r["index"]][0])
        r["p"] = [float(v) for v in pts[r["index"]][1]]
    r1 = np.asarray(st1.residuals)
    out = {"config": args.config, "scale": int(args.scale), "n": int(W.n), "n_systems": len(pts),
           "systems": idx, "records": recs,
           "p1": {"nnz": int(P1m.nnz), "resid_sum": float(r1.sum()),
                  "resid_max": float(r1.max()), "fro": float(sp.linalg.norm(P1m))},
           "reference": "pmorprec (real reference, /root/reference/pkg/src)",
           "numpy": np.__version__, "scipy": __import__("scipy").__version__,
           "solver": "SolverConfig(tol=1e-8)", "policy": "spai-update-first, pattern_level=0",
           "seconds": time.perf_counter() - t0}
    path = os.path.join(HERE, "seq_%s%s.json" % (args.config,
                                                 ("s%d" % args.scale) if args.scale else ""))
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    its = [r["iterations"] for r in recs]
    print("wrote", path, "iterations min %d max %d mean %.4f" % (min(its), max(its),
                                                                 float(np.mean(its))))


if __name__ == "__main__":
    main()
