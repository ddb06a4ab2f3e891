"""Run the first systems of a BASELINE config end to end on the device and
check every solution on the host (true relative residual <= tol).

    python tools/run_config.py --config 3 --systems 3 [--level 0]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1809_06574_b200 as pm  # noqa: E402
from paper_1809_06574_b200.workloads import make_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--systems", type=int, default=3)
    ap.add_argument("--level", type=int, default=0)
    ap.add_argument("--scale", type=int, default=0)
    a = ap.parse_args()
    t0 = time.time()
    W = make_config(a.config, scale=a.scale or None)
    print("generated c%d n=%d in %.1fs" % (a.config, W.n, time.time() - t0), flush=True)
    t0 = time.time()
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=a.level),
                           update=pm.UpdateConfig(pattern_level=a.level))
    cfg = pm.SolverConfig(tol=1e-8)
    s_grid, p_grid = W.s_grid[:1], W.p_grid[:a.systems]
    recs, info = pm.run_sequence(model, s_grid, p_grid, pol, cfg, keep_solutions=True)
    torch.cuda.synchronize()
    print("first run (incl. setup) %.2fs" % (time.time() - t0), flush=True)
    t0 = time.time()
    recs, info = pm.run_sequence(model, s_grid, p_grid, pol, cfg, keep_solutions=True)
    torch.cuda.synchronize()
    dt = time.time() - t0
    print("second run %.3fs  phases %s" % (dt, {k: round(v, 4) for k, v in info.items()}),
          flush=True)
    pts = [(s, np.atleast_1d(p)) for s in s_grid for p in p_grid]
    worst = 0.0
    for r in recs:
        A = model.assemble(*pts[r["index"]]).to_scipy()
        X = r["X"].cpu().numpy()
        rel = np.linalg.norm(W.rhs - A @ X, axis=0) / np.linalg.norm(W.rhs, axis=0)
        worst = max(worst, rel.max())
        print("system %d: iterations %d converged %s max true rel residual %.2e"
              % (r["index"], r["iterations"], r["converged"], rel.max()), flush=True)
    print("OK" if worst <= 1e-8 else "FAIL", "worst %.2e" % worst)


if __name__ == "__main__":
    main()
