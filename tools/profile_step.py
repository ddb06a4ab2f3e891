"""Host/device time split of a few c2 systems: torch.profiler (CUPTI) kernel
timeline + cProfile of the host loop.  Diagnostic only.

    python tools/profile_step.py [--systems 4] [--config 2]
"""
import argparse
import cProfile
import os
import pstats
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
    ap.add_argument("--systems", type=int, default=4)
    ap.add_argument("--config", type=int, default=2)
    a = ap.parse_args()
    W = make_config(a.config)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=0),
                           update=pm.UpdateConfig(pattern_level=0))
    cfg = pm.SolverConfig(tol=1e-8)
    Bd = torch.as_tensor(W.rhs, device="cuda")
    s_grid, p_grid = W.s_grid[:1], W.p_grid[:a.systems]
    for _ in range(2):
        pm.run_sequence(model, s_grid, p_grid, pol, cfg, B=Bd, timing=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    recs, _ = pm.run_sequence(model, s_grid, p_grid, pol, cfg, B=Bd, timing=False)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    iters = sum(r["iterations"] for r in recs)
    print("wall %.2f ms for %d systems, %d iterations -> %.1f us/iteration"
          % (wall * 1e3, len(recs), iters, wall * 1e6 / iters))
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        pm.run_sequence(model, s_grid, p_grid, pol, cfg, B=Bd, timing=False)
        torch.cuda.synchronize()
    ka = prof.key_averages()
    tot = 0.0
    rows = []
    for e in ka:
        t = getattr(e, "device_time_total", None) or getattr(e, "cuda_time_total", 0)
        if t and e.key.startswith(("void pmp", "pmp", "void cub", "cub")) or "pmp::" in e.key:
            rows.append((t, e.count, e.key[:70]))
            tot += t
    rows.sort(reverse=True)
    print("device kernel time %.2f ms (%.0f%% of wall)" % (tot / 1e3, 100 * tot / 1e3 / (wall * 1e3)))
    for t, c, k in rows[:15]:
        print("  %-70s %6d  %9.1f us  %7.2f us/launch" % (k, c, t, t / max(c, 1)))
    # host wall per phase, synchronising after each (diagnostic only)
    from paper_1809_06574_b200 import krylov
    krylov.PROFILE.clear()
    ph = {"assemble": 0.0, "build": 0.0, "solve": 0.0}
    pts = [(s, np.atleast_1d(p)) for s in s_grid for p in p_grid]
    A1 = model.assemble(*pts[0])
    P1, _ = pm.spai_build(A1, pol.spai)
    torch.cuda.synchronize()
    for s_, p_ in pts[1:]:
        t = time.perf_counter()
        A = model.assemble(s_, p_)
        torch.cuda.synchronize()
        ph["assemble"] += time.perf_counter() - t
        t = time.perf_counter()
        P, _ = pm.update_first(A1, A, P1, pol.update)
        torch.cuda.synchronize()
        ph["build"] += time.perf_counter() - t
        t = time.perf_counter()
        pm.block_gcro_solve(A, Bd, P=P, cfg=cfg)
        torch.cuda.synchronize()
        ph["solve"] += time.perf_counter() - t
    print("host wall per phase (ms, %d systems):" % (len(pts) - 1),
          {k: round(v * 1e3, 2) for k, v in ph.items()})
    print("solver phases (ms, count):",
          {k: (round(v[0] * 1e3, 2), v[1]) for k, v in krylov.PROFILE.items()})
    pr = cProfile.Profile()
    pr.enable()
    pm.run_sequence(model, s_grid, p_grid, pol, cfg, B=Bd, timing=False)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
