"""Host profile of the COLD symbolic path (pattern, LS plans, transposes):
spai_build + update_first on a freshly reset structure, under cProfile.

    python tools/cold_profile.py [--config 2]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1809_06574_b200 as pm  # noqa: E402
from paper_1809_06574_b200.workloads import make_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    a = ap.parse_args()
    W = make_config(a.config)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pts = W.points()
    pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=0),
                           update=pm.UpdateConfig(pattern_level=0))

    def cold():
        model.reset_symbolic()
        A1 = model.assemble(*pts[0])
        A2 = model.assemble(*pts[1])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P1, _ = pm.spai_build(A1, pol.spai)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        pm.update_first(A1, A2, P1, pol.update)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1

    for _ in range(2):
        print("cold spai %.4f s, update %.4f s" % cold())
    pr = cProfile.Profile()
    pr.enable()
    print("profiled: cold spai %.4f s, update %.4f s" % cold())
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
