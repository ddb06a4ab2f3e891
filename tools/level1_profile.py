"""Host profile of a pattern_level = 1 update_first (the reference's default
level, update.py:50) after one warm call: where the per-system time of the
level-1 path goes.  Diagnostic only.

    python tools/level1_profile.py [--config 4]
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
from paper_1809_06574_b200 import _abi  # noqa: E402
from paper_1809_06574_b200.workloads import make_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    a = ap.parse_args()
    W = make_config(a.config)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pts = W.points()
    A1 = model.assemble(*pts[0])
    As = [model.assemble(*p) for p in pts[1:4]]
    P1, st1 = pm.spai_build(A1, pm.SpaiConfig(pattern_level=1))
    print("spai level 1: augmented columns %d of %d" % (st1.augmented_columns, A1.n))
    cfg = pm.UpdateConfig(pattern_level=1)
    for A in As[:2]:
        t0 = time.perf_counter()
        Q, st = pm.update_first(A1, A, P1, cfg)
        torch.cuda.synchronize()
        print("update_first level 1: %.3f s, augmented %d" % (time.perf_counter() - t0,
                                                               st.augmented_columns))
    _abi.count_launches(True, timed=("pmp_ls_columns", "pmp_ls_columns_planned", "pmp_augment",
                                     "pmp_transpose", "pmp_ls_bound", "pmp_merge_columns"))
    pr = cProfile.Profile()
    pr.enable()
    t0 = time.perf_counter()
    pm.update_first(A1, As[2], P1, cfg)
    torch.cuda.synchronize()
    pr.disable()
    print("profiled update: %.3f s" % (time.perf_counter() - t0))
    for name, lst in _abi.timed_events().items():
        print("  %-26s %3d calls %9.3f ms" % (name, len(lst), sum(x.elapsed_time(y) for x, y, _ in lst)))
    _abi.count_launches(False)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(22)


if __name__ == "__main__":
    main()
