"""Per-phase timing of the orthogonalisation kernel (k_orth) from block 0's
%globaltimer stamps (pmp_orth_debug_stamps).  Diagnostic only.

    python tools/orth_phases.py [--systems 4] [--config 2]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1809_06574_b200 as pm  # noqa: E402
from paper_1809_06574_b200 import _abi  # noqa: E402
from paper_1809_06574_b200.workloads import make_config  # noqa: E402

PHASES = ["stage", "R1 gram", "R1 reduce", "R1 update", "R2 gram", "R2 reduce",
          "GW+update2", "chol", "R3 (trsm+gram+reduce+chol)", "final trsm+R"]


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
    cap = 20000
    buf = torch.zeros(16 * cap, dtype=torch.int64, device="cuda")
    _abi.lib().pmp_orth_debug_stamps(buf.data_ptr(), cap)
    pm.run_sequence(model, s_grid, p_grid, pol, cfg, B=Bd, timing=False)
    torch.cuda.synchronize()
    _abi.lib().pmp_orth_debug_stamps(None, 0)
    st = buf.view(cap, 16).cpu().numpy().astype(np.int64)
    st = st[st[:, 0] != 0]
    print("k_orth launches recorded: %d" % len(st))
    tot = np.where(st[:, 10] > 0, st[:, 10], st[:, 9]) - st[:, 0]
    print("block-0 span: median %.2f us  mean %.2f us" % (np.median(tot) / 1e3,
                                                          tot.mean() / 1e3))
    r3 = st[:, 9] > 0
    for i, name in enumerate(PHASES):
        a_, b_ = st[:, i], st[:, i + 1]
        ok = (a_ > 0) & (b_ > 0)
        if not ok.any():
            continue
        d = (b_[ok] - a_[ok]) / 1e3
        print("  %-28s n=%5d median %7.2f us  mean %7.2f us  p90 %7.2f" %
              (name, ok.sum(), np.median(d), d.mean(), np.percentile(d, 90)))
    print("launches with R3 stamp: %d" % r3.sum())


if __name__ == "__main__":
    main()
