"""Per-phase timing of the persistent cycle kernel (k_cycle) from the
%globaltimer stamps of blocks 0 (control) and 1 (worker)
(pmp_cycle_debug_stamps).  Diagnostic only.

    python tools/cycle_phases.py [--systems 4] [--config 2]
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

PH = ["spmm chain", "R1 gram", "R1 reduce", "R1 update", "R2 gram", "R2 reduce",
      "GW+upd2+chol", "R3", "trsm+Q", "ctl absorb", "decision barrier"]


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
    cap = 200
    buf = torch.zeros(4096 * cap, dtype=torch.int64, device="cuda")
    _abi.lib().pmp_cycle_debug_stamps(buf.data_ptr(), cap)
    pm.run_sequence(model, s_grid, p_grid, pol, cfg, B=Bd, timing=False)
    torch.cuda.synchronize()
    _abi.lib().pmp_cycle_debug_stamps(None, 0)
    st = buf.view(cap, 64, 32, 2).cpu().numpy().astype(np.int64)
    used = st[:, 63, 31, 0] != 0
    st = st[used]
    print("k_cycle launches recorded: %d" % len(st))
    tot = (st[:, 63, 29, 0] - st[:, 63, 31, 0]) / 1e3
    init = (st[:, 63, 30, 0] - st[:, 63, 31, 0]) / 1e3
    print("launch span (ctl block): median %.1f us; init %.1f us" % (np.median(tot),
                                                                       np.median(init)))
    for b, name in ((0, "control block"), (1, "worker block 1")):
        print(name)
        if b == 0:
            ab = []
            for L in st:
                for k in range(63):
                    if all(L[k, i, 0] for i in (16, 17, 18, 19)):
                        ab.append(np.diff(L[k, 16:20, 0].astype(np.float64)) / 1e3)
            if ab:
                ab = np.median(np.array(ab), axis=0)
                print("  absorb: old blocks %.2f  window factor %.2f  R/rank/est %.2f us" % tuple(ab))
            continue
        rows = []
        steps = []
        for L in st:
            for k in range(63):
                if L[k, 0, b] == 0 or L[k, 11, b] == 0:
                    continue
                d = np.diff(L[k, :12, b].astype(np.float64)) / 1e3
                rows.append(d)
                steps.append((L[k, 11, b] - L[k, 0, b]) / 1e3)
        rows = np.array(rows)
        sub = []
        r3 = 0
        for L in st:
            for k in range(63):
                v = L[k, [6, 12, 13, 14, 7], b]
                if all(v):
                    sub.append(np.diff(v.astype(np.float64)) / 1e3)
                if L[k, 0, b] and L[k, 15, b] == 1:
                    r3 += 1
        if sub:
            print("  GW %.2f  update2 %.2f  symm %.2f  chol %.2f us; steps with R3 pass: %d" %
                  (tuple(np.median(np.array(sub), axis=0)) + (r3,)))
        print("  steps %d, step median %.2f us" % (len(steps), np.median(steps)))
        a = []
        bb = []
        for L in st:
            for k in range(63):
                if L[k, 0, b] and L[k, 12, b] and L[k, 13, b]:
                    a.append((L[k, 12, b] - L[k, 0, b]) / 1e3)
                    bb.append((L[k, 13, b] - L[k, 12, b]) / 1e3)
        if a:
            print("  first spmm (+absorb) median %.2f us, its barrier %.2f us" % (np.median(a),
                                                                            np.median(bb)))
        if b == 0:
            # absorb sub-phases (stamped by block index q of the absorbed step)
            ab = []
            for L in st:
                for k in range(63):
                    if all(L[k, i, 0] for i in (16, 17, 18, 19)):
                        ab.append(np.diff(L[k, 16:20, 0].astype(np.float64)) / 1e3)
            if ab:
                ab = np.median(np.array(ab), axis=0)
                print("  absorb: old blocks %.2f  window factor %.2f  R/rank/est %.2f us" % tuple(ab))
            fj = []
            for L in st:
                for k in range(63):
                    v = L[k, [17, 28] + list(range(20, 28)), 0]
                    if all(v):
                        fj.append(np.diff(v.astype(np.float64)) / 1e3)
            if fj:
                print("  window: load, j0..j7:", " ".join("%.2f" % x for x in np.median(np.array(fj), axis=0)))
        for i, nm in enumerate(PH):
            col = rows[:, i]
            col = col[col >= 0]
            print("  %-18s median %7.2f  mean %7.2f  p90 %7.2f" % (nm, np.median(col), col.mean(),
                                                                 np.percentile(col, 90)))


if __name__ == "__main__":
    main()
