"""Per-phase timing of the persistent solve kernel (k_solve) for one batch
of c2 systems: %globaltimer stamps of group 0's lead worker, per block step
(pmp_cycle_debug_stamps).  Diagnostic only.

    python tools/solve_phases.py [--groups 4] [--config 2]
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

PH = ["spmm chain", "R1 gram", "R1 reduce", "R1 update", "R2 gram", "R2 reduce"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", type=int, default=4)
    ap.add_argument("--config", type=int, default=2)
    a = ap.parse_args()
    W = make_config(a.config)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pts = W.points()
    A1 = model.assemble(*pts[0])
    P1, _ = pm.spai_build(A1, pm.SpaiConfig(pattern_level=0))
    systems = []
    for pt in pts[1:1 + a.groups]:
        A = model.assemble(*pt)
        P, _ = pm.update_first(A1, A, P1, pm.UpdateConfig(pattern_level=0))
        systems.append((A, P))
    Bd = torch.as_tensor(W.rhs, device="cuda")
    cfg = pm.SolverConfig(tol=1e-8)
    for _ in range(2):
        pm.block_gcro_solve_batch(systems, Bd, cfg=cfg, groups=a.groups)
    torch.cuda.synchronize()
    buf = torch.zeros(4096 * 4, dtype=torch.int64, device="cuda")
    _abi.lib().pmp_cycle_debug_stamps(buf.data_ptr(), 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = pm.block_gcro_solve_batch(systems, Bd, cfg=cfg, groups=a.groups)
    e1.record()
    torch.cuda.synchronize()
    _abi.lib().pmp_cycle_debug_stamps(None, 0)
    print("batch of %d: %.3f ms; iterations %s" % (a.groups, e0.elapsed_time(e1),
                                                    [r.iterations for _, r in res]))
    alg = sum(getattr(r, "algorithmic_bytes", 0.0) for _, r in res)
    strict = sum(getattr(r, "algorithmic_bytes_strict", 0.0) for _, r in res)
    print("algorithmic bytes of the batch: %.6e (SURVEY 8(d) unit), %.6e (every operand once)"
          % (alg, strict))
    st = buf[:4096].view(64, 32, 2).cpu().numpy().astype(np.int64)[:, :, 1]
    rows = []
    for it in range(64):
        v = st[it]
        if v[0] and v[11]:
            rows.append(v)
    rows = np.array(rows, dtype=np.float64)
    print("steps recorded (group 0):", len(rows))
    if len(rows):
        step = (rows[:, 11] - rows[:, 0]) / 1e3
        print("  step median %.2f us" % np.median(step))
        for i, nm in enumerate(PH):
            d = (rows[:, i + 1] - rows[:, i]) / 1e3
            print("  %-12s %7.2f us" % (nm, np.median(d)))
        for nm, a_, b_ in (("GW", 6, 12), ("update2", 12, 13), ("symm", 13, 14), ("chol", 14, 7),
                           ("R3", 7, 8), ("trsm+Q+R", 8, 9), ("V barrier", 9, 10),
                           ("decision", 10, 11)):
            d = (rows[:, b_] - rows[:, a_]) / 1e3
            print("  %-12s %7.2f us" % (nm, np.median(d)))
        cyc = np.array([st[it][16] for it in range(64) if st[it][0] and st[it][11]], dtype=float)
        print("  chol call on warp 0: median %.0f cycles" % np.median(cyc))
        cs = buf[:4096].view(64, 32, 2).cpu().numpy().astype(np.int64)[48:64, :, 1]
        names = ["start orth", "gbar", "ctl init+gbar+inner", "inner->gbar", "cycle end",
                 "gbar", "fold", "gbar"]
        for c in range(16):
            v = cs[c]
            if not v[0]:
                continue
            parts = []
            for i, nm in enumerate(names):
                if v[i] and v[i + 1] and 0 <= v[i + 1] - v[i] < 10 ** 12:
                    parts.append("%s %.1f" % (nm, (v[i + 1] - v[i]) / 1e3))
            print("  cycle %d: %s" % (c, ", ".join(parts)))


if __name__ == "__main__":
    main()
