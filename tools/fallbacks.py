"""Which systems of a sequence leave the device solve path, and why
(diagnostic).   python tools/fallbacks.py [--config 2] [--batch 4]"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1809_06574_b200 as pm  # noqa: E402
from paper_1809_06574_b200 import krylov  # noqa: E402
from paper_1809_06574_b200.workloads import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--batch", type=int, default=4)
ap.add_argument("--scale", type=int, default=0)
ap.add_argument("--systems", type=int, default=0)
a = ap.parse_args()
W = make_config(a.config, scale=a.scale or None)
model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms, rhs=W.rhs)
pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=0),
                       update=pm.UpdateConfig(pattern_level=0))
Bd = torch.as_tensor(W.rhs, device="cuda")
p_grid = W.p_grid[:a.systems] if a.systems else W.p_grid
recs, _ = pm.run_sequence(model, W.s_grid, p_grid, pol, pm.SolverConfig(tol=1e-8), B=Bd,
                          batch=a.batch, timing=False)
print("fallback reasons:", krylov.FALLBACK_REASONS)
print("iterations:", [r["iterations"] for r in recs])
