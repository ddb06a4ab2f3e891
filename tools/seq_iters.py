"""Per-system iteration counts of a config's sequence (diagnostic)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1809_06574_b200 as pm  # noqa: E402
from paper_1809_06574_b200.workloads import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
W = make_config(cfg)
model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms, rhs=W.rhs)
pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=0),
                       update=pm.UpdateConfig(pattern_level=0))
recs, info = pm.run_sequence(model, W.s_grid, W.p_grid, pol, solver_cfg=pm.SolverConfig(tol=1e-8))
for r in recs:
    print(r["index"], "sigma %.3g p %s iters %d" % (r["sigma"], r["p"], r["iterations"]))
