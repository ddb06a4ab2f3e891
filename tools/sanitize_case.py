"""A small sequence through the benchmarked composition (k_assemble_multi,
k_ls_seg via pmp_ls_columns_multi, k_solve) for compute-sanitizer runs
(tools/gpu_sanitize.sh).  Diagnostic only."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1809_06574_b200 as pm  # noqa: E402
from paper_1809_06574_b200.workloads import make_config  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    W = make_config(1, scale=scale)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=0),
                           update=pm.UpdateConfig(pattern_level=0))
    recs, _ = pm.run_sequence(model, W.s_grid, W.p_grid, pol, pm.SolverConfig(tol=1e-8), batch=4,
                              keep_solutions=True)
    torch.cuda.synchronize()
    print("n = %d, systems %d, iterations %s, converged %s, fallbacks %s"
          % (model.dim, len(recs), [r["iterations"] for r in recs],
             all(r["converged"] for r in recs), pm.krylov.FALLBACK_REASONS))


if __name__ == "__main__":
    main()
