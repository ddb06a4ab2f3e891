import cProfile, pstats, sys, os, io
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1809_06574_b200 as pm
from paper_1809_06574_b200.workloads import make_config
W = make_config(2)
model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms, rhs=W.rhs)
pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=0), update=pm.UpdateConfig(pattern_level=0))
cfg = pm.SolverConfig(tol=1e-8)
Bd = torch.as_tensor(W.rhs, device="cuda")
for _ in range(3):
    pm.run_sequence(model, W.s_grid, W.p_grid, pol, cfg, B=Bd, batch=6)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(3):
    pm.run_sequence(model, W.s_grid, W.p_grid, pol, cfg, B=Bd, batch=6)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25); print(s.getvalue()[:6000])
