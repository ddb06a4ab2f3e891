import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1809_06574_b200 as pm
from paper_1809_06574_b200 import krylov
import goldens as G
g = G.load("c1s24")
A1, Al, B = G.csr(g, "A1"), G.csr(g, "Al"), g["B"]
P0, _ = pm.spai_build(A1, pm.SpaiConfig(pattern_level=0))
Bd = torch.as_tensor(B, device="cuda")
for mi in (1, 2, 3, 30):
    cfg = pm.SolverConfig(tol=1e-8, max_iters=mi)
    (X, rep), = pm.block_gcro_solve_batch([(A1, P0)], Bd, cfg=cfg, groups=1)
    krylov.DEVICE_CYCLE = False
    Xh, rh = pm.block_gcro_solve(A1, Bd, P=P0, cfg=cfg)
    krylov.DEVICE_CYCLE = True
    Xc, rc = pm.block_gcro_solve(A1, Bd, P=P0, cfg=cfg)
    print("max_iters", mi, "iters", rep.iterations, rh.iterations, rc.iterations)
    print("  dev   hist", [np.round(r, 4).tolist() for r in rep.residual_history[:4]])
    print("  host  hist", [np.round(r, 4).tolist() for r in rh.residual_history[:4]])
    print("  |X-Xh|", float((X - Xh).abs().max()), "|Xc-Xh|", float((Xc - Xh).abs().max()))
