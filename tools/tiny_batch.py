"""Persistent solve kernel (pmp_solve_batch) at tiny sizes against the
host-driven path: n in {24, 40, 64, 100, 256}, s in {1, 3, 4}, 1-3 block
groups.  Diagnostic (each case in a subprocess so a fault is reported, not
fatal)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = r'''
import sys, numpy as np, scipy.sparse as sp, torch
sys.path.insert(0, %r)
import paper_1809_06574_b200 as pm
from paper_1809_06574_b200 import krylov
n, s, groups, prec = %d, %d, %d, %d
rs = np.random.RandomState(7)
A = sp.random(n, n, density=min(1.0, 4.0 / n), random_state=rs, format="csr") + 4.0 * sp.identity(n)
A = sp.csr_matrix(A)
B = np.random.default_rng(3).standard_normal((n, s))
P = None
if prec:
    P, _ = pm.spai_build(A, pm.SpaiConfig(pattern_level=0))
Ad = krylov._as_dev_csr(A)
Bd = torch.as_tensor(B, device="cuda")
cfg = pm.SolverConfig(tol=1e-10)
res = krylov.block_gcro_solve_batch([(Ad, P)] * groups, Bd, cfg=cfg, groups=groups)
torch.cuda.synchronize()
Xh, rh = pm.block_gcro_solve(A, B, P=P, cfg=cfg)
for X, r in res:
    X = X.cpu().numpy()
    rel = np.linalg.norm(B - A @ X, axis=0) / np.linalg.norm(B, axis=0)
    assert r.converged and rel.max() <= 1e-9, (r.converged, rel)
    assert abs(r.iterations - rh.iterations) <= 2, (r.iterations, rh.iterations)
print("ok", res[0][1].iterations, rh.iterations, dict(krylov.FALLBACK_REASONS))
'''


def main():
    bad = 0
    quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
    for n in ((24, 40) if quick else (24, 40, 64, 100, 256)):
        for s in ((3, 4) if quick else (1, 3, 4)):
            for groups in ((1, 3) if quick else (1, 2, 3)):
                for prec in (0, 1):
                    code = CASE % (ROOT, n, s, groups, prec)
                    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                                       timeout=300)
                    out = (p.stdout.strip().splitlines() or [""])[-1]
                    if p.returncode != 0:
                        bad += 1
                        err = [l for l in p.stderr.splitlines() if "Error" in l or "error" in l][-1:]
                        out = "FAIL rc=%d %s" % (p.returncode, err)
                    print("n=%d s=%d groups=%d prec=%d: %s" % (n, s, groups, prec, out), flush=True)
    print("failures:", bad)


if __name__ == "__main__":
    main()
