"""The two pure-streaming kernels of the path at c4 size, timed with CUDA
events against their algorithmic bytes: multi-system
assembly (k_assemble_multi: term values read once, 16 systems written) and
the standalone CSR SpMM (k_spmm: Y = A X, n x 8 block).  Also the target of
tools/gpu_ncu_stream.sh.  Diagnostic only.

    python tools/stream_kernels.py [--config 4]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1809_06574_b200 as pm  # noqa: E402
from paper_1809_06574_b200.workloads import make_config  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    a = ap.parse_args()
    W = make_config(a.config)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pts = W.points()[:17]
    A1 = model.assemble(*pts[0])
    n, nnz = A1.n, A1.nnz
    k = len(pts) - 1
    t = timeit(lambda: model.assemble_many(pts[1:]))
    # union-expanded terms (8 B per entry) + diagonal terms (8 B per row) read
    # once per launch, one 8 B value per entry and system written
    nt_full = sum(1 for kd in model._union().kinds if kd == 0)
    nt_diag = sum(1 for kd in model._union().kinds if kd == 1)
    byts = 8.0 * nnz * nt_full + 8.0 * n * nt_diag + 8.0 * nnz * k + 8.0 * nnz
    print("assemble_many: %d systems, n = %d, nnz = %d: %.3f ms, %.1f GB/s algorithmic "
          "(%d union + %d diagonal terms + row / column ids read, %d outputs written)"
          % (k, n, nnz, t * 1e3, byts / t / 1e9, nt_full, nt_diag, k))
    X = torch.randn(n, 8, dtype=torch.float64, device="cuda")
    P = pm.Preconditioner(matrix=A1)
    t = timeit(lambda: P.apply(X))
    byts = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n * 8
    print("spmm (Preconditioner.apply, n x 8): %.3f ms, %.1f GB/s algorithmic" % (t * 1e3, byts / t / 1e9))


if __name__ == "__main__":
    main()
