"""Micro-benchmarks backing DESIGN.md numbers (diagnostic only):
grid-barrier cost of the cooperative kernels, kernel launch overhead."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1809_06574_b200 import _abi  # noqa: E402


def main():
    lib = _abi.load()
    st = torch.cuda.current_stream().cuda_stream
    for bps in (1, 2):
        for iters in (1, 100, 1000):
            for _ in range(3):
                _abi.check(lib.pmp_bench_grid_sync(bps, iters, st), "bench")
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                _abi.check(lib.pmp_bench_grid_sync(bps, iters, st), "bench")
            b.record()
            b.synchronize()
            ms = a.elapsed_time(b) / 10
            print("blocks/SM %d  iters %5d  kernel %.1f us  per-barrier %.2f us"
                  % (bps, iters, ms * 1e3, ms * 1e3 / iters))


if __name__ == "__main__":
    main()
