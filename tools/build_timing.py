"""GPU-only time of the SPAI-update builds of a c2 window, with the host kept
ahead of the device (a long spin kernel first, so every launch is already
queued when the device reaches it), next to the same loop timed normally
(host enqueue overhead included).  Diagnostic only.

    python tools/build_timing.py [--config 2] [--systems 16]
"""
import argparse
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1809_06574_b200 as pm  # noqa: E402
from paper_1809_06574_b200.workloads import make_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--systems", type=int, default=16)
    a = ap.parse_args()
    W = make_config(a.config)
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    pts = W.points()[:a.systems + 1]
    A1 = model.assemble(*pts[0])
    P1, _ = pm.spai_build(A1, pm.SpaiConfig(pattern_level=0))
    As = model.assemble_many(pts[1:])
    cfg = pm.UpdateConfig(pattern_level=0)
    for A in As[:2]:
        pm.update_first(A1, A, P1, cfg)
    torch.cuda.synchronize()

    def run():
        return [pm.update_first(A1, A, P1, cfg) for A in As]

    # host-bound: plain loop
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    run()
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    plain = e0.elapsed_time(e1)
    host = (t1 - t0) * 1e3
    # device-bound: a spin kernel keeps the device busy while the host enqueues
    torch.cuda._sleep(int(2e9 * (host / 1e3) + 2e7))
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1)
    n = len(As)
    print("updates: %d systems, n=%d: host enqueue %.3f ms (%.1f us/system); plain %.3f ms; "
          "device-only %.3f ms (%.1f us/system)" % (n, A1.n, host, 1e3 * host / n, plain, dev,
                                                    1e3 * dev / n))


if __name__ == "__main__":
    main()
