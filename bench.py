"""Benchmark: the parametric SPAI / SPAI-update / block-GCRO sequence on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One step = one full pass of BASELINE config c2 (configs[1]):
for each of its 40 (sigma, p) systems in pmor_l_sequence order, assemble
A(sigma, p) = s^2 M(p) + s D(p) + K(p) on the device, build the SPAI
(system 1) or the SPAI update (systems 2..40, update_first), and solve the
n x 8 block to 1e-8 with block GCRO.  Inputs (the model's terms and B) are
resident in HBM when the timed region starts; the L2 (126 MB > the c2
working set) is flushed before every step by writing a 256 MB buffer.

metric "SPAI(+update) columns/s": value = (n * systems) / sequence seconds,
i.e. SPAI + update columns delivered per second of the WHOLE sequence
(assembly + builds + solves); ms_per_step is the sequence time itself, the
other half of BASELINE.json's metric.  Build-only columns/s is reported as
"spai_update_columns_per_s".

--impl reference times the CPU oracle (oracle/pmor_oracle.py, a restatement
of the reference's numpy/scipy path, "port") on this host's cores: each
step is a bounded sample -- one update_first system (all n columns, column
chunks over a process pool) plus its block solve -- reported in the same
columns/s unit.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SPAI(+update) columns/s"
UNIT = "columns/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--systems", type=int, default=0, help="limit #systems (debug)")
    ap.add_argument("--workers", type=int, default=1,
                    help="host threads / CUDA streams driving independent systems "
                         "(per-system path, --batch 1)")
    ap.add_argument("--batch", type=int, default=6,
                    help="systems per persistent solve launch (1 = per-system path)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def workload(cfg, systems=0):
    from paper_1809_06574_b200.workloads import make_config
    W = make_config(cfg)
    pts = W.points()
    if systems:
        pts = pts[:systems]
    return W, pts


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# algorithmic bytes per launch of the dominant kernel families
def ls_flops(m, n):
    return 2.0 * m * n * n - (2.0 / 3.0) * n ** 3 + 4.0 * m * n - n * n


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1809_06574_b200 as pm
    from paper_1809_06574_b200 import _abi

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    W, pts = workload(args.config, args.systems)
    s_grid, p_grid = W.s_grid, W.p_grid
    if args.systems:
        s_grid, p_grid = W.s_grid[:1], W.p_grid[:args.systems]
    nsys = len(s_grid) * len(p_grid)
    n = W.n
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    level = W.pattern_level
    pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=level),
                           update=pm.UpdateConfig(pattern_level=level))
    cfg = pm.SolverConfig(tol=1e-8)
    Bd = torch.as_tensor(np.ascontiguousarray(W.rhs), device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        return pm.run_sequence(model, s_grid, p_grid, pol, cfg, B=Bd, rank=rank, world=world,
                               group=group, timing=True, workers=args.workers,
                               batch=args.batch)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        flush.zero_()
        step()
    barrier()
    clk = ClockSampler(local)
    clk.start()
    step_ms = []
    infos = []
    # per-kernel device time: "k_orth" = the fused orthogonalisation kernel
    # inside each native block step (events recorded in the C driver)
    dominant = ("pmp_solve_batch", "k_orth", "pmp_ls_columns", "pmp_ls_columns_planned", "pmp_fold", "pmp_gcro_cycle_end", "pmp_orth_step",
                "pmp_tsqr_r", "pmp_gram", "pmp_spmm", "pmp_tsmm", "pmp_copy_cols",
                "pmp_axpby_cols", "pmp_assemble", "pmp_permute", "pmp_permute_batch",
                "pmp_ls_columns_multi",
                "pmp_assemble_multi")
    _abi.count_launches(True)
    recs_all = None
    for k in range(args.steps):
        flush.zero_()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        recs, info = step()
        e1.record()
        barrier()
        step_ms.append(e0.elapsed_time(e1))
        infos.append(info)
        recs_all = recs
    launches = _abi.launches()
    counters = dict(_abi.COUNTERS)
    _abi.count_launches(False)
    clocks = clk.stop()
    # one extra, untimed step with CUDA events around every launch of the
    # candidate kernels (per-kernel device time and share of the step)
    flush.zero_()
    barrier()
    _abi.count_launches(True, timed=dominant)
    i0 = torch.cuda.Event(enable_timing=True)
    i1 = torch.cuda.Event(enable_timing=True)
    i0.record()
    # single stream, so each event pair brackets one kernel and nothing else
    recs_i, _ = pm.run_sequence(model, s_grid, p_grid, pol, cfg, B=Bd, rank=rank, world=world,
                                group=group, timing=True, workers=1, batch=args.batch)
    i1.record()
    barrier()
    instr_ms = i0.elapsed_time(i1)
    timed = dict(_abi.timed_events())
    _abi.count_launches(False)
    t_local = float(np.sum(step_ms))
    t = torch.tensor([t_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = n * nsys * args.steps / (total_ms / 1e3)

    # per-kernel device time over the timed region (events around each call)
    kern = {}
    for name, lst in timed.items():
        ms = [a.elapsed_time(b) for a, b, _ in lst]
        kern[name] = {"launches": len(ms), "total_ms": float(np.sum(ms)),
                      "avg_us": float(np.mean(ms) * 1e3) if ms else 0.0,
                      "share_of_step": float(np.sum(ms)) / instr_ms}
    build_s = float(np.mean([i["build_s"] for i in infos]))
    solve_s = float(np.mean([i["solve_s"] for i in infos]))
    asm_s = float(np.mean([i["assemble_s"] for i in infos]))
    cols = infos[-1]["build_columns"]
    iters = [r["iterations"] for r in recs_all]
    conv = all(r["converged"] for r in recs_all)

    roof = roofline(kern, timed, n, W, model, recs_i)
    roof_ls = roofline_ls(kern, model, nsys)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, pm, model, W, s_grid, p_grid, pol, cfg, rank, world, group, barrier)

    line = None
    if rank == 0:
        hbm, _ = peaks()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded generator, SURVEY.md 8.1)",
            "config": {"workload": "c%d" % args.config, "n": n, "systems": nsys,
                       "rhs_block": int(W.rhs.shape[1]), "pattern_level": level,
                       "precond": "spai-update-first", "tol": 1e-8,
                       "l2": "flushed before every step (256 MB write)",
                       "parallelism": "systems round-robin over %d GPU(s); %s" % (
                           world, ("%d systems per persistent solve launch" % args.batch)
                           if args.batch > 1 else "%d concurrent streams" % args.workers)},
            "sequence_s": ms_per_step / 1e3,
            "phases_s": {"assemble": asm_s, "build": build_s, "solve": solve_s},
            "spai_update_columns_per_s": cols / build_s if build_s > 0 else None,
            "iterations": {"min": int(min(iters)), "max": int(max(iters)),
                           "mean": float(np.mean(iters))},
            "converged": conv,
            "gpu_launches": int(launches),
            "gpu_launches_per_step": int(launches) // args.steps,
            "abi_calls": counters,
            "kernels": kern,
            "roofline": roof,
            "roofline_ls": roof_ls,
            "clocks": clocks,
        }
        if e2e is not None:
            line["e2e"] = e2e
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args, W, pts)
    if world > 1:
        dist.destroy_process_group()
    return line


def roofline(kern, timed, n, W, model, recs=None):
    """Dominant kernel vs its roofline.  Candidates: the persistent solve
    kernel and the n-sized Krylov kernels (HBM; algorithmic bytes) and the
    batched LS kernel (FP64 pipe)."""
    hbm, which = peaks()
    if not kern:
        return None
    name = max(kern, key=lambda k: kern[k]["total_ms"])
    lst = timed[name]
    st = model.structure
    nnz = st.nnz
    if name == "pmp_solve_batch":
        # the kernel accumulates its algorithmic bytes per system (solve.cu:
        # operator matrices once per application, [C | V] once per block
        # step, the n x s blocks it gathers / writes)
        tot = sum(r.get("algorithmic_bytes") or 0.0 for r in (recs or []))
        byts = [tot / max(len(lst), 1)] * len(lst)
    elif name == "k_orth":
        # [C | V] rows read once, W read, Q written: 8 n (k + total + 2 sb)
        byts = [8.0 * a[0] * (a[1] + a[2] + 2 * a[3]) for _, _, a in lst]
    elif name == "pmp_spmm":
        # 12 B per nnz + 4 (n+1) + 16 n s_b (X gathered once + Y written)
        byts = [12.0 * nnz + 4.0 * (n + 1) + 16.0 * n * a[4] for _, _, a in lst]
    elif name == "pmp_gram":
        byts = [8.0 * n * (a[1] + a[4]) for _, _, a in lst]
    elif name == "pmp_tsmm":
        byts = [8.0 * n * (a[1] + a[4] * (2 if a[7] != 0.0 else 1)) for _, _, a in lst]
    elif name == "pmp_tsqr_r":
        byts = [8.0 * n * a[1] for _, _, a in lst]
    else:
        byts = None
    ms = np.array([a.elapsed_time(b) for a, b, _ in lst])
    traffic = None
    try:
        tj = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                         "ncu_traffic.json")))
        if name in tj:
            # DRAM bytes of one launch from the committed ncu --set full capture
            traffic = tj[name]["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        pass
    if byts is not None:
        ach = float(np.sum(byts) / (np.sum(ms) / 1e3) / 1e9)
        return {"kernel": name, "bound": "hbm", "achieved": ach, "peak": hbm,
                "unit": "GB/s", "frac": ach / hbm, "traffic": traffic,
                "algorithmic_bytes_per_launch": float(np.mean(byts)),
                "peak_source": which + " (MEASURED_PEAKS.json hbm_gbs)",
                "launches": len(lst), "avg_us": kern[name]["avg_us"],
                "share_of_step": kern[name]["share_of_step"]}
    # LS kernel: FP64 flops of the Householder solves
    fp64_peak = 148 * 64 * 2 * 1.965e9 / 1e12
    return {"kernel": name, "bound": "fp64", "achieved": None, "peak": fp64_peak,
            "unit": "TFLOP/s", "frac": None, "traffic": None,
            "peak_source": "nominal FP64 (148 SM x 64 DFMA/clk x 1.965 GHz)"}


def roofline_ls(kern, model, nsys):
    """Secondary roofline: the batched least-squares kernels (SPAI base build
    + all update builds of the step) against the FP64 pipe.  Algorithmic
    flops per column F_j = 2 m n^2 - 2/3 n^3 + 4 m n - n^2 (m = |J_j|,
    n = |I_j|, level-0 patterns: I_j = rows(A(:, j)), J_j = rows(A(:, I_j)),
    the same for the SPAI and every update of the sequence); nsys builds."""
    import scipy.sparse as sp
    names = [k for k in ("pmp_ls_columns_multi", "pmp_ls_columns_planned", "pmp_ls_columns")
             if k in kern]
    if not names:
        return None
    st = model.structure
    Ab = sp.csr_matrix((np.ones(st.nnz), st.colidx.cpu().numpy(), st.rowptr.cpu().numpy()),
                       shape=(st.n, st.n))
    ni = Ab.getnnz(axis=0).astype(np.float64)
    mj = (Ab @ Ab).getnnz(axis=0).astype(np.float64)
    f_sys = float(np.sum(ls_flops(mj, ni)))
    t = sum(kern[k]["total_ms"] for k in names) / 1e3
    ach = nsys * f_sys / t / 1e12
    peak = 148 * 64 * 2 * 1.965e9 / 1e12
    return {"kernels": names, "bound": "fp64", "achieved": ach, "peak": peak,
            "unit": "TFLOP/s", "frac": ach / peak, "flops_per_build": f_sys, "builds": nsys,
            "seconds": t,
            "peak_source": "nominal FP64 (148 SM x 64 DFMA/clk x 2 x 1.965 GHz; "
                           "no measured FP64 peak in MEASURED_PEAKS.json)"}


def run_e2e(args, pm, model, W, s_grid, p_grid, pol, cfg, rank, world, group, barrier):
    """Same metric through the public API with host buffers: every step
    copies the model's term values and B host->device (pinned) and reads
    every solution back device->host."""
    import torch

    u = model._union()
    host_terms = [v.cpu().pin_memory() for v in u.vals]
    Bh = torch.as_tensor(np.ascontiguousarray(W.rhs)).pin_memory()
    Bd = torch.empty_like(Bh, device="cuda")
    nsys = len(s_grid) * len(p_grid)
    from paper_1809_06574_b200.sequence import owned_systems
    mine = owned_systems(nsys, rank, world, pol.kind)
    Xh = torch.empty((len(mine),) + tuple(W.rhs.shape), dtype=torch.float64).pin_memory()
    h2d = sum(t.numel() * 8 for t in host_terms) + Bh.numel() * 8
    d2h = Xh.numel() * 8
    times = []
    for k in range(args.warmup + args.steps):
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for hv, dv in zip(host_terms, u.vals):
            dv.copy_(hv, non_blocking=True)
        Bd.copy_(Bh, non_blocking=True)
        recs, _ = pm.run_sequence(model, s_grid, p_grid, pol, cfg, B=Bd, rank=rank, world=world,
                                  group=group, keep_solutions=True, timing=False,
                                  workers=args.workers, batch=args.batch)
        for i, r in enumerate(recs):
            Xh[i].copy_(r["X"], non_blocking=True)
        e1.record()
        barrier()
        if k >= args.warmup:
            times.append(e0.elapsed_time(e1))
    t = torch.tensor([float(np.sum(times))], dtype=torch.float64, device="cuda")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_s = float(t.item()) / 1e3
    return {"value": W.n * nsys * args.steps / total_s, "unit": UNIT,
            "ms_per_step": total_s * 1e3 / args.steps,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}


# ---------------------------------------------------------------------------
# CPU side (oracle port)
# ---------------------------------------------------------------------------

def _cpu_chunk(payload):
    import pmor_oracle as orc
    A1, A2, cols = payload
    return orc.update_factor(A1, A2, pattern_level=0, columns=cols)


def cpu_sample(W, pts, cores):
    """One update_first system (all columns, process pool over column
    chunks) + its block solve; returns seconds and the column count."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pmor_oracle as orc
    from concurrent.futures import ProcessPoolExecutor
    A1 = orc.assemble_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms, *pts[0])
    A2 = orc.assemble_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms, *pts[1])
    P1, _ = orc.spai_build(A1, pattern_level=0) if not hasattr(cpu_sample, "_P1") else \
        (cpu_sample._P1, None)
    cpu_sample._P1 = P1
    n = W.n
    t0 = time.perf_counter()
    chunks = np.array_split(np.arange(n), cores)
    if cores > 1:
        with ProcessPoolExecutor(cores) as ex:
            parts = list(ex.map(_cpu_chunk, [(A1, A2, c) for c in chunks]))
    else:
        parts = [_cpu_chunk((A1, A2, chunks[0]))]
    res = [r for p in parts for r in p]
    Q, _ = orc.assemble_columns(n, res)
    t1 = time.perf_counter()
    X, info = orc.block_gcro(A2, W.rhs, orc.Chain([Q, P1]), tol=1e-8)
    t2 = time.perf_counter()
    return t2 - t0, t1 - t0, t2 - t1, n, info["iterations"]


def cpu_baseline(args, W, pts):
    cores = max(1, len(os.sched_getaffinity(0)))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(cores))
    tot, tb, ts, n, it = cpu_sample(W, pts, cores)
    return {"value": n / tot, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": ("one update_first system of c%d (all %d columns over %d processes) + "
                       "its block GCRO solve to 1e-8 (%d iterations); build %.2f s, solve %.2f s"
                       % (args.config, n, cores, it, tb, ts))}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    W, pts = workload(args.config, args.systems)
    cores = max(1, len(os.sched_getaffinity(0)))
    times = []
    last = None
    for k in range(args.warmup + args.steps):
        tot, tb, ts, n, it = cpu_sample(W, pts, cores)
        last = (tb, ts, it)
        if k >= args.warmup:
            times.append(tot)
    value = n * args.steps / float(np.sum(times))
    ms = float(np.mean(times)) * 1e3
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, SURVEY.md 8.1)", "impl": "reference",
            "config": {"workload": "c%d" % args.config, "n": W.n, "systems": len(pts),
                       "pattern_level": 0, "precond": "spai-update-first", "tol": 1e-8},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": "per step: one update_first system (all %d columns, "
                                       "%d processes) + its block GCRO solve (%d iterations)"
                                       % (W.n, cores, last[2])},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    if args.impl == "reference":
        line = run_reference(args)
    else:
        line = run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
