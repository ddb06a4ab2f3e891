"""Benchmark: the parametric SPAI / SPAI-update / block-GCRO sequence on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

Workload (default): BASELINE config c4 (configs[3], the largest one that
fits one GPU): 3D 128^3 grid, n = 2,097,152, 512 (sigma, p)
systems in pmor_l_sequence order, B n x 8.  One step = one COLD pass of
the whole sequence: the model's symbolic caches (level-0 pattern, its
transpose plan, the least-squares size plans and recorded symbolic plans)
are dropped first, so every step pays them again, as a new sequence does;
then every system is assembled on the device, system 1 gets the SPAI and
systems 2..512 the SPAI update (update_first), and every n x 8 block is
solved to 1e-8 by block GCRO.  Inputs (the model's term values and B) are
resident in HBM when the timed region starts; the working set (tens of GB)
is far larger than the 126 MB L2, and the L2 is also flushed before every
step by writing a 256 MB buffer.

metric "SPAI(+update) columns/s": value = (n * systems) / sequence seconds
-- SPAI + update columns delivered per second of the WHOLE sequence
(assembly + builds + solves); ms_per_step is the cold sequence time, the
other half of BASELINE.json's metric.  Also reported:
``spai_columns_per_s`` = n / spai_build time (device A -> device P, cold:
pattern, plan and transpose included), ``update_columns_per_s`` = n /
update_first time (one system), ``update_window_columns_per_s`` (the
sequence's batched update_first_many), ``warm_ms_per_step`` (symbolic
caches kept).

Multi-GPU: ``--gpus N`` without a torchrun environment re-executes itself
under ``torch.distributed.run`` with N ranks.  Systems are dealt
round-robin over the ranks (fixed total work: "scaling": "strong"), the base
SPAI is built column-sharded and all-gathered over NCCL (pmp_nccl_*), the
per-system records are summed over ranks; the step time is the max over
ranks of CUDA-event time.

--impl reference: the CPU oracle (oracle/pmor_oracle.py, a restatement of
the reference's numpy/scipy path: "port") on this host's cores, on the same
config / metric, each step a bounded sample (see ``cpu_sample``):
extrapolated to the whole sequence and labelled so.
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
CPU_SAMPLE_COLUMNS = 20000


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2,
                    help="timed end-to-end steps (after one warm-up step)")
    ap.add_argument("--warm", action="store_true", default=True,
                    help="also time one step with the symbolic caches kept")
    ap.add_argument("--no-warm", dest="warm", action="store_false")
    ap.add_argument("--systems", type=int, default=0, help="limit #systems (debug)")
    ap.add_argument("--batch", type=int, default=6,
                    help="block groups (systems in flight) per persistent solve launch")
    ap.add_argument("--level1-systems", type=int, default=3,
                    help="systems of the pattern_level=1 sample (0: skip)")
    ap.add_argument("--cpu-solve-iters", type=int, default=5,
                    help="block steps of the truncated CPU solve sample")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def maybe_spawn(args):
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


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
                 "--format=csv,noheader,nounits", "-lms", "200"],
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
    s_grid, p_grid = list(W.s_grid), list(W.p_grid)
    if systems:
        s_grid, p_grid = s_grid[:1], p_grid[:systems]
    pts = [(s, np.atleast_1d(np.asarray(p, dtype=np.float64))) for s in s_grid for p in p_grid]
    return W, s_grid, p_grid, pts


def config_dict(args, W, nsys, world):
    """The workload description both arms print (identical keys/values)."""
    return {"workload": "c%d" % args.config, "n": int(W.n), "systems": int(nsys),
            "rhs_block": int(W.rhs.shape[1]), "pattern_level": int(W.pattern_level),
            "precond": "spai-update-first", "tol": 1e-8,
            "step": "cold sequence (symbolic caches rebuilt every step)",
            "l2": "working set >> 126 MB L2; L2 also flushed before every step (256 MB write)",
            "parallelism": "systems round-robin over %d GPU(s), base SPAI column-sharded" % world}


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ls_flops(m, n):
    """Householder QR + Q^T b + back substitution of an m x n LS problem."""
    return 2.0 * m * n * n - (2.0 / 3.0) * n ** 3 + 4.0 * m * n - n * n


def fp64_peaks():
    """Live DFMA / DMMA peaks of this GPU (pmp_fp64_peak)."""
    import ctypes
    from paper_1809_06574_b200 import _abi
    out = {}
    for kind, name in ((0, "dfma_tflops"), (1, "dmma_tflops")):
        v = ctypes.c_double()
        _abi.check(_abi.lib().pmp_fp64_peak(kind, 2000, ctypes.byref(v), _abi.stream()),
                   "pmp_fp64_peak")
        out[name] = v.value
    return out


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

TIMED_KERNELS = ("pmp_solve_batch", "pmp_ls_columns_multi", "pmp_ls_columns_planned",
                 "pmp_ls_columns", "pmp_assemble_multi", "pmp_assemble", "pmp_permute",
                 "pmp_permute_batch", "pmp_transpose", "pmp_pattern_l0", "pmp_pattern_l0_ptr",
                 "pmp_ls_bound")


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1809_06574_b200 as pm
    from paper_1809_06574_b200 import _abi

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    W, s_grid, p_grid, pts = workload(args.config, args.systems)
    nsys = len(pts)
    n = W.n
    model = pm.SecondOrderModel.from_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                         rhs=W.rhs)
    level = W.pattern_level
    pol = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=level),
                           update=pm.UpdateConfig(pattern_level=level))
    cfg = pm.SolverConfig(tol=1e-8)
    Bd = torch.as_tensor(np.ascontiguousarray(W.rhs), device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step(cold=True):
        if cold:
            model.reset_symbolic()
        return pm.run_sequence(model, s_grid, p_grid, pol, cfg, B=Bd, rank=rank, world=world,
                               timing=True, batch=args.batch)

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
    step_ms, infos = [], []
    # every ABI call of the timed steps counted; the candidate kernels are
    # bracketed by CUDA events on the launching (current) stream
    _abi.count_launches(True, timed=TIMED_KERNELS)
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
    timed = dict(_abi.timed_events())
    _abi.count_launches(False)
    clocks = clk.stop()
    t = torch.tensor([float(np.sum(step_ms))], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = n * nsys * args.steps / (total_ms / 1e3)
    step_local = float(np.sum(step_ms))

    kern = {}
    for name, lst in timed.items():
        ms = [a.elapsed_time(b) for a, b, _ in lst]
        kern[name] = {"launches": len(ms), "launches_per_step": len(ms) / args.steps,
                      "total_ms": float(np.sum(ms)), "avg_us": float(np.mean(ms) * 1e3),
                      "share_of_step": float(np.sum(ms)) / step_local}
    phase = {k: float(np.mean([i[k + "_s"] for i in infos])) for k in ("assemble", "build",
                                                                       "solve")}
    iters = [r["iterations"] for r in recs_all]
    conv = all(r["converged"] for r in recs_all)
    if world > 1:
        allrec = infos[-1].get("records_all") or []
        iters = [r["iterations"] for r in allrec] or iters
        conv = all(r["converged"] for r in allrec) if allrec else conv

    warm = None
    if args.warm:
        flush.zero_()
        barrier()
        w0 = torch.cuda.Event(enable_timing=True)
        w1 = torch.cuda.Event(enable_timing=True)
        w0.record()
        step(cold=False)
        w1.record()
        barrier()
        warm = w0.elapsed_time(w1)
        tw = torch.tensor([warm], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        warm = float(tw.item())

    rates = build_rates(pm, model, pts, pol, barrier, torch)
    peaks = fp64_peaks()
    roof = roofline(kern, timed, recs_all, args.steps)
    roof_ls = roofline_ls(kern, model, nsys / world, args.steps, peaks)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, pm, model, W, s_grid, p_grid, pol, cfg, rank, world, barrier)

    lvl1 = None
    if args.level1_systems > 0 and world == 1:
        lvl1 = level1_sample(args, pm, model, s_grid, p_grid, cfg, Bd, barrier, torch)

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded generator, SURVEY.md 8.1)",
            "config": config_dict(args, W, nsys, world),
            "sequence_s": ms_per_step / 1e3,
            "warm_ms_per_step": warm,
            "phases_s": phase,
            "spai_columns_per_s": rates["spai_columns_per_s"],
            "update_columns_per_s": rates["update_columns_per_s"],
            "update_window_columns_per_s": rates["update_window_columns_per_s"],
            "build_rates_detail": rates,
            "iterations": {"min": int(min(iters)), "max": int(max(iters)),
                           "mean": float(np.mean(iters)), "systems": len(iters)},
            "converged": conv,
            "gpu_launches": int(launches),
            "gpu_launches_per_step": int(launches) // args.steps,
            "abi_calls": counters,
            "kernels": kern,
            "roofline": roof,
            "roofline_ls": roof_ls,
            "fp64_peaks_measured": peaks,
            "clocks": clocks,
        }
        if e2e is not None:
            line["e2e"] = e2e
        if lvl1 is not None:
            line["level1_sample"] = lvl1
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(args, W, pts, model, pol, iters)
    if world > 1:
        dist.destroy_process_group()
    return line


def level1_sample(args, pm, model, s_grid, p_grid, cfg, Bd, barrier, torch):
    """pattern_level = 1 (the reference's default, spai.py:143 / update.py:50)
    on the first systems of the same sequence: cold spai_build + update_first
    with residual-driven augmentation (spai.py:285-289) + the solves.  Level 1
    has no window path (its supports depend on every system's values): the
    systems run one at a time on the same device kernels.  A bounded sample,
    outside the timed steps."""
    k = min(args.level1_systems, len(p_grid))
    pol1 = pm.PrecondPolicy("spai-update-first", spai=pm.SpaiConfig(pattern_level=1),
                            update=pm.UpdateConfig(pattern_level=1))
    model.reset_symbolic()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    recs, info = pm.run_sequence(model, s_grid[:1], p_grid[:k], pol1, cfg, B=Bd, timing=True,
                                 batch=args.batch)
    e1.record()
    barrier()
    t = e0.elapsed_time(e1) / 1e3
    model.reset_symbolic()
    return {"pattern_level": 1, "systems": k, "sequence_s": t,
            "columns_per_s": model.dim * k / t,
            "phases_s": {ph: float(info[ph + "_s"]) for ph in ("assemble", "build", "solve")},
            "iterations": [int(r["iterations"]) for r in recs],
            "converged": bool(all(r["converged"] for r in recs)),
            "note": "first %d systems of the sequence, cold, systems one at a time" % k}


def build_rates(pm, model, pts, pol, barrier, torch, reps=3):
    """SPAI columns/s = n / spai_build (device A -> device P,
    cold symbolic state: pattern, plans and transpose included); update
    columns/s = n / update_first of one system; the window rate of the
    sequence's batched update_first_many.  Median of `reps` (untimed by the
    step clock)."""
    from paper_1809_06574_b200.update import update_first_many
    n = model.dim
    sp_t, up_t, win_t, spw_t, upw_t = [], [], [], [], []
    k = max(1, min(len(pts) - 1, 16))
    for _ in range(reps):
        model.reset_symbolic()
        A1 = model.assemble(*pts[0])
        A2 = model.assemble(*pts[min(1, len(pts) - 1)])
        barrier()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record()
        P1, _ = pm.spai_build(A1, pol.spai)
        e[1].record()
        pm.update_first(A1, A2, P1, pol.update)
        e[2].record()
        barrier()
        sp_t.append(e[0].elapsed_time(e[1]) / 1e3)
        up_t.append(e[1].elapsed_time(e[2]) / 1e3)
        As = model.assemble_many(pts[1:1 + k])
        barrier()
        e[0].record()
        update_first_many(A1, As, P1, pol.update)
        e[3].record()
        barrier()
        win_t.append(e[0].elapsed_time(e[3]) / 1e3)
        # the same two calls again with the structure's symbolic state kept
        # (pattern, LS plans, transpose plan): what every later build of a
        # sequence on this structure costs
        barrier()
        e[0].record()
        P1w, _ = pm.spai_build(A1, pol.spai)
        e[1].record()
        pm.update_first(A1, A2, P1w, pol.update)
        e[2].record()
        barrier()
        spw_t.append(e[0].elapsed_time(e[1]) / 1e3)
        upw_t.append(e[1].elapsed_time(e[2]) / 1e3)
        del As, A1, A2, P1, P1w
    ts, tu, tw = float(np.median(sp_t)), float(np.median(up_t)), float(np.median(win_t))
    tsw, tuw = float(np.median(spw_t)), float(np.median(upw_t))
    return {"spai_columns_per_s": n / ts, "update_columns_per_s": n / tu,
            "update_window_columns_per_s": n * k / tw, "spai_build_s": ts,
            "update_first_s": tu, "update_window_systems": k, "update_window_s": tw,
            "spai_columns_per_s_warm": n / tsw, "update_columns_per_s_warm": n / tuw,
            "spai_build_warm_s": tsw, "update_first_warm_s": tuw,
            "reps": reps, "note": "device-resident A in, device-resident factor + stats out; "
                                  "spai_build / update_first on a cold structure (symbolic "
                                  "planning included), then with the structure's plans kept "
                                  "(_warm)"}


def roofline(kern, timed, recs, steps):
    """The dominant kernel (pmp_solve_batch: the persistent block-GCRO
    solve, ~85-90 % of the step) against the measured HBM peak.  Algorithmic
    bytes per launch: the kernel itself accumulates, per system and per block
    step, SURVEY.md 8(d)'s units -- SpMM 12 nnz + 4 (n + 1) + 16 n s_b per
    matrix of the operator chain, block orthogonalisation 32 n total + 48 n
    s_b + 16 n k (CGS2: two Gram products and two updates over [C | V]) --
    summed over the step's systems, divided by the step's launches.  The
    stricter every-operand-once figure round 1 reported rides along as
    `achieved_strict` / `frac_strict`."""
    hbm, which = hbm_peak()
    name = "pmp_solve_batch"
    if name not in kern:
        return None
    lst = timed[name]
    per_step_bytes = sum(r.get("algorithmic_bytes") or 0.0 for r in (recs or []))
    strict_bytes = sum(r.get("algorithmic_bytes_strict") or 0.0 for r in (recs or []))
    launches_per_step = len(lst) / steps
    ms = np.array([a.elapsed_time(b) for a, b, _ in lst])
    ach = per_step_bytes * steps / (np.sum(ms) / 1e3) / 1e9
    ach_strict = strict_bytes * steps / (np.sum(ms) / 1e3) / 1e9
    # DRAM bytes from the committed ncu --set full capture of this config's
    # k_solve (a 6-system batch, tools/gpu_ncu_solve.sh), scaled to this
    # run's launch by the ratio of algorithmic bytes
    traffic = None
    traffic_note = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        ent = tj.get(name + "_c%s" % os.environ.get("PMP_BENCH_CONFIG", "4"))
        if ent:
            per_launch = per_step_bytes / max(launches_per_step, 1e-9)
            traffic = ent["dram_bytes"] * per_launch / ent["algorithmic_bytes"]
            traffic_note = ("%s: %.4g DRAM bytes for %.4g algorithmic (x%.2f), scaled to this "
                            "launch" % (ent["source"], ent["dram_bytes"], ent["algorithmic_bytes"],
                                        ent["dram_bytes"] / ent["algorithmic_bytes"]))
    except (OSError, ValueError, KeyError):
        pass
    return {"kernel": name, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
            "frac": ach / hbm, "traffic": traffic, "traffic_source": traffic_note,
            "algorithmic_bytes_per_launch": per_step_bytes / max(launches_per_step, 1e-9),
            "algorithmic_unit": "SURVEY.md 8(d): per block step, operator chain (12 nnz + 4 (n+1) "
                                "+ 16 n s_b per matrix) + block CGS2 (32 n total + 48 n s_b + "
                                "16 n k); summed by the kernel per system",
            "achieved_strict": ach_strict, "frac_strict": ach_strict / hbm,
            "strict_unit": "every operand once per block step ([C | V] read once: the "
                           "round-1 figure)",
            "peak_source": which, "launches": len(lst),
            "avg_us": kern[name]["avg_us"], "share_of_step": kern[name]["share_of_step"]}


def roofline_ls(kern, model, nsys, steps, peaks):
    """Batched least-squares kernels (SPAI + every update of the step)
    against the MEASURED FP64 peaks.  Algorithmic flops per column
    F_j = 2 m n^2 - 2/3 n^3 + 4 m n - n^2 (m = |J_j|, n = |I_j|, level-0
    supports: I_j = rows(A(:, j)), J_j = rows(A(:, I_j)); the same for the
    SPAI and every update), `nsys` builds per step on this rank."""
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
    t = sum(kern[k]["total_ms"] for k in names) / 1e3 / steps
    ach = nsys * f_sys / t / 1e12
    dfma = peaks["dfma_tflops"]
    return {"kernels": names, "bound": "fp64", "achieved": ach, "peak": dfma,
            "unit": "TFLOP/s", "frac": ach / dfma, "frac_vs_dmma": ach / peaks["dmma_tflops"],
            "flops_per_build": f_sys, "builds_per_step": nsys, "seconds_per_step": t,
            "peak_source": "measured live (pmp_fp64_peak: DFMA chains; DMMA m8n8k4 also "
                           "reported)"}


def run_e2e(args, pm, model, W, s_grid, p_grid, pol, cfg, rank, world, barrier):
    """Same metric through the public API (run_sequence) from HOST buffers:
    every step copies the model's term values and B host->device from
    pinned memory and reads every solution block back device->host (each
    window's X as soon as its solve launch is done, into a pinned ring:
    every byte of every system's X crosses the link).  Cold steps like the
    device-resident ones."""
    import torch

    u = model._union()
    host_terms = [v.cpu().pin_memory() for v in u.vals]
    Bh = torch.as_tensor(np.ascontiguousarray(W.rhs)).pin_memory()
    Bd = torch.empty_like(Bh, device="cuda")
    n, s = W.rhs.shape
    ring = torch.empty((4, n, s), dtype=torch.float64).pin_memory()
    from paper_1809_06574_b200.sequence import owned_systems
    nsys = len(s_grid) * len(p_grid)
    mine = owned_systems(nsys, rank, world, pol.kind)
    h2d = sum(t.numel() * 8 for t in host_terms) + Bh.numel() * 8
    d2h = len(mine) * n * s * 8

    def sink(idx, X):
        ring[idx % ring.shape[0]].copy_(X, non_blocking=True)

    times = []
    nsteps = max(1, min(args.e2e_steps, args.steps))
    for k in range(1 + nsteps):
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for hv, dv in zip(host_terms, u.vals):
            dv.copy_(hv, non_blocking=True)
        Bd.copy_(Bh, non_blocking=True)
        model.reset_symbolic()
        pm.run_sequence(model, s_grid, p_grid, pol, cfg, B=Bd, rank=rank, world=world,
                        timing=False, batch=args.batch, on_solution=sink)
        e1.record()
        barrier()
        if k >= 1:
            times.append(e0.elapsed_time(e1))
    t = torch.tensor([float(np.sum(times))], dtype=torch.float64, device="cuda")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_s = float(t.item()) / 1e3
    return {"value": W.n * nsys * nsteps / total_s, "unit": UNIT,
            "ms_per_step": total_s * 1e3 / nsteps, "steps": nsteps, "warmup": 1,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "api": "run_sequence(..., on_solution=D2H into pinned host ring)"}


# ---------------------------------------------------------------------------
# CPU side (oracle port): bounded samples, extrapolated to the sequence
# ---------------------------------------------------------------------------

_CPU = {}


def _cpu_init(A1, A2):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pmor_oracle as orc
    _CPU["orc"] = orc
    _CPU["sys"] = orc.canon(A2).tocsc()
    _CPU["tgt"] = orc.canon(A1).tocsc()


def _cpu_cols(cols):
    orc = _CPU["orc"]
    S, T = _CPU["sys"], _CPU["tgt"]
    pat = {int(j): orc.level0_support(S, int(j)) for j in cols}
    return orc.solve_columns(S, T, pat, 1e-4, 0, 80, [int(j) for j in cols])


class CpuSampler:
    """The reference's algorithm (oracle port) on this host's cores.

    Per sample: (a) the update_first least squares (update.py:78-87,
    spai.py:273-292) of the first CPU_SAMPLE_COLUMNS columns of
    default_rng(7).permutation(n), chunked over a process
    pool created beforehand (not timed); (b) block GCRO (krylov.py:105-275)
    on the same system, truncated after `solve_iters` block steps (its
    cycle end included).  Extrapolation to the whole sequence:
    t_seq = systems * n / rate_cols + systems * t_solve_iters * (iters /
    solve_iters) -- a per-step cost taken from the FIRST block steps, whose
    Gram work is below the average step's, so the CPU estimate errs fast."""

    def __init__(self, W, pts, cores, P1, Q):
        import multiprocessing as mp
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pmor_oracle as orc
        self.orc = orc
        self.W = W
        self.cores = cores
        self.A1 = orc.assemble_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms, *pts[0])
        self.A2 = orc.assemble_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                                   *pts[min(1, len(pts) - 1)])
        n = W.n
        self.cols = np.random.default_rng(7).permutation(n)[:min(CPU_SAMPLE_COLUMNS, n)]
        self.pool = mp.get_context("fork").Pool(cores, initializer=_cpu_init,
                                                initargs=(self.A1, self.A2))
        self.chain = orc.Chain([Q, P1])
        self.pool.map(_cpu_cols, [self.cols[:cores]] * cores)   # warm the workers

    def close(self):
        self.pool.close()
        self.pool.join()

    def sample(self, solve_iters):
        chunks = np.array_split(self.cols, self.cores * 4)
        t0 = time.perf_counter()
        parts = self.pool.map(_cpu_cols, chunks)
        t1 = time.perf_counter()
        _, info = self.orc.block_gcro(self.A2, self.W.rhs, self.chain, tol=1e-8,
                                      max_iters=solve_iters)
        t2 = time.perf_counter()
        ncols = sum(len(p) for p in parts)
        return {"cols_s": t1 - t0, "cols": ncols, "solve_s": t2 - t1,
                "solve_iters": int(info["iterations"])}


def extrapolate(smp, n, nsys, iters_mean):
    rate = smp["cols"] / smp["cols_s"]
    t_solve = smp["solve_s"] * iters_mean / max(smp["solve_iters"], 1)
    t_seq = nsys * n / rate + nsys * t_solve
    return t_seq, rate, t_solve


def _cpu_factors_from_device(pm, model, pts, pol):
    """P1 and Q of system 2 as host CSR (for the CPU solve sample only: the
    truncated solve's cost depends on their sizes, not their values; the
    values are the reference's to ~1e-16 -- pinned by the parity tests)."""
    A1 = model.assemble(*pts[0])
    A2 = model.assemble(*pts[min(1, len(pts) - 1)])
    P1, _ = pm.spai_build(A1, pol.spai)
    P2, _ = pm.update_first(A1, A2, P1, pol.update)
    return P1.matrix.to_scipy(), P2.q.to_scipy()


def cpu_baseline(args, W, pts, model, pol, iters):
    import paper_1809_06574_b200 as pm
    cores = max(1, len(os.sched_getaffinity(0)))
    os.environ["OPENBLAS_NUM_THREADS"] = str(cores)
    P1, Q = _cpu_factors_from_device(pm, model, pts, pol)
    cs = CpuSampler(W, pts, cores, P1, Q)
    try:
        smp = cs.sample(args.cpu_solve_iters)
    finally:
        cs.close()
    it = float(np.mean(iters))
    t_seq, rate, t_solve = extrapolate(smp, W.n, len(pts), it)
    return {"value": W.n * len(pts) / t_seq, "unit": UNIT, "cores": cores, "kind": "port",
            "extrapolated": True, "sequence_s": t_seq,
            "sample": ("c%d: update_first least squares of %d columns (default_rng(7) "
                       "permutation) over %d processes (%.0f columns/s) + block GCRO truncated "
                       "at %d block steps (%.2f s), extrapolated to %d systems x %d columns and "
                       "%.2f iterations per solve (this run's mean)"
                       % (args.config, smp["cols"], cores, rate, smp["solve_iters"],
                          smp["solve_s"], len(pts), W.n, it))}


def run_reference(args):
    """--impl reference: the reference's algorithm (oracle port) on the host
    cores, on our arm's config / metric.  Setup (untimed): host assembly,
    the full base SPAI and one full update (process pool), and ONE full
    block GCRO solve of system 2 (its iteration count drives the
    extrapolation).  Each step: a fresh bounded sample (CpuSampler)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    W, s_grid, p_grid, pts = workload(args.config, args.systems)
    nsys = len(pts)
    cores = max(1, len(os.sched_getaffinity(0)))
    os.environ["OPENBLAS_NUM_THREADS"] = str(cores)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pmor_oracle as orc
    import multiprocessing as mp
    t0 = time.perf_counter()
    A1 = orc.assemble_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms, *pts[0])
    A2 = orc.assemble_mdk(W.mass_terms, W.damping_terms, W.stiffness_terms,
                          *pts[min(1, len(pts) - 1)])
    n = W.n
    chunks = np.array_split(np.arange(n), cores * 8)
    with mp.get_context("fork").Pool(cores, initializer=_cpu_init, initargs=(A1, A1)) as pool:
        resP = [r for part in pool.map(_cpu_cols_spai, chunks) for r in part]
    P1, _ = orc.assemble_columns(n, resP)
    with mp.get_context("fork").Pool(cores, initializer=_cpu_init, initargs=(A1, A2)) as pool:
        resQ = [r for part in pool.map(_cpu_cols, chunks) for r in part]
    Q, _ = orc.assemble_columns(n, resQ)
    t_build_full = time.perf_counter() - t0
    t1 = time.perf_counter()
    _, info = orc.block_gcro(A2, W.rhs, orc.Chain([Q, P1]), tol=1e-8)
    t_solve_full = time.perf_counter() - t1
    it_ref = int(info["iterations"])
    cs = CpuSampler(W, pts, cores, P1, Q)
    times, last = [], None
    try:
        for k in range(args.warmup + args.steps):
            smp = cs.sample(args.cpu_solve_iters)
            t_seq, rate, t_solve = extrapolate(smp, n, nsys, it_ref)
            last = (smp, rate, t_solve)
            if k >= args.warmup:
                times.append(t_seq)
    finally:
        cs.close()
    ms = float(np.mean(times)) * 1e3
    value = n * nsys * args.steps / float(np.sum(times))
    smp, rate, t_solve = last
    sample = ("per step: update_first least squares of %d columns of c%d (default_rng(7) "
              "permutation, %d processes; %.0f columns/s) + block GCRO on system 2 truncated at "
              "%d block steps, extrapolated to %d systems x %d columns at %d iterations per "
              "solve (the oracle's full solve of system 2 in setup: %d iterations, %.1f s; "
              "full base + update builds in setup %.1f s)"
              % (smp["cols"], args.config, cores, rate, smp["solve_iters"], nsys, n, it_ref,
                 it_ref, t_solve_full, t_build_full))
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, SURVEY.md 8.1)", "impl": "reference",
            "config": config_dict(args, W, nsys, world),
            "extrapolated": True, "sample": sample,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "extrapolated": True, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def _cpu_cols_spai(cols):
    """SPAI columns (target = identity) on the worker's system."""
    orc = _CPU["orc"]
    S = _CPU["tgt"]
    import scipy.sparse as sp
    if "eye" not in _CPU:
        _CPU["eye"] = sp.identity(S.shape[0], format="csc")
    pat = {int(j): orc.level0_support(S, int(j)) for j in cols}
    return orc.solve_columns(S, _CPU["eye"], pat, 1e-4, 0, 80, [int(j) for j in cols])


def main():
    args = parse()
    if args.impl == "ours":
        maybe_spawn(args)
        os.environ["PMP_BENCH_CONFIG"] = str(args.config)
        line = run_ours(args)
    else:
        line = run_reference(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
