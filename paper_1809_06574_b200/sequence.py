"""Sequence driver: assemble -> SPAI / SPAI-update -> block GCRO over the
(sigma, p) grid, on one or several GPUs.

Mirrors the reference's ``PrecondPolicy`` / ``SequencePreconditioner``
(rpmor.py:177-218) and the composition of SURVEY.md 3.4 (``pmor_l_sequence``
order, zoo.py:268-284: sigma outermost, p inner; first system gets a fresh
SPAI, the others the configured update).

Multi-GPU (one process per GPU; collectives through NCCL behind the C-ABI,
comm.py): with the "first" approach every system depends only on (A1, P1)
(rpmor.py:208-210), so systems are dealt round-robin over ranks by their
global sequence index.  Every rank assembles A1 and its own systems locally
from the replicated terms.  P1 is built column-sharded at pattern level 0
(rank r solves its contiguous column range, one grouped all-gather
replicates the coefficients: spai.spai_build_sharded); at level >= 1 rank 0
builds it and broadcasts structure and values.  Per-system scalar records
are summed over ranks at the end (one allreduce of a zero-padded table:
every system has exactly one owner) into ``info["records_all"]``;
solutions stay on their owner GPU.  "spai" runs independently per rank;
"spai-update-second" has a true chain dependency and therefore runs as
replicas (every rank walks the whole chain).
"""

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import krylov as _krylov
from .krylov import SolverConfig, block_gcro_solve, block_gcro_solve_batch
from .spai import Preconditioner, SpaiConfig, spai_build, spai_build_sharded
from .update import UpdateConfig, update_first, update_first_many, update_second

PRECOND_KINDS = ("none", "spai", "spai-update-first", "spai-update-second")


@dataclass
class PrecondPolicy:
    kind: str = "none"
    spai: SpaiConfig = field(default_factory=SpaiConfig)
    update: UpdateConfig = field(default_factory=UpdateConfig)
    threads: int = 1

    def __post_init__(self):
        if self.kind not in PRECOND_KINDS:
            raise ValueError("unknown preconditioner kind %r" % self.kind)


class SequencePreconditioner:
    """Stateful producer of per-system preconditioners (rpmor.py:189-218)."""

    def __init__(self, policy=None):
        self.policy = policy or PrecondPolicy()
        self._initial_system = None
        self._initial_pre = None
        self._prev_system = None
        self._prev_pre = None

    def seed(self, A1, P1):
        """Install an externally built initial pair (the broadcast P1)."""
        self._initial_system, self._initial_pre = A1, P1
        self._prev_system, self._prev_pre = A1, P1

    def for_system(self, A):
        """Returns (preconditioner-or-None, build_seconds, kind_label, stats)."""
        pol = self.policy
        if pol.kind == "none":
            return None, 0.0, "none", None
        t0 = time.perf_counter()
        if pol.kind == "spai" or self._initial_pre is None:
            P, stats = spai_build(A, pol.spai, threads=pol.threads)
            label = "spai"
        elif pol.kind == "spai-update-first":
            P, stats = update_first(self._initial_system, A, self._initial_pre, pol.update)
            label = "update-first"
        else:
            P, stats = update_second(self._prev_system, A, self._prev_pre, pol.update)
            label = "update-second"
        seconds = time.perf_counter() - t0
        if self._initial_pre is None:
            self._initial_system, self._initial_pre = A, P
        self._prev_system, self._prev_pre = A, P
        return P, seconds, label, stats

    def for_systems(self, systems):
        """for_system over a list; under the first approach the updates of
        systems sharing a structure are built together (update_first_many,
        bitwise the one-at-a-time results)."""
        systems = list(systems)
        out = []
        if self.policy.kind == "spai-update-first" and systems:
            if self._initial_pre is None:
                out.append(self.for_system(systems[0]))
                systems = systems[1:]
            if systems:
                t0 = time.perf_counter()
                res = update_first_many(self._initial_system, systems, self._initial_pre,
                                        self.policy.update)
                seconds = (time.perf_counter() - t0) / len(systems)
                for P, stats in res:
                    out.append((P, seconds, "update-first", stats))
                self._prev_system, self._prev_pre = systems[-1], res[-1][0]
            return out
        return [self.for_system(A) for A in systems]


# ---------------------------------------------------------------------------
# sharding helpers (host logic; tested with gloo on CPU)
# ---------------------------------------------------------------------------

def owned_systems(n_systems, rank, world, kind="spai-update-first"):
    """Global sequence indices this rank solves: round-robin for independent
    systems, the whole chain (replica) for the second approach."""
    if world <= 1 or kind == "spai-update-second":
        return list(range(n_systems))
    return [i for i in range(n_systems) if i % world == rank]


RECORD_FIELDS = ("index", "iterations", "converged", "matvec_count", "precond_apply_count",
                 "max_final_residual")


def gather_records(records, n_systems, group=None):
    """Every system's scalar record on every rank: the zero-padded
    (n_systems x fields) table of this rank's systems, summed over ranks
    (each system has exactly one owner) -- pmp_nccl_allreduce_f64 on the
    device under NCCL, a host allreduce under gloo."""
    from .comm import get_comm, record_table
    table = record_table(records, n_systems, RECORD_FIELDS)
    comm = get_comm(group)
    if comm.world > 1:
        t = torch.as_tensor(table)
        if comm.uses_nccl:
            t = t.cuda()
        comm.allreduce_sum_f64(t)
        table = t.cpu().numpy()
    out = []
    for row in table:
        if row[0] == 0:
            continue
        d = dict(zip(RECORD_FIELDS, row.tolist()))
        d["index"] = int(d["index"]) - 1
        d["iterations"] = int(d["iterations"])
        d["converged"] = bool(d["converged"])
        d["matvec_count"] = int(d["matvec_count"])
        d["precond_apply_count"] = int(d["precond_apply_count"])
        out.append(d)
    return out


# ---------------------------------------------------------------------------
# the driver
# ---------------------------------------------------------------------------

# HBM budget for one solve window (operators + preconditioner factors + X)
WINDOW_BYTES = int(__import__("os").environ.get("PMP_WINDOW_BYTES", str(64 << 30)))


def _window_systems(model, B):
    """Systems per solve window: every system's A (values), its update factor
    (indices + values) and X stay resident until the window's launch ends."""
    n, s = B.shape
    st = model.structure
    nnz = st.nnz
    nonsym = not model._union().symmetric
    # per system: assembled values (+ their CSC copy when unsymmetric), the
    # update factor's coefficient and CSR value rows (pattern nnz <= nnz of
    # the structure at level 0), residual / flag rows, X
    per = 8 * nnz * (2 if nonsym else 1) + 16 * nnz + 12 * n + 8 * n * s
    # the persistent solve's per-group workspace (V n x cap, C / U n x kc,
    # nine n x s blocks) comes out of the same budget
    cap = 50 + 2 * s + 2
    ws = 8 * n * (cap + 2 * (10 + s) + 9 * s) * 6
    return max(1, (WINDOW_BYTES - ws) // per)

def run_sequence(model, s_grid, p_grid, policy=None, solver_cfg=None, B=None, rank=0, world=1,
                 group=None, keep_solutions=False, timing=True, workers=1, batch=None,
                 window=None, on_solution=None):
    """Run the whole parametric sequence; returns (records, info).

    records: one dict per system this rank owns (index, sigma, p, label,
    iterations, converged, counts, final residuals, optional X).
    info: phase times from CUDA events (summed assemble / build / solve
    seconds; with workers > 1 the phases of different systems overlap) and
    the number of SPAI / update columns built.

    batch > 1 (the default, PMP_BATCH_GROUPS; first-approach / independent
    policies): a window of systems is assembled and preconditioned (all
    launches asynchronous, no host synchronisation), then solved by ONE
    persistent device launch in which ``batch`` block groups take the
    window's systems from a device queue (block_gcro_solve_batch).  The
    window is every remaining system, capped so the window's operators,
    preconditioners and solutions stay under WINDOW_BYTES of HBM (``window``
    overrides).  batch=1 keeps the per-system path below.

    workers > 1 (first-approach / independent policies): after the initial
    system (and one update that warms the plan caches), the remaining
    systems are dealt to `workers` host threads, each driving its own CUDA
    stream, so the latency-bound block solves of independent systems overlap
    on the device; grid-barrier kernels are serialised through one shared
    stream (pmp_set_coop_stream).

    on_solution(index, X): called with every solution block (device tensor,
    on the current stream) as soon as its solve is done -- e.g. to copy it to
    the host -- without keeping every X alive (keep_solutions).

    Memory: a window's solutions live in one [k, n, s] allocation (as do its
    assembled values and factor coefficients); keep_solutions therefore
    stores a private copy of each X, so holding one system's solution never
    pins the whole window's block.
    """
    import threading
    from . import _abi

    policy = policy or PrecondPolicy("spai-update-first")
    solver_cfg = solver_cfg or SolverConfig(tol=1e-8)
    B = model.rhs if B is None else B
    if torch.is_tensor(B):
        Bd = B
    elif np.iscomplexobj(B) and np.any(np.asarray(B).imag != 0):
        Bd = np.asarray(B, dtype=np.complex128)   # complex: realified per solve (cplx.py)
    else:
        Bd = torch.as_tensor(np.ascontiguousarray(np.real(B), dtype=np.float64), device="cuda")
    points = [(s, np.atleast_1d(p)) for s in s_grid for p in p_grid]
    nsys = len(points)
    mine = owned_systems(nsys, rank, world, policy.kind)
    seq = SequencePreconditioner(policy)
    lock = threading.Lock()

    def mark():
        if not timing:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    phases = {"assemble": [], "build": [], "solve": []}
    state = {"build_cols": 0}
    records = []
    sharded = world > 1 and policy.kind == "spai-update-first"
    A1 = P1 = None
    if sharded:
        # every rank: A1 locally; P1 column-sharded over the ranks (level 0)
        # or built by rank 0 and broadcast with its structure (level >= 1)
        from .comm import get_comm
        comm = get_comm(group)
        if comm.world != world or comm.rank != rank:
            raise ValueError("rank/world (%d/%d) do not match the process group (%d/%d)"
                             % (rank, world, comm.rank, comm.world))
        t0 = mark()
        A1 = model.assemble(*points[0])
        t1 = mark()
        phases["assemble"].append((t0, t1))
        P1, _ = spai_build_sharded(A1, policy.spai, comm)
        if policy.spai.pattern_level == 0:   # this rank's share of P1's columns
            state["build_cols"] += A1.n * (rank + 1) // world - A1.n * rank // world
        elif rank == 0:
            state["build_cols"] += A1.n
        t2 = mark()
        phases["build"].append((t1, t2))
        seq.seed(A1, P1)

    def do_system(idx):
        s, p = points[idx]
        t0 = mark()
        A = A1 if (sharded and idx == 0) else model.assemble(s, p)
        t1 = mark()
        if sharded and idx == 0:
            P, label, cols = P1, "spai", 0
        else:
            P, _, label, _ = seq.for_system(A)
            cols = A.n if P is not None else 0
        t2 = mark()
        X, rep = block_gcro_solve(A, Bd, P=P, cfg=solver_cfg)
        t3 = mark()
        rec = {"index": idx, "sigma": float(s), "p": [float(v) for v in p], "label": label,
               "iterations": rep.iterations, "converged": rep.converged,
               "matvec_count": rep.matvec_count, "precond_apply_count": rep.precond_apply_count,
               "final_residuals": np.asarray(rep.final_residuals, dtype=float).tolist(),
               "max_final_residual": float(np.max(rep.final_residuals)),
               "launches": getattr(rep, "device_launches", 0)}
        if keep_solutions:
            rec["X"] = X
        if on_solution is not None:
            on_solution(idx, X)
        with lock:
            records.append(rec)
            state["build_cols"] += cols
            if timing:
                phases["assemble"].append((t0, t1))
                phases["build"].append((t1, t2))
                phases["solve"].append((t2, t3))

    if batch is None:
        batch = _krylov.BATCH_GROUPS if workers <= 1 else 0
    batched = batch > 1 and policy.kind in ("spai-update-first", "spai", "none")
    if batched:
        # assemble + precondition a chunk of systems, then solve the chunk in
        # one persistent launch (one block group per system)
        todo = list(mine)
        if window is None:
            window = _window_systems(model, Bd)
        window = max(batch, int(window))
        for c0 in range(0, len(todo), window):
            chunk = todo[c0:c0 + window]

            def run_window(defer):
                built = []
                t0 = mark()
                # sharded: system 0 is (A1, P1), already assembled and built
                head = sharded and chunk[0] == 0
                pts_ = [points[idx] for idx in (chunk[1:] if head else chunk)]
                if defer:
                    As, zc = model.assemble_many(pts_, defer_zero_check=True)
                else:
                    As, zc = model.assemble_many(pts_), None
                t1 = mark()
                # (the window's assembly and its build are one phase each:
                # charged to the window's first system)
                pres = seq.for_systems(As) if As else []
                if head:
                    As = [A1] + As
                    pres = [(P1, 0.0, "spai", None)] + pres
                t2 = mark()
                for j, (idx, A, (P, _, label, _)) in enumerate(zip(chunk, As, pres)):
                    if j == 0:
                        built.append((idx, A, P, label, t0, t1, t2, t1))
                    else:
                        built.append((idx, A, P, label, None, None, None, None))
                t3 = mark()
                res = block_gcro_solve_batch([(b[1], b[2]) for b in built], Bd,
                                             cfg=solver_cfg, groups=batch)
                t4 = mark()
                return built, res, t3, t4, zc

            # the window is enqueued without a host synchronisation: its
            # systems are assembled on the union structure and the exact-zero
            # counts are checked once the solves are back; a window with an
            # exact zero (the reference's as_csr drops it: compacted
            # structures) is redone from the same preconditioner state
            seq_state = (seq._initial_system, seq._initial_pre, seq._prev_system,
                         seq._prev_pre)
            built, res, t3, t4, zc = run_window(True)
            if zc is not None and int(zc.max().item()) > 0:
                (seq._initial_system, seq._initial_pre, seq._prev_system,
                 seq._prev_pre) = seq_state
                built, res, t3, t4, _ = run_window(False)
            for (idx, A, P, label, t0, t1, t2, ta), (X, rep) in zip(built, res):
                s, p = points[idx]
                rec = {"index": idx, "sigma": float(s), "p": [float(v) for v in p],
                       "label": label, "iterations": rep.iterations,
                       "converged": rep.converged, "matvec_count": rep.matvec_count,
                       "precond_apply_count": rep.precond_apply_count,
                       "final_residuals": np.asarray(rep.final_residuals, dtype=float).tolist(),
                       "max_final_residual": float(np.max(rep.final_residuals)),
                       "launches": getattr(rep, "device_launches", 0),
                       "algorithmic_bytes": getattr(rep, "algorithmic_bytes", None),
                       "algorithmic_bytes_strict": getattr(rep, "algorithmic_bytes_strict",
                                                           None)}
                if keep_solutions:
                    rec["X"] = X.clone()   # (X is a view of the window's block)
                if on_solution is not None:
                    on_solution(idx, X)
                records.append(rec)
                if P is not None and not (sharded and idx == 0):  # (P1: counted above)
                    state["build_cols"] += A.n
                if timing and t0 is not None:
                    phases["assemble"].append((t0, t1))
                    phases["build"].append((ta, t2))
            if timing:
                phases["solve"].append((t3, t4))
        mine = []
    parallel = workers > 1 and policy.kind in ("spai-update-first", "spai", "none")
    head = mine[:2] if parallel else mine
    for idx in head:
        do_system(idx)
    rest = mine[len(head):]
    if rest:
        main = torch.cuda.current_stream()
        coop = torch.cuda.Stream()
        coop.wait_stream(main)
        streams = [torch.cuda.Stream() for _ in range(min(workers, len(rest)))]
        for st in streams:
            st.wait_stream(main)
        errors = []

        def worker(w):
            try:
                with torch.cuda.stream(streams[w]):
                    for idx in rest[w::len(streams)]:
                        do_system(idx)
            except BaseException as e:  # surfaced after join
                errors.append(e)

        _abi.check(_abi.lib().pmp_set_coop_stream(coop.cuda_stream), "pmp_set_coop_stream")
        try:
            threads = [threading.Thread(target=worker, args=(w,)) for w in range(len(streams))]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
        finally:
            _abi.lib().pmp_set_coop_stream(None)
        for st in streams:
            main.wait_stream(st)
        main.wait_stream(coop)
        if errors:
            raise errors[0]
    records.sort(key=lambda r: r["index"])
    info = {"build_columns": state["build_cols"]}
    if world > 1:
        info["records_all"] = gather_records(records, nsys, group)
    if timing:
        torch.cuda.synchronize()
        for k, lst in phases.items():
            info[k + "_s"] = sum(a.elapsed_time(b) for a, b in lst) / 1e3
    return records, info
