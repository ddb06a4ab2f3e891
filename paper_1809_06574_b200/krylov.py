"""Right-preconditioned block GCRO on the B200 -- same API and control flow
as ``pmorprec.krylov`` (krylov.py:32-290).

Split of the work:
  * every n-sized operation runs on the device through libpmorb200:
    the operator A P V (CSR SpMM chain, krylov.py:140-147), the outer
    projection and the two-pass block Gram-Schmidt (tall-skinny Gram +
    update, krylov.py:189-196), the R factor of the rank-revealing QR
    (TSQR, krylov.py:88) and the new basis block Q = Z Pi R^-1 (tall-skinny
    multiply), solution / residual / outer-space updates (krylov.py:221-269);
  * the tiny dense algebra stays on the host, in native code
    (csrc/hostls.cpp): the pivoted QR of the s x s R factor (geqp3
    semantics, krylov.py:88) and an incremental Householder QR of the
    (k + total) x (k + m) projected least-squares problem (the reference
    re-solves it from scratch with gelsd, krylov.py:211; the minimum-norm
    gelsd solve is kept as the fallback for a rank-deficient G), plus every
    control-flow decision (restart, deflation rank, stopping, breakdown,
    outer-space fold and truncation: krylov.py:152-271).
One small device->host copy (a few KB) per block step carries all the
small matrices the host needs; n-sized data never leaves HBM.
"""

import ctypes
import os as _os
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import torch

from . import _abi
from .device import DeviceCSR, _dev, scratch
from .spai import Preconditioner, _as_dev_csr, _block_to_dev


class SolverBreakdown(RuntimeError):
    """No new Krylov direction while the residual is above tolerance
    (krylov.py:32-34)."""


@dataclass
class SolverConfig:
    tol: float = 1e-10
    max_iters: int = 1000
    outer_space_dim: int = 10
    inner_restart: int = 50
    deflation_tol: float = 1e-12

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        if self.inner_restart < 1:
            raise ValueError("inner_restart must be at least 1")


@dataclass
class SolveReport:
    iterations: int = 0
    converged: bool = False
    residual_history: list = field(default_factory=list)
    matvec_count: int = 0
    precond_apply_count: int = 0
    wall_time: float = 0.0
    reorth_passes: int = 0
    deflation_fallbacks: int = 0

    @property
    def final_residuals(self):
        return self.residual_history[-1] if self.residual_history else None


def apply_preconditioner(P, V):
    """Apply a right preconditioner to a block (krylov.py:68-76)."""
    if not isinstance(P, Preconditioner):
        raise TypeError("expected a Preconditioner")
    return P.apply(V)


def _safe_rel(norms, refs):
    out = np.zeros_like(norms)
    nz = refs > 0
    out[nz] = norms[nz] / refs[nz]
    return out


# reorthogonalise a new basis block when cond(R11) exceeds this (the block
# Q = Z Pi R11^-1 then loses more than ~1e-13 of orthogonality)
_REORTH_COND = 1e3


class _Dev:
    """Device buffers and direct ctypes handles for one block solve (the
    inner loop issues ~15 library calls per block step, so the per-call
    Python overhead is kept to a plain ctypes call)."""

    def __init__(self, n, s, cap, kc):
        self.n, self.s, self.cap, self.kc = n, s, cap, kc
        dev = _dev()
        f = lambda size: torch.empty(max(size, 1), dtype=torch.float64, device=dev)
        self.V = f(n * cap)
        self.C = f(n * kc)
        self.U = f(n * kc)
        self.bufs = {name: f(n * s) for name in
                     ("W", "T0", "T1", "T2", "Z", "dX", "Xa", "Rb", "Q")}
        self.w1 = f(n)
        self.z1 = f(n)
        self.ptr = {k: v.data_ptr() for k, v in self.bufs.items()}
        for name in ("V", "C", "U", "w1", "z1"):
            self.ptr[name] = getattr(self, name).data_ptr()
        # small device matrices, fetched to the host in one copy
        self.off = {}
        o = 0
        for name, size in (("G1", kc * s), ("G2", cap * s), ("G3", cap * s), ("RT", s * s),
                           ("FLAG", 1), ("NRM", s * s), ("H", (cap + kc) * s), ("T", s * s),
                           ("H1", kc + 1)):
            self.off[name] = o
            o += size
        self.sm = f(o)
        self.hm = torch.empty(o, dtype=torch.float64, pin_memory=True)
        self.hin = torch.empty(o, dtype=torch.float64, pin_memory=True)
        self.hm_np = self.hm.numpy()
        self.hin_np = self.hin.numpy()
        self.smbase = self.sm.data_ptr()
        self.smp_ = {k: self.smbase + 8 * v for k, v in self.off.items()}
        sc = scratch()
        self.gram_ws = sc.get("gram", _abi.lib().pmp_gram_workspace(n, cap + kc, s), zero=True)
        self.tsqr_ws = sc.get("tsqr", _abi.lib().pmp_tsqr_workspace(n, s), zero=True)
        self.gws, self.gwb = self.gram_ws.data_ptr(), self.gram_ws.numel()
        self.tws, self.twb = self.tsqr_ws.data_ptr(), self.tsqr_ws.numel()
        self.fused = s <= 16
        if self.fused:
            self.orth_ws = sc.get("orth", _abi.lib().pmp_orth_workspace(n, cap, kc, s))
            self.ows, self.owb = self.orth_ws.data_ptr(), self.orth_ws.numel()
        self.st = _abi.stream()
        self.cstream = torch.cuda.current_stream()
        L = _abi.lib()
        self.f_gram, self.f_tsmm, self.f_tsqr = L.pmp_gram, L.pmp_tsmm, L.pmp_tsqr_r
        self.f_copy, self.f_axpby = L.pmp_copy_cols, L.pmp_axpby_cols
        self.f_defl, self.f_hls = L.pmp_host_deflate, L.pmp_host_hls_append
        self.f_orth = L.pmp_orth_step
        self.f_fold = L.pmp_fold
        self.f_step, self.f_wait, self.f_absorb = L.pmp_gcro_step, L.pmp_host_wait_flag, \
            L.pmp_gcro_absorb
        # native per-step path: results land in mapped host memory (two
        # buffers so a speculative next step never overwrites unread ones)
        self.f_cend = L.pmp_gcro_cycle_end
        self._chain_key = None
        self.native = self.fused
        if self.native:
            self.mapped = _mapped_pair(o)
            self.mptr = [b.ptr for b in self.mapped]
            self.colsbuf = np.zeros((kc + cap) * (kc + s))
        self.fold_ws = sc.get("fold", L.pmp_fold_workspace(n, kc))
        self.counting = _abi._counting
        self.timing = _abi._timing_names
        self.launches = 0
        # host scratch for the deflation helper
        self.h_rank = np.zeros(1, dtype=np.int32)
        self.h_cond = np.zeros(1)
        self.h_T = np.zeros(s * s)
        self.h_R = np.zeros(s * s)

    def _call(self, name, fn, *args):
        if self.timing and name in self.timing:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            rc = fn(*args)
            b.record()
            _abi._timed.setdefault(name, []).append((a, b, args))
        else:
            rc = fn(*args)
        if rc:
            _abi.check(rc, name)
        self.launches += 1
        if self.counting:
            _abi.COUNTERS[name] = _abi.COUNTERS.get(name, 0) + 1

    def set_active(self, active):
        """Active column list on the device without a synchronising
        pageable copy (pinned staging + async copy); returns its pointer."""
        if not hasattr(self, "act_d"):
            self.act_d = torch.empty(self.s, dtype=torch.int32, device=_dev())
            self.act_h = torch.empty(self.s, dtype=torch.int32, pin_memory=True)
        na = len(active)
        self.act_h.numpy()[:na] = active
        self.act_d[:na].copy_(self.act_h[:na], non_blocking=True)
        return self.act_d.data_ptr()

    def p(self, name, col=0):
        return self.ptr[name] + 8 * col

    def smp(self, name):
        return self.smp_[name]

    def gram(self, Vp, ldv, kv, Wp, ldw, nw, out):
        if kv == 0 or nw == 0:
            return
        self._call("pmp_gram", self.f_gram, self.n, kv, Vp, ldv, nw, Wp, ldw, self.smp_[out], self.gws,
                             self.gwb, self.st)

    def tsmm(self, Vp, ldv, kv, Hp, nc, alpha, beta, Op, ldo):
        if nc == 0:
            return
        if kv == 0:
            if beta == 0.0:
                self._call("pmp_axpby_cols", self.f_axpby, self.n, nc, 0.0, Op, ldo, None, 0.0, Op, ldo, None,
                                      self.st)
            return
        self._call("pmp_tsmm", self.f_tsmm, self.n, kv, Vp, ldv, nc, Hp, alpha, beta, Op, ldo, self.st)

    def orth(self, k, total, npass, Wp, sb, qout):
        """Fused C projection + CGS2 + Cholesky-QR2 (pmp_orth_step).  Returns
        (rank, R rows) after one fetch, falling back to Householder TSQR +
        host pivoted QR when the kernel flags a near-deficient block."""
        self._call("pmp_orth_step", self.f_orth, self.n, self.ptr["C"], self.kc, k,
                   self.ptr["V"], self.cap, total, npass, Wp, self.s, sb, qout,
                   self.smp_["G1"], self.smp_["G2"], self.smp_["G3"], self.smp_["RT"],
                   self.smp_["FLAG"], self.ows, self.owb, self.st)

    def fold(self, k, na):
        """Outer-space fold of the images in Rb / directions in dX
        (pmp_fold, one cooperative launch); returns the new dimension."""
        self._call("pmp_fold", self.f_fold, self.n, na, self.ptr["Rb"], self.s, self.ptr["dX"],
                   self.s, self.ptr["C"], self.ptr["U"], self.kc, self.kc, k, self.smp_["H"],
                   self.fold_ws.data_ptr(), self.fold_ws.numel(), self.st)
        self.fetch(("H", 1))
        return int(round(self.get("H", 1, 1)[0, 0]))

    def step(self, chain, A, q0, sb, k, total, buf):
        """Enqueue one native block step (pmp_gcro_step) whose small results
        go to mapped buffer `buf`."""
        self._chain_arrays(chain)
        st = A.structure
        off = self.off
        self._call("pmp_gcro_step", self.f_step, self.n, self.s, len(chain), self._fr, self._fc,
                   self._fv, st.rowptr.data_ptr(), st.colidx.data_ptr(), A.vals.data_ptr(),
                   self.ptr["V"], self.cap, q0, sb, self.ptr["W"], self.ptr["T0"],
                   self.ptr["T1"], self.ptr["T2"], self.ptr["C"], self.kc, k, total,
                   self.smbase, self.mptr[buf], off["G1"], off["G2"], off["G3"], off["RT"],
                   off["FLAG"],
                   self.ows, self.owb, self.st, *self._orth_events(k, total, sb))

    def _orth_events(self, k, total, sb):
        """CUDA events around the orthogonalisation kernel of a native step
        when per-kernel timing of "k_orth" is requested (bench.py)."""
        if not (self.timing and "k_orth" in self.timing):
            return (None, None)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        b.record()          # materialise the underlying cudaEvent_t handles
        _abi._timed.setdefault("k_orth", []).append((a, b, (self.n, k, total, sb)))
        return (a.cuda_event, b.cuda_event)

    def _chain_arrays(self, chain):
        key = tuple(id(F) for F in chain)
        if key != self._chain_key:
            nf = len(chain)
            arr = lambda vals: (ctypes.c_void_p * max(nf, 1))(*vals)
            self._fr = arr([F.structure.rowptr.data_ptr() for F in chain])
            self._fc = arr([F.structure.colidx.data_ptr() for F in chain])
            self._fv = arr([F.vals.data_ptr() for F in chain])
            self._chain_key = key

    def cycle_end(self, na, act_p, m, hv, k, hu, Xtp, Xp, Bp, Rp, chain, A):
        """Solution / true-residual update of a finished cycle
        (pmp_gcro_cycle_end); column norms land in NRM."""
        self._chain_arrays(chain)
        st = A.structure
        self._call("pmp_gcro_cycle_end", self.f_cend, self.n, self.s, na, act_p, self.ptr["V"],
                   self.cap, m, hv, self.ptr["U"], self.kc, k, hu, self.ptr["dX"], Xtp,
                   self.ptr["Z"], self.ptr["Xa"], Xp, Bp, self.ptr["Rb"], Rp, len(chain),
                   self._fr, self._fc, self._fv, st.rowptr.data_ptr(), st.colidx.data_ptr(),
                   A.vals.data_ptr(), self.ptr["T0"], self.ptr["T1"], self.smp_["NRM"],
                   self.gws, self.gwb, self.st)

    def inner_state(self, A, chain):
        """PmpGcroInner with the solve-constant fields filled (pointers,
        offsets, stream); the caller sets the per-cycle fields."""
        if getattr(self, "_inner", None) is None:
            self._chain_arrays(chain)
            g = _InnerState()
            g.n, g.s, g.cap, g.kc, g.ldq = self.n, self.s, self.cap, self.kc, self.kc + self.cap
            g.nfac = len(chain)
            g.fac_rowptr = ctypes.cast(self._fr, ctypes.c_void_p)
            g.fac_colidx = ctypes.cast(self._fc, ctypes.c_void_p)
            g.fac_vals = ctypes.cast(self._fv, ctypes.c_void_p)
            st = A.structure
            g.a_rowptr, g.a_colidx = st.rowptr.data_ptr(), st.colidx.data_ptr()
            g.a_vals = A.vals.data_ptr()
            for name in ("V", "W", "T0", "T1", "T2", "C"):
                setattr(g, name, self.ptr[name])
            g.d_small = self.smbase
            g.mirror[0], g.mirror[1] = self.mptr[0], self.mptr[1]
            g.offB, g.offH1, g.offH2 = self.off["G1"], self.off["G2"], self.off["G3"]
            g.offR, g.offFlag = self.off["RT"], self.off["FLAG"]
            g.orth_ws, g.orth_ws_bytes = self.ows, self.owb
            g.stream = self.st
            g.colsbuf = self.colsbuf.ctypes.data
            self.hist = np.zeros((self.cap + 2, self.s))
            g.hist = self.hist.ctypes.data
            self.f_inner = _abi.lib().pmp_gcro_inner
            self._inner = g
        return self._inner

    def cycle_ok(self, na, bs, chain, restart):
        """The device cycle handles block sizes <= 16, up to 3 factors and
        restart lengths with restart + block <= 96."""
        return 1 <= bs <= 16 and na <= 16 and len(chain) <= 3 and restart + bs <= 96

    def cycle_bufs(self):
        if getattr(self, "_cbufs", None) is None:
            self._cbufs = _CycleBufs(self)
        return self._cbufs

    def cycle_state(self, A, chain):
        """PmpGcroCycle with the solve-constant fields filled."""
        if getattr(self, "_cyc", None) is None:
            self._chain_arrays(chain)
            cb = self.cycle_bufs()
            g = _CycleState()
            g.n, g.s, g.cap, g.kc, g.nfac = self.n, self.s, self.cap, self.kc, len(chain)
            g.fac_rowptr = ctypes.cast(self._fr, ctypes.c_void_p)
            g.fac_colidx = ctypes.cast(self._fc, ctypes.c_void_p)
            g.fac_vals = ctypes.cast(self._fv, ctypes.c_void_p)
            st = A.structure
            g.a_rowptr, g.a_colidx = st.rowptr.data_ptr(), st.colidx.data_ptr()
            g.a_vals = A.vals.data_ptr()
            for name in ("V", "W", "T0", "T1", "C"):
                setattr(g, name, self.ptr[name])
            g.d_small, g.mirror = self.smbase, self.mptr[0]
            g.offB, g.offH1, g.offH2 = self.off["G1"], self.off["G2"], self.off["G3"]
            g.offR = self.off["RT"]
            g.ws, g.ws_bytes = cb.ws.data_ptr(), cb.ws.numel()
            g.stream = self.st
            g.hist_cap = cb.hist_cap
            g.d_proj = cb.d.data_ptr()
            for name in ("Bmat", "Hb", "QR", "Tau", "Cq", "Y", "Res", "Bn", "Hist"):
                setattr(g, "o" + name, cb.off[name])
            g.blocks_per_sm = _CYCLE_BPS
            g.d_istate = cb.di.data_ptr()
            self._cyc = g
        return self._cyc

    def wait(self, buf):
        rc = self.f_wait(self.mptr[buf] + 8 * self.off["FLAG"], -1.0, 60_000_000, self.st)
        if rc:
            _abi.check(rc, "pmp_host_wait_flag")

    def mget(self, buf, name, rows, cols):
        o = self.off[name]
        return self.mapped[buf].array[o:o + rows * cols].reshape(rows, cols)

    def tsqr(self, Zp, ldz, nz):
        self._call("pmp_tsqr_r", self.f_tsqr, self.n, nz, Zp, ldz, self.smp_["RT"], self.tws, self.twb, self.st)

    def put(self, name, arr):
        """Stage a small host matrix into the device small buffer."""
        a = np.ascontiguousarray(arr, dtype=np.float64).ravel()
        o = self.off[name]
        self.hin_np[o:o + a.size] = a
        self.sm[o:o + a.size].copy_(self.hin[o:o + a.size], non_blocking=True)
        return self.smp_[name]

    def fetch(self, upto=None):
        if upto is None:
            self.hm.copy_(self.sm, non_blocking=True)
        else:
            e = self.off[upto[0]] + upto[1]
            self.hm[:e].copy_(self.sm[:e], non_blocking=True)
        self.cstream.synchronize()

    def get(self, name, rows, cols):
        o = self.off[name]
        return self.hm_np[o:o + rows * cols].reshape(rows, cols)

    def copy_cols(self, nc, src, lds, sc, dst, ldd, dc):
        self._call("pmp_copy_cols", self.f_copy, self.n, nc, src, lds, sc, dst, ldd, dc, self.st)

    def axpby(self, nc, alpha, src, lds, sc, beta, dst, ldd, dc):
        self._call("pmp_axpby_cols", self.f_axpby, self.n, nc, alpha, src, lds, sc, beta, dst, ldd, dc, self.st)


def _deflate_finish(D, Zp, ldz, mz, outp, ldo, tol, report):
    """Rank-revealing QR of the n x mz block at Zp (krylov.py:79-95) from its
    TSQR factor (already fetched): host pivoted QR of R, then on the device
    Q = Z Pi R11^-1 written to outp.  Returns (rank, R[:rank] un-pivoted)."""
    RT = np.ascontiguousarray(np.triu(D.get("RT", mz, mz)))
    rc = D.f_defl(mz, RT.ctypes.data, float(tol), D.h_rank.ctypes.data, D.h_T.ctypes.data,
                  D.h_R.ctypes.data, D.h_cond.ctypes.data)
    if rc:
        _abi.check(rc, "pmp_host_deflate")
    r = int(D.h_rank[0])
    if r == 0:
        return 0, np.zeros((0, mz))
    Rout = D.h_R[:r * mz].reshape(r, mz).copy()
    T = D.h_T[:mz * r]
    if D.h_cond[0] > _REORTH_COND:
        # Q1 = Z T, then one Cholesky-QR pass restores orthogonality:
        # Q = Q1 R2^-1, R = R2 R
        D.tsmm(Zp, ldz, mz, D.put("T", T), r, 1.0, 0.0, D.p("Q"), D.s)
        D.gram(D.p("Q"), D.s, r, D.p("Q"), D.s, r, "NRM")
        D.fetch()
        G2 = D.get("NRM", r, r)
        R2 = np.linalg.cholesky(0.5 * (G2 + G2.T)).T
        R2inv = scipy.linalg.solve_triangular(R2, np.eye(r), lower=False)
        D.tsmm(D.p("Q"), D.s, r, D.put("T", R2inv), r, 1.0, 0.0, outp, ldo)
        report.reorth_passes += 1
        return r, R2 @ Rout
    D.tsmm(Zp, ldz, mz, D.put("T", T), r, 1.0, 0.0, outp, ldo)
    return r, Rout


def _project_deflate(D, k, total, npass, Wp, sb, qout, tol, report):
    """W -= C (C^T W); npass x {W -= V (V^T W)}; rank-revealing QR of W with
    the orthonormal block written to V[:, qout:] (krylov.py:156-165,
    :189-202).  C^T W, the two CGS coefficient blocks land in the small
    buffer slots G1, G2, G3 (fetched)."""
    _project_launch(D, k, total, npass, Wp, sb, qout)
    return _project_finish(D, Wp, sb, qout, tol, report)


def _project_launch(D, k, total, npass, Wp, sb, qout):
    """Enqueue the projection + QR of one block step (no host sync)."""
    s, cap, kc = D.s, D.cap, D.kc
    if D.fused:
        D.orth(k, total, npass, Wp, sb, qout)
        return
    if k:
        D.gram(D.p("C"), kc, k, Wp, s, sb, "G1")
        D.tsmm(D.p("C"), kc, k, D.smp("G1"), sb, -1.0, 1.0, Wp, s)
    for g in ("G2", "G3")[:npass]:
        D.gram(D.p("V"), cap, total, Wp, s, sb, g)
        D.tsmm(D.p("V"), cap, total, D.smp(g), sb, -1.0, 1.0, Wp, s)
    D.tsqr(Wp, s, sb)


def _project_finish(D, Wp, sb, qout, tol, report):
    """Fetch the step's small results; finish the rank-revealing QR on the
    host when the fused kernel could not (or the unfused path is used).
    Returns (rank, R[:rank] un-pivoted)."""
    s, cap = D.s, D.cap
    D.fetch(("FLAG", 1))
    if D.fused:
        if D.get("FLAG", 1, 1)[0, 0] == 0.0:
            return sb, D.get("RT", sb, sb).copy()
        report.deflation_fallbacks += 1
        D.tsqr(Wp, s, sb)
        D.fetch(("FLAG", 1))
    return _deflate_finish(D, Wp, s, sb, D.p("V", qout), cap, tol, report)


def _colnorms(D, Wp, ldw, nw):
    D.gram(Wp, ldw, nw, Wp, ldw, nw, "NRM")
    D.fetch(("NRM", nw * nw))
    g = np.diag(D.get("NRM", nw, nw)).copy()
    return np.sqrt(np.maximum(g, 0.0))


# A single solve goes through the same persistent kernel as the sequence
# windows (pmp_solve_batch, one block group); the host-driven path (k_cycle
# per cycle, host between cycles) serves what that kernel hands back
# (status 10: deflation, rank-deficient projected problem), complex systems,
# chains longer than 3 factors and PMP_SINGLE_HOST=1.
SINGLE_VIA_BATCH = _os.environ.get("PMP_SINGLE_HOST", "0")[:1] == "0"


def block_gcro_solve(A, B, P=None, cfg=None, _host=False):
    """Solve A X = B for all columns of B simultaneously (krylov.py:105-275).

    ``A`` may be a scipy matrix or a DeviceCSR; ``B`` a numpy array (the
    solution comes back as numpy) or a CUDA tensor (solution stays on the
    device)."""
    cfg = cfg or SolverConfig()
    if P is not None and not isinstance(P, Preconditioner):
        raise TypeError("P must be a Preconditioner or None")
    from .spai import _any_complex
    if _any_complex(A, B, P) or (torch.is_tensor(B) and torch.is_complex(B)):
        return _solve_complex(A, B, P, cfg)
    A = _as_dev_csr(A)
    n = A.n
    host_out = not torch.is_tensor(B)
    if host_out:
        B = np.asarray(B)
        if B.ndim == 2 and B.shape[0] != n:
            raise ValueError("right-hand side has %d rows, matrix is %dx%d" % (B.shape[0], n, n))
    Bd = _block_to_dev(B)
    if Bd.shape[0] != n:
        raise ValueError("right-hand side has %d rows, matrix is %dx%d" % (Bd.shape[0], n, n))
    if P is not None and not isinstance(P, Preconditioner):
        raise TypeError("P must be a Preconditioner or None")
    if P is not None and P.dim != n:
        raise ValueError("preconditioner dimension %d does not match system %d" % (P.dim, n))
    if SINGLE_VIA_BATCH and not _host and Bd.shape[1] >= 1 and n > 0:
        t0 = time.perf_counter()
        X, report = block_gcro_solve_batch([(A, P)], Bd, cfg=cfg, groups=1)[0]
        if not report.wall_time:   # (the record's D2H synchronised the launch)
            report.wall_time = time.perf_counter() - t0
    else:
        X, report = _solve(A, Bd, P, cfg)
    return (X.cpu().numpy() if host_out else X), report


def _solve_complex(A, B, P, cfg):
    """Complex block GCRO (krylov.py:105-275) on the real form (cplx.py):
    the 2s-column block [R(b_0), R(i b_0), ...] with the restart length and
    the outer-space dimension doubled (both count real columns), X from the
    even columns; counts and residual rows reported per complex column."""
    from . import cplx as _cx
    R = _as_dev_csr(A, cplx=True)
    n = R.complex_n
    host_out = not torch.is_tensor(B)
    Bh = np.asarray(B) if host_out else B
    vec = Bh.ndim == 1
    if Bh.shape[0] != n:
        raise ValueError("right-hand side has %d rows, matrix is %dx%d" % (Bh.shape[0], n, n))
    if P is not None:
        P = P.as_complex()
        if P.dim != n:
            raise ValueError("preconditioner dimension %d does not match system %d" % (P.dim, n))
    Br = _cx.block_to_real(Bh, pairs=True)
    cfg2 = SolverConfig(tol=cfg.tol, max_iters=cfg.max_iters,
                        outer_space_dim=2 * cfg.outer_space_dim,
                        inner_restart=2 * cfg.inner_restart, deflation_tol=cfg.deflation_tol)
    X2, rep = _solve(R, Br, P, cfg2)
    X = _cx.block_from_real(X2, 2)
    rep.matvec_count //= 2
    rep.precond_apply_count //= 2
    rep.residual_history = [np.asarray(h)[0::2].copy() for h in rep.residual_history]
    if vec:
        X = X[:, 0]
    return (X.cpu().numpy() if host_out else X), rep


class _Projected:
    """The projected least-squares problem of one cycle (krylov.py:171-212),
    factorised incrementally on the host (pmp_host_hls_append)."""

    def __init__(self, D, k, cap, na, rhs_c, S0, bs):
        self.D = D
        self.k, self.na = k, na
        self.ldq = k + cap
        self.QR = np.zeros((self.ldq, self.ldq), order="F")
        self.tau = np.zeros(self.ldq)
        self.ext = np.zeros(self.ldq, dtype=np.int32)
        self.C = np.zeros((self.ldq, na), order="F")
        self.C[:k] = rhs_c
        self.C[k:k + bs] = S0
        self.rhs0 = self.C.copy()
        self.ncols = 0
        self.Y = np.zeros((na, self.ldq))
        self.res = np.zeros(na)

    def append(self, Bmat, Hb, q0, q1, total, m):
        """Append the block columns q0:q1 of G (rows k + total); returns
        (Y, residual norms) of min ||rhs - G Y||."""
        k = self.k
        nrows = k + total
        sb = q1 - q0
        first = self.ncols == 0
        nnew = (k + sb) if first else sb
        cols = np.zeros((nrows, nnew), order="F")
        o = 0
        if first:
            cols[:k, :k] = np.eye(k)
            o = k
        if k:
            cols[:k, o:o + sb] = Bmat[:, q0:q1]
        cols[k:, o:o + sb] = Hb[:total, q0:q1]
        n1 = self.ncols + nnew
        rc = self.D.f_hls(self.ldq, self.na, self.ncols, nnew, nrows, cols.ctypes.data,
                          self.QR.ctypes.data, self.tau.ctypes.data, self.ext.ctypes.data,
                          self.C.ctypes.data, self.Y.ctypes.data, self.res.ctypes.data)
        self.ncols = n1
        Y = self.Y.ravel()[:n1 * self.na].reshape(self.na, n1).T.copy()
        if rc == 1:
            # (near) rank-deficient G: the reference's minimum-norm gelsd
            G = _build_G(k, Bmat, Hb, total, m)
            rhs = self.rhs0[:nrows]
            Y, _, _, _ = np.linalg.lstsq(G, rhs, rcond=None)
            return Y, np.linalg.norm(rhs - G @ Y, axis=0)
        if rc:
            _abi.check(rc, "pmp_host_hls_append")
        return Y, self.res.copy()


    def absorb(self, D, buf, q0, sb, total, Bmat, Hb):
        """Native fast path: fold a full-rank step (results in mapped buffer
        `buf`) into Bmat / Hb and the incremental QR (pmp_gcro_absorb)."""
        k = self.k
        nnew = (k + sb) if self.ncols == 0 else sb
        n1 = self.ncols + nnew
        off = D.off
        rc = D.f_absorb(D.mptr[buf], off["G1"], off["G2"], off["G3"], off["RT"], D.cap, k, q0,
                        sb, total, Bmat.ctypes.data, Hb.ctypes.data, self.ldq, self.na,
                        self.ncols, self.QR.ctypes.data, self.tau.ctypes.data,
                        self.ext.ctypes.data, self.C.ctypes.data, self.Y.ctypes.data,
                        self.res.ctypes.data, D.colsbuf.ctypes.data)
        self.ncols = n1
        total_new = total + sb
        m = total
        if rc == 1:
            G = _build_G(k, Bmat, Hb, total_new, m)
            rhs = self.rhs0[:k + total_new]
            Y, _, _, _ = np.linalg.lstsq(G, rhs, rcond=None)
            return Y, np.linalg.norm(rhs - G @ Y, axis=0)
        if rc:
            _abi.check(rc, "pmp_gcro_absorb")
        Y = self.Y.ravel()[:n1 * self.na].reshape(self.na, n1).T.copy()
        return Y, self.res.copy()


# the inner loop runs natively (pmp_gcro_inner) unless PMP_PY_INNER=1 selects
# the equivalent Python loop (kept for debugging and A/B comparisons)
NATIVE_INNER = __import__("os").environ.get("PMP_PY_INNER") != "1"


class _InnerState(ctypes.Structure):
    """ctypes mirror of PmpGcroInner (include/pmorb200.h)."""
    _fields_ = [(f, ctypes.c_int) for f in ("n", "s", "na", "k", "cap", "kc", "ldq")] + [
        ("tol", ctypes.c_double), ("max_iters", ctypes.c_int), ("inner_restart", ctypes.c_int),
        ("nfac", ctypes.c_int)] + [
        (f, ctypes.c_void_p) for f in ("fac_rowptr", "fac_colidx", "fac_vals", "a_rowptr",
                                       "a_colidx", "a_vals", "V", "W", "T0", "T1", "T2", "C",
                                       "d_small")] + [
        ("mirror", ctypes.c_void_p * 2)] + [
        (f, ctypes.c_int) for f in ("offB", "offH1", "offH2", "offR", "offFlag")] + [
        ("orth_ws", ctypes.c_void_p), ("orth_ws_bytes", ctypes.c_size_t),
        ("stream", ctypes.c_void_p)] + [
        (f, ctypes.c_void_p) for f in ("Bmat", "Hb", "QR", "tau", "ext", "Cq", "Y", "res",
                                       "colsbuf", "bn", "hist")] + [
        (f, ctypes.c_int) for f in ("m", "total", "ncols", "iterations", "launched", "buf")] + [
        ("prev_max", ctypes.c_double)] + [
        (f, ctypes.c_int) for f in ("matvecs", "precond_applies", "status", "steps_done")]


class _CycleState(ctypes.Structure):
    """ctypes mirror of PmpGcroCycle (include/pmorb200.h)."""
    _fields_ = [(f, ctypes.c_int) for f in ("n", "s", "cap", "kc", "ldq", "nfac")] + [
        (f, ctypes.c_void_p) for f in ("fac_rowptr", "fac_colidx", "fac_vals", "a_rowptr",
                                       "a_colidx", "a_vals", "V", "W", "T0", "T1", "C",
                                       "d_small", "mirror")] + [
        (f, ctypes.c_int) for f in ("offB", "offH1", "offH2", "offR")] + [
        ("ws", ctypes.c_void_p), ("ws_bytes", ctypes.c_size_t), ("stream", ctypes.c_void_p)] + [
        (f, ctypes.c_int) for f in ("k", "na", "sb", "max_iters", "inner_restart",
                                    "hist_cap")] + [
        ("tol", ctypes.c_double), ("d_proj", ctypes.c_void_p)] + [
        (f, ctypes.c_int) for f in ("oBmat", "oHb", "oQR", "oTau", "oCq", "oY", "oRes", "oBn",
                                    "oHist", "blocks_per_sm")] + [
        ("d_istate", ctypes.c_void_p)]


# the whole inner loop of a cycle runs in one persistent kernel
# (pmp_gcro_cycle_dev) unless PMP_DEVICE_CYCLE=0; PMP_CYCLE_BPS forces the
# blocks per SM of that kernel (diagnostics)
DEVICE_CYCLE = __import__("os").environ.get("PMP_DEVICE_CYCLE", "1") != "0"
_CYCLE_BPS = int(__import__("os").environ.get("PMP_CYCLE_BPS", "0"))


class _CycleBufs:
    """Device / pinned-host mirrors of the projected state of a device
    cycle (layout of PmpGcroCycle: Cq, bn, res, Y, hist, tau, QR, Bmat, Hb
    as doubles; the int state + ext separately)."""

    def __init__(self, D):
        s, cap, kc = D.s, D.cap, D.kc
        ldq = kc + cap
        self.hist_cap = cap + 2
        off = {}
        o = 0
        for name, size in (("Cq", ldq * s), ("Bn", s), ("Res", s), ("Y", s * ldq),
                           ("Hist", self.hist_cap * s), ("Tau", ldq), ("QR", ldq * ldq),
                           ("Bmat", kc * cap), ("Hb", cap * cap)):
            off[name] = o
            o += size
        self.off, self.size = off, o
        dev = _dev()
        self.d = torch.zeros(o, dtype=torch.float64, device=dev)
        self.h = torch.zeros(o, dtype=torch.float64, pin_memory=True)
        self.hn = self.h.numpy()
        # int state: [0..5] m, total, ncols, iterations, status, history
        # rows; [7..9] step / done / barrier flags; [16 + j] decision of
        # step j (-1 = not yet posted)
        self.nint = 16 + 128
        self.di = torch.zeros(self.nint, dtype=torch.int32, device=dev)
        self.hi = torch.zeros(self.nint, dtype=torch.int32, pin_memory=True)
        self.hin = self.hi.numpy()
        sc = scratch()
        L = _abi.lib()
        self.ws = sc.get("cycle", L.pmp_cycle_workspace(D.n, cap, kc, s))
        self.f = L.pmp_gcro_cycle_dev

    def view(self, name, size):
        o = self.off[name]
        return self.hn[o:o + size]


def _device_cycle(D, A, chain, cfg, report, k, na, bs, bn_act, prev_max, Bmat, Hb, proj,
                  last_rel, active):
    """Inner loop of one cycle in one persistent kernel (pmp_gcro_cycle_dev);
    the rare host fallbacks (status 4 / 5) continue in _native_cycle from
    the state the kernel reached.  Returns (m, total, Y, converged,
    exhausted)."""
    cb = D.cycle_bufs()
    g = D.cycle_state(A, chain)
    s, cap, ldq = D.s, D.cap, proj.ldq
    g.k, g.na, g.sb, g.ldq = k, na, bs, ldq
    g.max_iters, g.inner_restart, g.tol = cfg.max_iters, cfg.inner_restart, float(cfg.tol)
    # Q^T rhs (rhs_c ; S0) and the column norms, one pinned upload
    cq = cb.view("Cq", ldq * na)
    cq[:] = proj.C[:, :na].ravel(order="F")
    cb.view("Bn", na)[:] = bn_act
    up = cb.off["Bn"] + s
    cb.d[:up].copy_(cb.h[:up], non_blocking=True)
    it0 = report.iterations
    cb.hin[:16] = 0
    cb.hin[:4] = (0, bs, 0, it0)
    cb.hin[16:] = -1
    cb.di.copy_(cb.hi, non_blocking=True)
    D._call("pmp_gcro_cycle_dev", cb.f, ctypes.byref(g))
    cb.h.copy_(cb.d, non_blocking=True)
    cb.hi.copy_(cb.di, non_blocking=True)
    D.cstream.synchronize()
    m, total, ncols, it, st, hrows = (int(v) for v in cb.hin[:6])
    steps = it - it0
    report.iterations = it
    report.matvec_count += bs * steps
    if chain:
        report.precond_apply_count += bs * steps
    hist = cb.view("Hist", cb.hist_cap * na)
    for i in range(hrows):
        last_rel[active] = hist[i * na:(i + 1) * na]
        report.residual_history.append(last_rel.copy())
    if k:
        Bmat[:, :] = cb.view("Bmat", k * cap).reshape(k, cap)
    Hb[:, :] = cb.view("Hb", cap * cap).reshape(cap, cap)
    Y = None
    if ncols and st in (0, 2, 3):
        Y = cb.view("Y", na * ncols).reshape(na, ncols).T.copy()
    if st in (0, 2, 3):
        return m, total, Y, st == 0, False
    # host fallbacks: re-factor G (block columns absorbed so far) on the
    # host and hand the cycle to the native host loop
    proj.C[:, :] = proj.rhs0
    proj.QR[:, :] = 0.0
    proj.tau[:] = 0.0
    proj.ext[:] = 0
    proj.ncols = 0
    if m:
        proj.append(Bmat, Hb, 0, m, total, m)
    ncols = proj.ncols
    return _native_cycle(D, A, chain, cfg, report, k, na, bs, bn_act, prev_max, Bmat, Hb, proj,
                         last_rel, active, resume=(st, m, total, ncols))


def _native_cycle(D, A, chain, cfg, report, k, na, bs, bn_act, prev_max, Bmat, Hb, proj,
                  last_rel, active, resume=None):
    """Inner loop of one cycle through pmp_gcro_inner (native, GIL released
    while it runs); the rare host fallbacks (rank-deficient G: min-norm
    gelsd; near-deficient block: Householder deflation) are handled here and
    the native loop resumed.  Returns (m, total, Y, converged, exhausted)."""
    g = D.inner_state(A, chain)
    bn = np.ascontiguousarray(bn_act, dtype=np.float64)
    g.na, g.k, g.m, g.total, g.ncols = na, k, 0, bs, 0
    g.ldq = proj.ldq                      # leading dimension of this cycle's QR / C / Y
    g.launched, g.buf, g.prev_max = 0, 0, prev_max
    g.iterations, g.max_iters, g.inner_restart = report.iterations, cfg.max_iters, \
        cfg.inner_restart
    g.tol = cfg.tol
    g.Bmat, g.Hb = Bmat.ctypes.data, Hb.ctypes.data
    g.QR, g.tau, g.ext = proj.QR.ctypes.data, proj.tau.ctypes.data, proj.ext.ctypes.data
    g.Cq, g.Y, g.res = proj.C.ctypes.data, proj.Y.ctypes.data, proj.res.ctypes.data
    g.bn = bn.ctypes.data
    Y = None
    conv = exh = False
    s, cap = D.s, D.cap
    if resume is not None:
        # continue after the device cycle stopped at a host fallback
        st, g.m, g.total, g.ncols = resume
        g.iterations, g.buf = report.iterations, 0
    while True:
        if resume is not None:
            resume = None
        else:
            g.matvecs = g.precond_applies = 0
            it0 = g.iterations
            rc = D.f_inner(ctypes.byref(g))
            if rc:
                _abi.check(rc, "pmp_gcro_inner")
            if D.counting:
                _abi.COUNTERS["pmp_gcro_step"] = (_abi.COUNTERS.get("pmp_gcro_step", 0)
                                                  + g.iterations - it0 + g.launched)
            hist = D.hist.ravel()
            for i in range(g.steps_done):
                last_rel[active] = hist[i * na:(i + 1) * na]
                report.residual_history.append(last_rel.copy())
            report.iterations = g.iterations
            report.matvec_count += g.matvecs
            report.precond_apply_count += g.precond_applies
            proj.ncols = g.ncols
            if g.steps_done:
                Y = proj.Y.ravel()[:g.ncols * na].reshape(na, g.ncols).T.copy()
            st = g.status
        if st == 0:
            conv = True
            break
        if st in (2, 3):
            break
        if st == 4:
            # G (near) rank deficient: the reference's minimum-norm gelsd solve
            G = _build_G(k, Bmat, Hb, g.total, g.m)
            rhs = proj.rhs0[:k + g.total]
            Y, _, _, _ = np.linalg.lstsq(G, rhs, rcond=None)
            rn = np.linalg.norm(rhs - G @ Y, axis=0)
        else:
            # st == 5: the pending step needs the Householder deflation
            q0, q1 = g.m, g.total
            sb = q1 - q0
            buf = g.buf
            report.iterations += 1
            report.matvec_count += sb
            if chain:
                report.precond_apply_count += sb
            report.deflation_fallbacks += 1
            if k:
                Bmat[:, q0:q1] = D.mget(buf, "G1", k, sb)
            Hb[:q1, q0:q1] += D.mget(buf, "G2", q1, sb)
            Hb[:q1, q0:q1] += D.mget(buf, "G3", q1, sb)
            Wp = D.p("W")
            D.tsqr(Wp, s, sb)
            D.fetch(("FLAG", 1))
            bs_next, Rn = _deflate_finish(D, Wp, s, sb, D.p("V", q1), cap, cfg.deflation_tol,
                                          report)
            Hb[q1:q1 + bs_next, q0:q1] = Rn
            m, total = q1, q1 + bs_next
            Y, rn = proj.append(Bmat, Hb, q0, q1, total, m)
            g.m, g.total, g.ncols = m, total, proj.ncols
            g.launched, g.iterations = 0, report.iterations
            exh = bs_next == 0
        est = _safe_rel(rn, bn_act)
        g.prev_max = float(np.max(est)) if est.size else 0.0
        last_rel[active] = est
        report.residual_history.append(last_rel.copy())
        if bool(np.all(est <= cfg.tol)):
            conv = True
            break
        if exh:
            break
    return g.m, g.total, Y, conv, exh


_MAPPED = {}


def _mapped_pair(ndoubles):
    """Two mapped host buffers of at least `ndoubles`, cached per thread."""
    import threading
    key = threading.get_ident()
    pair = _MAPPED.get(key)
    if pair is None or pair[0].array.size < ndoubles:
        size = max(ndoubles, 2 * (pair[0].array.size if pair else 0))
        pair = [_abi.MappedBuffer(size), _abi.MappedBuffer(size)]
        _MAPPED[key] = pair
    return pair


def _build_G(k, Bmat, Hb, total, m):
    G = np.zeros((k + total, k + m))
    if k:
        G[:k, :k] = np.eye(k)
        G[:k, k:] = Bmat[:, :m]
    G[k:, k:] = Hb[:total, :m]
    return G


import os as _os

PROFILE = {}                      # phase -> host seconds (PMP_PROFILE=1)
_PROF_ON = _os.environ.get("PMP_PROFILE") == "1"
_last_tick = [0.0]


def _tick(name):
    if _PROF_ON:
        t = time.perf_counter()
        acc = PROFILE.setdefault(name, [0.0, 0])
        acc[0] += t - _last_tick[0]
        acc[1] += 1
        _last_tick[0] = t


def _solve(A, B, P, cfg):
    n, s = B.shape
    t_start = time.perf_counter()
    _last_tick[0] = t_start
    report = SolveReport()
    cap = cfg.inner_restart + 2 * s + 2
    kc = cfg.outer_space_dim + s
    D = _Dev(n, s, cap, kc)
    _tick("setup-alloc")
    dev = _dev()
    X = torch.zeros(n, s, dtype=torch.float64, device=dev)
    Xt = torch.zeros(n, s, dtype=torch.float64, device=dev)
    R = B.clone()
    Xp, Xtp, Rp, Bp = X.data_ptr(), Xt.data_ptr(), R.data_ptr(), B.data_ptr()
    bnorms = _colnorms(D, Bp, s, s)
    _tick("setup-norms")
    last_rel = np.where(bnorms > 0, 1.0, 0.0)
    report.residual_history.append(last_rel.copy())
    active = np.flatnonzero(bnorms > 0)
    prev_norms = bnorms.copy()     # ||R[:, j]|| as of the last true residual
    tmp = [D.bufs["T0"], D.bufs["T1"]]
    chain = P.factors() if P is not None else []
    spmm = _abi.lib().pmp_spmm
    T2 = D.p("T2")

    def op(Vp, ldv, sb, Wp):
        # W = A P V: the preconditioner chain right to left, then A
        # (krylov.py:140-147; spai.py:82-89)
        src, lds = Vp, ldv
        for i, F in enumerate(reversed(chain)):
            dst = T2 if i == len(chain) - 1 else D.p("T%d" % (i % 2))
            st = F.structure
            D._call("pmp_spmm", spmm, st.n, st.rowptr.data_ptr(), st.colidx.data_ptr(), F.vals.data_ptr(), sb,
                       src, lds, 1.0, 0.0, None, 0, dst, s, D.st)
            src, lds = dst, s
        st = A.structure
        D._call("pmp_spmm", spmm, st.n, st.rowptr.data_ptr(), st.colidx.data_ptr(), A.vals.data_ptr(), sb,
                   src, lds, 1.0, 0.0, None, 0, Wp, s, D.st)


    k = 0          # outer-space dimension (columns of C / U in use)
    while active.size and report.iterations < cfg.max_iters:
        _tick("setup/cycle-end")
        na = active.size
        act_p = D.set_active(active)
        start_rel = _safe_rel(prev_norms[active], bnorms[active])
        # Ract -> Z buffer (n x na, ld s);  Z0 = Ract - C (C^T Ract)
        D.copy_cols(na, Rp, s, act_p, D.p("Z"), s, None)
        bs, S0 = _project_deflate(D, k, 0, 0, D.p("Z"), na, 0, cfg.deflation_tol, report)
        rhs_c = D.get("G1", k, na).copy() if k else np.zeros((0, na))
        if bs == 0:
            raise SolverBreakdown(
                "projected residual block vanished with %d unconverged column(s)" % na)
        Hb = np.zeros((cap, cap))
        Bmat = np.zeros((k, cap))
        proj = _Projected(D, k, cap, na, rhs_c, S0, bs)
        m = 0
        total = bs
        Y = None
        _tick("cycle-start")
        exhausted = False
        cycle_converged = False
        bn_act = bnorms[active]
        Wp = D.p("W")
        Vp = D.p("V")
        Cp = D.p("C")
        launched = False   # the current step's kernels are already enqueued
        buf = 0            # mapped result buffer of the pending native step
        prev_max = float(np.max(start_rel)) if start_rel.size else 0.0
        if D.native and DEVICE_CYCLE and D.cycle_ok(na, bs, chain, cfg.inner_restart):
            m, total, Y, cycle_converged, exhausted = _device_cycle(
                D, A, chain, cfg, report, k, na, bs, bn_act, prev_max, Bmat, Hb, proj,
                last_rel, active)
        elif D.native and NATIVE_INNER:
            m, total, Y, cycle_converged, exhausted = _native_cycle(
                D, A, chain, cfg, report, k, na, bs, bn_act, prev_max, Bmat, Hb, proj,
                last_rel, active)
        while (report.iterations < cfg.max_iters and not cycle_converged and not exhausted
               and m < cfg.inner_restart and D.native and not NATIVE_INNER):
            # native fast path: two library calls per block step
            q0, q1 = m, total
            sb = q1 - q0
            if not launched:
                D.step(chain, A, q0, sb, k, total, buf)
            launched = False
            report.iterations += 1
            if chain:
                report.precond_apply_count += sb
            report.matvec_count += sb
            D.wait(buf)
            ms = D.mapped[buf].array
            if ms[D.off["FLAG"]] == 0.0:
                bs_next = sb
                m_new, total_new = total, total + sb
                # enqueue the next step before the host-side projected solve;
                # if that solve declares convergence the speculative step is
                # discarded (it only writes scratch and V columns >= total)
                # (skipped when the last estimate is within 20x of tol: this
                # step will very likely converge, the speculation be wasted)
                if (report.iterations < cfg.max_iters and m_new < cfg.inner_restart
                        and prev_max > 20.0 * cfg.tol):
                    D.step(chain, A, m_new, sb, k, total_new, buf ^ 1)
                    launched = True
                Y, rn = proj.absorb(D, buf, q0, sb, total, Bmat, Hb)
                m, total = m_new, total_new
                if launched:
                    buf ^= 1
            else:
                # Cholesky could not decide the rank: Householder fallback
                report.deflation_fallbacks += 1
                if k:
                    Bmat[:, q0:q1] = D.mget(buf, "G1", k, sb)
                Hb[:total, q0:q1] += D.mget(buf, "G2", total, sb)
                Hb[:total, q0:q1] += D.mget(buf, "G3", total, sb)
                D.tsqr(Wp, s, sb)
                D.fetch(("FLAG", 1))
                bs_next, Rn = _deflate_finish(D, Wp, s, sb, D.p("V", total), cap,
                                              cfg.deflation_tol, report)
                Hb[total:total + bs_next, q0:q1] = Rn
                m = total
                total += bs_next
                Y, rn = proj.append(Bmat, Hb, q0, q1, total, m)
            est = _safe_rel(rn, bn_act)
            prev_max = float(np.max(est)) if est.size else 0.0
            last_rel[active] = est
            report.residual_history.append(last_rel.copy())
            cycle_converged = bool(np.all(est <= cfg.tol))
            exhausted = bs_next == 0
        while (report.iterations < cfg.max_iters and not cycle_converged and not exhausted
               and m < cfg.inner_restart and not D.native):
            q0, q1 = m, total
            sb = q1 - q0
            if not launched:
                op(D.p("V", q0), cap, sb, Wp)
                _project_launch(D, k, total, 2, Wp, sb, total)
            launched = False
            report.iterations += 1
            if chain:
                report.precond_apply_count += sb
            report.matvec_count += sb
            fb0 = report.deflation_fallbacks
            bs_next, Rn = _project_finish(D, Wp, sb, total, cfg.deflation_tol, report)
            fast = D.fused and bs_next == sb and report.deflation_fallbacks == fb0
            if k:
                Bmat[:, q0:q1] = D.get("G1", k, sb)
            Hb[:total, q0:q1] += D.get("G2", total, sb)
            Hb[:total, q0:q1] += D.get("G3", total, sb)
            Hb[total:total + bs_next, q0:q1] = Rn
            m = total
            total += bs_next
            # enqueue the next step before the host solves the projected
            # problem: if that solve declares convergence the speculative
            # step is simply discarded (it only writes scratch and columns
            # of V beyond `total`)
            if (fast and bs_next > 0 and report.iterations < cfg.max_iters
                    and m < cfg.inner_restart):
                op(D.p("V", m), cap, bs_next, Wp)
                _project_launch(D, k, total, 2, Wp, bs_next, total)
                launched = True
            Y, rn = proj.append(Bmat, Hb, q0, q1, total, m)
            est = _safe_rel(rn, bn_act)
            last_rel[active] = est
            report.residual_history.append(last_rel.copy())
            cycle_converged = bool(np.all(est <= cfg.tol))
            exhausted = bs_next == 0

        _tick("inner")
        if Y is None:
            break

        # dXt = V Y_v + U Y_u ; Xt[:, active] += dXt     (krylov.py:221-224)
        # X = P Xt ; R = B - A X                          (krylov.py:225-233)
        # (one native call enqueues the whole chain; pmp_gcro_cycle_end)
        hv = D.put("H", Y[k:])
        hu = D.put("G1", Y[:k]) if k else None
        D.cycle_end(na, act_p, m, hv, k, hu, Xtp, Xp, Bp, Rp, chain, A)
        if P is not None:
            report.precond_apply_count += na
        report.matvec_count += na
        D.fetch(("NRM", na * na))
        tn = np.sqrt(np.maximum(np.diag(D.get("NRM", na, na)), 0.0))
        _tick("cycle-end-resid")
        prev_norms[active] = tn
        true_rel = _safe_rel(tn, bn_act)
        last_rel[active] = true_rel
        report.residual_history.append(last_rel.copy())

        still = true_rel > cfg.tol
        if exhausted and np.all(still) and np.all(true_rel >= start_rel * (1 - 1e-10)):
            raise SolverBreakdown(
                "Krylov subspace exhausted without residual reduction "
                "(%d column(s) above tolerance)" % int(np.sum(still)))

        # fold the cycle's directions into the outer space (krylov.py:244-269);
        # skipped when no further cycle can run -- (U, C) are never read again
        if np.any(still) and report.iterations < cfg.max_iters:
            G = _build_G(k, Bmat, Hb, total, m)
            img = G @ Y
            D.tsmm(Vp, cap, total, D.put("H", img[k:]), na, 1.0, 0.0, D.p("Rb"), s)
            if k:
                D.tsmm(Cp, kc, k, D.put("G1", img[:k]), na, 1.0, 1.0, D.p("Rb"), s)
            kk = D.fold(k, na)
            _tick("fold")
            if kk > cfg.outer_space_dim:
                drop = kk - cfg.outer_space_dim
                keep = cfg.outer_space_dim
                for name in ("C", "U"):
                    _shift_left(D, name, kc, drop, keep)
                kk = keep
            k = kk
        active = active[still]

    _tick("setup/cycle-end")
    report.converged = active.size == 0
    report.wall_time = time.perf_counter() - t_start
    report.device_launches = D.launches
    return X, report


def _shift_left(D, name, kc, drop, keep):
    """Keep the last `keep` columns of the outer matrix (krylov.py:267-269),
    staging through a scratch block so the copy never overlaps itself."""
    n = D.n
    tmp = torch.empty(max(n * keep, 1), dtype=torch.float64, device=_dev())
    D.copy_cols(keep, D.p(name, drop), kc, None, tmp.data_ptr(), keep, None)
    D.copy_cols(keep, tmp.data_ptr(), keep, None, D.p(name), kc, None)


def gcro_solve(A, b, P=None, cfg=None):
    """Single right-hand side: the 1-column block solve, iterate for
    iterate (krylov.py:278-290)."""
    if torch.is_tensor(b):
        if b.dim() != 1:
            raise ValueError("gcro_solve expects a vector; use block_gcro_solve for blocks")
        X, report = block_gcro_solve(A, b[:, None], P=P, cfg=cfg)
    else:
        b = np.asarray(b)
        if b.ndim != 1:
            raise ValueError("gcro_solve expects a vector; use block_gcro_solve for blocks")
        X, report = block_gcro_solve(A, b[:, None], P=P, cfg=cfg)
    report.residual_history = [float(r[0]) for r in report.residual_history]
    return X[:, 0], report


# ---------------------------------------------------------------------------
# whole solves on the device, several systems per launch (pmp_solve_batch)
# ---------------------------------------------------------------------------

class _SysDesc(ctypes.Structure):
    """ctypes mirror of PmpSysDesc (include/pmorb200.h)."""
    _fields_ = [("nfac", ctypes.c_int), ("fac_rowptr", ctypes.c_void_p * 3),
                ("fac_colidx", ctypes.c_void_p * 3),
                ("fac_vals", ctypes.c_void_p * 3)] + [
        (f, ctypes.c_void_p) for f in ("a_rowptr", "a_colidx", "a_vals", "B", "X")]


class _SolveBatchArgs(ctypes.Structure):
    """ctypes mirror of PmpSolveBatch (include/pmorb200.h)."""
    _fields_ = [(f, ctypes.c_int) for f in (
        "n", "s", "cap", "kc", "outer_dim", "inner_restart", "max_iters", "groups",
        "gsz", "rows_per_block", "hist_cap", "log_cap", "isz")] + [
        ("tol", ctypes.c_double), ("d_sys", ctypes.c_void_p), ("d_ws", ctypes.c_void_p),
        ("wsz", ctypes.c_size_t), ("d_istate", ctypes.c_void_p)] + [
        (f, ctypes.c_size_t) for f in ("oV", "oC", "oU", "oW", "oT0", "oT1", "oQ1", "oXt", "oR",
                                       "oDX", "oRB", "oZ", "oPart", "oGout", "oSbuf", "oProj",
                                       "oLog", "oAux")] + [
        (f, ctypes.c_int) for f in ("pBmat", "pHb", "pCq", "pY", "pRes", "pBn", "pHist",
                                    "pCtl")] + [
        ("nsys", ctypes.c_int), ("d_queue", ctypes.c_void_p), ("d_result", ctypes.c_void_p),
        ("d_result_log", ctypes.c_void_p), ("stream", ctypes.c_void_p)]


_SOLVE_ISZ = 256
_SOLVE_RSZ = 8       # ints per system record (PmpSolveBatch::d_result)
_SOLVE_FALLBACK = 10
# reason code -> count of systems handed back to the host path (diagnostics:
# 1 cycle-start QR needs deflation, 2 projected problem rank deficient,
# 3 block step needs deflation, 4 fold drop test ambiguous, 5 fold CholQR)
FALLBACK_REASONS = {}


def _solve_layout(n, s, cap, kc, gsz, hist_cap, log_cap, ctl=0):
    """Per-system workspace layout of pmp_solve_batch (offsets in doubles);
    ``ctl`` doubles for the control block's state (pmp_solve_ctl_doubles)."""
    def al(x):
        return (x + 31) // 32 * 32
    ldq = kc + cap
    kmax = (kc + cap + s) * s
    proj = {}
    o = 32          # (offset 0 is reserved: pCtl = 0 means "not provided")
    for name, size in (("pCq", ldq * s), ("pBn", s), ("pRes", s), ("pY", s * ldq),
                       ("pHist", hist_cap * s), ("pBmat", kc * cap), ("pHb", cap * cap),
                       ("pCtl", ctl)):
        proj[name] = o
        o += al(size)
    proj_size = o
    off = {}
    o = 0
    for name, size in (("oV", n * cap), ("oC", n * kc), ("oU", n * kc)) + tuple(
            (nm, n * s) for nm in ("oW", "oT0", "oT1", "oQ1", "oXt", "oR", "oDX", "oRB", "oZ")) + (
            ("oPart", (gsz + 1) * kmax), ("oGout", kmax), ("oSbuf", 2 * (kc + 2 * cap + s) * s),
            ("oProj", proj_size), ("oLog", log_cap * s), ("oAux", 64 + (kc + cap) * s)):
        off[name] = o
        o += al(size)
    return off, proj, o


def block_gcro_solve_batch(systems, B, cfg=None, groups=None):
    """Solve A_i X_i = B for every (A_i, P_i) in ``systems`` (krylov.py:105-275
    for each) in ONE persistent kernel (pmp_solve_batch): ``groups`` block
    groups share the GPU, each solving one system at a time and taking the
    next unsolved one from a device queue when it finishes.  B is an n x s
    CUDA tensor shared by all systems.  Returns [(X_i, SolveReport_i)] in
    order.  Systems the device path hands back (status 10: deflation /
    rank-deficient projected problem / an ambiguous drop test) are
    re-solved on the host-driven path."""
    cfg = cfg or SolverConfig()
    Bd = _block_to_dev(B)
    n, s = Bd.shape
    if not systems:
        return []
    nsys = len(systems)
    groups = groups or BATCH_GROUPS
    groups = max(1, min(groups, nsys))
    L = _abi.lib()
    cap = cfg.inner_restart + 2 * s + 2
    kc = cfg.outer_space_dim + s
    ok = (s <= 16 and cfg.inner_restart + s <= 96 and cfg.outer_space_dim + s <= kc)
    chains = []
    from .spai import _any_complex
    for A, P in systems:
        if P is not None and not isinstance(P, Preconditioner):
            raise TypeError("P must be a Preconditioner or None")
        chains.append(P.factors() if P is not None else [])
    if any(_any_complex(A, P) for A, P in systems):
        return [block_gcro_solve(A, Bd, P=P, cfg=cfg, _host=True) for A, P in systems]
    if not ok or max(len(c) for c in chains) > 3:
        return [block_gcro_solve(A, Bd, P=P, cfg=cfg, _host=True) for A, P in systems]
    gsz = ctypes.c_int()
    rows = ctypes.c_int()
    cached = ctypes.c_int()
    smem = ctypes.c_size_t()
    while groups > 1 and L.pmp_solve_geometry(n, s, cap, kc, cfg.inner_restart, groups,
                                              ctypes.byref(gsz), ctypes.byref(rows),
                                              ctypes.byref(cached), ctypes.byref(smem)):
        groups -= 1
    rc = L.pmp_solve_geometry(n, s, cap, kc, cfg.inner_restart, groups, ctypes.byref(gsz),
                              ctypes.byref(rows), ctypes.byref(cached), ctypes.byref(smem))
    if rc:
        return [block_gcro_solve(A, Bd, P=P, cfg=cfg, _host=True) for A, P in systems]
    hist_cap = cap + 2
    log_cap = 2 * cfg.max_iters + 4
    off, poff, wsz = _solve_layout(n, s, cap, kc, gsz.value, hist_cap, log_cap,
                                   int(L.pmp_solve_ctl_doubles(s, kc, cap, cfg.inner_restart)))
    dev = _dev()
    sc = scratch()
    ws = sc.get("solve_ws", 8 * wsz * groups).view(torch.float64)
    ist = sc.get("solve_ist", 4 * _SOLVE_ISZ * groups).view(torch.int32)
    rlen = 2 + log_cap * s
    rint = sc.get("solve_rint", 4 * (_SOLVE_RSZ * nsys + 1)).view(torch.int32)
    rdbl = sc.get("solve_rdbl", 8 * rlen * nsys).view(torch.float64)
    sysd = (_SysDesc * nsys)()
    d_sys = torch.empty(ctypes.sizeof(sysd), dtype=torch.uint8, device=dev)
    h_sys = torch.empty(ctypes.sizeof(sysd), dtype=torch.uint8, pin_memory=True)
    args = _SolveBatchArgs()
    args.n, args.s, args.cap, args.kc = n, s, cap, kc
    args.outer_dim, args.inner_restart, args.max_iters = (cfg.outer_space_dim,
                                                          cfg.inner_restart, cfg.max_iters)
    args.groups, args.gsz, args.rows_per_block = groups, gsz.value, rows.value
    args.hist_cap, args.log_cap, args.isz, args.tol = hist_cap, log_cap, _SOLVE_ISZ, float(cfg.tol)
    args.d_sys, args.d_ws, args.wsz = d_sys.data_ptr(), ws.data_ptr(), wsz
    args.d_istate = ist.data_ptr()
    for k_, v in off.items():
        setattr(args, k_, v)
    for k_, v in poff.items():
        setattr(args, k_, v)
    args.nsys = nsys
    args.d_result = rint.data_ptr()
    args.d_queue = rint.data_ptr() + 4 * _SOLVE_RSZ * nsys
    args.d_result_log = rdbl.data_ptr()
    args.stream = _abi.stream()
    stream = torch.cuda.current_stream()
    X_block = torch.empty(nsys, n, s, dtype=torch.float64, device=dev)   # one allocation
    Xs = []
    keep = []   # device operands must outlive the launch
    for i, (A, P) in enumerate(systems):
        A = _as_dev_csr(A)
        keep.append(A)
        st = A.structure
        d = sysd[i]
        d.nfac = len(chains[i])
        for j, F in enumerate(chains[i]):
            fs = F.structure
            d.fac_rowptr[j] = fs.rowptr.data_ptr()
            d.fac_colidx[j] = fs.colidx.data_ptr()
            d.fac_vals[j] = F.vals.data_ptr()
        d.a_rowptr, d.a_colidx, d.a_vals = (st.rowptr.data_ptr(), st.colidx.data_ptr(),
                                            A.vals.data_ptr())
        X = X_block[i]
        Xs.append(X)
        d.B, d.X = Bd.data_ptr(), X.data_ptr()
    ctypes.memmove(h_sys.data_ptr(), ctypes.addressof(sysd), ctypes.sizeof(sysd))
    d_sys.copy_(h_sys, non_blocking=True)
    ist.zero_()
    if _abi._counting:
        _abi.COUNTERS["pmp_solve_batch"] = _abi.COUNTERS.get("pmp_solve_batch", 0) + 1
    if _abi._timing_names and "pmp_solve_batch" in _abi._timing_names:
        ea = torch.cuda.Event(enable_timing=True)
        eb = torch.cuda.Event(enable_timing=True)
        ea.record()
        _abi.check(L.pmp_solve_batch(ctypes.byref(args)), "pmp_solve_batch")
        eb.record()
        _abi._timed.setdefault("pmp_solve_batch", []).append((ea, eb, (n, s, nsys)))
    else:
        _abi.check(L.pmp_solve_batch(ctypes.byref(args)), "pmp_solve_batch")
    h_rint = torch.empty(_SOLVE_RSZ * nsys, dtype=torch.int32, pin_memory=True)
    h_rint.copy_(rint[:_SOLVE_RSZ * nsys], non_blocking=True)
    stream.synchronize()
    recs = h_rint.numpy().reshape(nsys, _SOLVE_RSZ).copy()
    out = [None] * nsys
    fallback = []
    done = []
    for i in range(nsys):
        if recs[i, 0] == _SOLVE_FALLBACK:
            fallback.append(i)
            FALLBACK_REASONS[int(recs[i, 1])] = FALLBACK_REASONS.get(int(recs[i, 1]), 0) + 1
        else:
            done.append(i)
    if done:
        # one gather + one D2H for every solved system's bytes and residual log
        rv = rdbl[:rlen * nsys].view(nsys, rlen)
        parts = [rv[i, :2 + int(recs[i, 4]) * s] for i in done]
        flat = torch.cat(parts).cpu().numpy()
        o = 0
        for i in done:
            rows_ = int(recs[i, 4])
            seg = flat[o:o + 2 + rows_ * s]
            o += seg.size
            rep = SolveReport()
            # one copy per system; the history rows are views of it
            rep.residual_history = list(seg[2:].reshape(rows_, s).copy())
            rep.iterations = int(recs[i, 2])
            rep.converged = int(recs[i, 3]) == 0
            rep.matvec_count = int(recs[i, 5])
            rep.precond_apply_count = int(recs[i, 6])
            rep.device_launches = 1
            # SURVEY.md 8(d)'s unit (block CGS2 reads [C | V] four times per
            # step) and the strict every-operand-once figure of round 1
            rep.algorithmic_bytes = float(seg[1])
            rep.algorithmic_bytes_strict = float(seg[0])
            out[i] = (Xs[i], rep)
    for i in fallback:
        A, P = systems[i]
        out[i] = block_gcro_solve(A, Bd, P=P, cfg=cfg, _host=True)
    return out


# systems per persistent solve launch (PMP_BATCH_GROUPS overrides)
BATCH_GROUPS = int(_os.environ.get("PMP_BATCH_GROUPS", "6"))
