"""Sparse approximate inverse on the B200 -- same API as the reference's
``pmorprec.spai`` (spai.py:37-373), computed by libpmorb200.

``spai_build`` (spai.py:341-364) runs, entirely on the device:
  level-0 pattern gather (pmp_pattern_l0)                     spai.py:182-207
  per-column least squares, tiered by subproblem size
  (pmp_ls_columns: warp / CTA / global-memory teams)          spai.py:229-292
  [level 1] selection of columns with resid > ep, two-hop
  augmentation (pmp_augment) and a second solve pass           spai.py:210-222, :287-290
  CSC -> CSR of the factor (pmp_permute over a cached
  transpose plan of the pattern)                               spai.py:295-315
The per-pattern plan (size tiers of the |J| x |I| subproblems) and the
transpose are computed once and cached on the pattern, so every later
build over the same structure -- the SPAI-update sequence -- is a fixed
list of kernel launches with no host synchronisation.
"""

import json
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import scipy.sparse as sp
import torch

from . import _abi, mmio
from .device import (DeviceCSR, DevicePattern, Structure, _dev, i32, level0_pattern, scratch)

# ---------------------------------------------------------------------------
# configs and stats (spai.py:131-171)
# ---------------------------------------------------------------------------


@dataclass
class SpaiConfig:
    """Knobs of the sparse-approximate-inverse build (spai.py:131-150)."""

    ep: float = 1e-4
    pattern_level: int = 1
    max_fill_per_column: int = 80

    def __post_init__(self):
        if self.ep <= 0:
            raise ValueError("ep must be positive")
        if self.pattern_level not in (0, 1):
            raise ValueError("pattern_level must be 0 or 1")


class BuildStats:
    """Per-column diagnostics of a build (spai.py:153-171).  Device results
    are copied to the host lazily, on first access."""

    def __init__(self, resid=None, flags=None, augmented=0, t_events=None, seconds=None,
                 share=1, stride=1):
        self._share = share   # builds that shared the timed interval
        # complex builds solve the real form's 2n columns: column 2j is the
        # complex column j (cplx.py), so every other entry is reported
        if stride > 1:
            resid = resid[::stride].contiguous() if resid is not None else None
            flags = flags[::stride].contiguous() if flags is not None else None
        self._resid = resid
        self._flags = flags
        self._aug = augmented
        self._events = t_events
        self._seconds = seconds
        self._res_host = None
        self._def = None

    @property
    def residuals(self):
        if self._res_host is None:
            self._res_host = (self._resid.cpu().numpy() if self._resid is not None
                              else np.zeros(0))
        return self._res_host

    @property
    def augmented_columns(self):
        return int(self._aug)

    @property
    def rank_deficient_columns(self):
        if self._def is None:
            if self._flags is None:
                self._def = 0
            else:
                cnt = torch.zeros(1, dtype=torch.int32, device=self._flags.device)
                _abi.call("pmp_count_flags", self._flags.numel(), _abi.ptr(self._flags), 1,
                          _abi.ptr(cnt), _abi.stream())
                self._def = int(cnt.item())
        return self._def

    @property
    def seconds(self):
        if self._seconds is None and self._events is not None:
            a, b = self._events
            b.synchronize()
            self._seconds = a.elapsed_time(b) / 1e3 / self._share
        return float(self._seconds or 0.0)

    def summary(self):
        res = np.asarray(self.residuals, dtype=float)
        return {
            "columns": int(res.size),
            "max_residual": float(res.max()) if res.size else 0.0,
            "mean_residual": float(res.mean()) if res.size else 0.0,
            "augmented_columns": self.augmented_columns,
            "rank_deficient_columns": self.rank_deficient_columns,
            "seconds": self.seconds,
        }


# ---------------------------------------------------------------------------
# preconditioner object (spai.py:37-128)
# ---------------------------------------------------------------------------


def _as_dev_csr(M, cplx=False):
    """Device CSR of M; complex inputs (or ``cplx``) as their real form R(M)
    (cplx.py)."""
    from . import cplx as _cx
    if isinstance(M, DeviceCSR):
        if cplx and not M.cplx:
            return _cx.realify_csr(M.to_scipy())
        return M
    if cplx or _cx.is_complex_host(M):
        return _cx.realify_csr(M)
    return DeviceCSR.from_scipy(M)


def _any_complex(*ms):
    from . import cplx as _cx
    for M in ms:
        if M is None:
            continue
        if isinstance(M, Preconditioner):
            if M.cplx:
                return True
        elif _cx.is_complex(M):
            return True
    return False


class Preconditioner:
    """Right preconditioner: explicit device CSR or factored chain
    Q * base, applied as successive SpMMs (never materialised;
    spai.py:37-101)."""

    def __init__(self, matrix=None, q=None, base=None):
        if matrix is not None:
            if q is not None or base is not None:
                raise ValueError("give either an explicit matrix or (q, base)")
            matrix = _as_dev_csr(matrix)
            self.matrix, self.q, self.base = matrix, None, None
        else:
            if q is None or base is None:
                raise ValueError("factored form needs both q and base")
            q = _as_dev_csr(q, cplx=base.cplx)
            if q.cplx and not base.cplx:
                base = base.as_complex()
            if q.complex_n != base.dim:
                raise ValueError("factor dimension does not match base preconditioner")
            self.matrix, self.q, self.base = None, q, base

    @property
    def kind(self):
        return "explicit" if self.matrix is not None else "factored"

    @property
    def cplx(self):
        """Complex preconditioner (factors held as real forms, cplx.py)."""
        return (self.matrix if self.matrix is not None else self.q).cplx

    def as_complex(self):
        """The same operator on complex vectors (real factors realified)."""
        if self.cplx:
            return self
        if self.matrix is not None:
            return Preconditioner(matrix=_as_dev_csr(self.matrix, cplx=True))
        return Preconditioner(q=_as_dev_csr(self.q, cplx=True), base=self.base.as_complex())

    @property
    def dim(self):
        return (self.matrix if self.matrix is not None else self.q).complex_n

    @property
    def depth(self):
        return 1 if self.matrix is not None else 1 + self.base.depth

    @classmethod
    def identity(cls, n):
        return cls(matrix=sp.identity(n, format="csr"))

    def factors(self):
        """Device factors outermost first: P = f[0] @ ... @ f[-1]."""
        if self.matrix is not None:
            return [self.matrix]
        return [self.q] + self.base.factors()

    def apply_dev(self, X, ldx, s, Y, ldy, tmp):
        """Y = P X on raw device pointers; ``tmp`` = two scratch tensors of at
        least n*s doubles (only used for chains)."""
        f = self.factors()
        src, lds = X, ldx
        for i, F in enumerate(reversed(f)):
            last = i == len(f) - 1
            dst, ldd = (Y, ldy) if last else (_abi.ptr(tmp[i % 2]), s)
            F.spmm(src, lds, s, dst, ldd)
            src, lds = dst, ldd

    def apply(self, V):
        from . import cplx as _cx
        host = not torch.is_tensor(V)
        if self.cplx or (host and _cx.is_complex_host(V)) or (
                torch.is_tensor(V) and torch.is_complex(V)):
            P = self.as_complex()
            n = P.dim
            vec = (np.ndim(V) == 1) if host else V.dim() == 1
            Vr = _cx.block_to_real(V, pairs=False)
            if Vr.shape[0] != 2 * n:
                raise ValueError("preconditioner is %dx%d, block has %d rows"
                                 % (n, n, Vr.shape[0] // 2))
            s = Vr.shape[1]
            Y = torch.empty_like(Vr)
            tmp = [torch.empty_like(Vr), torch.empty_like(Vr)] if P.depth > 1 else None
            P.apply_dev(_abi.ptr(Vr), s, s, _abi.ptr(Y), s, tmp)
            out = _cx.block_from_real(Y, 1)
            if vec:
                out = out[:, 0]
            return out.cpu().numpy() if host else out
        Vd = _block_to_dev(V)
        n, s = Vd.shape
        if n != self.dim:
            raise ValueError("preconditioner is %dx%d, block has %d rows" % (self.dim, self.dim, n))
        Y = torch.empty_like(Vd)
        tmp = [torch.empty_like(Vd), torch.empty_like(Vd)] if self.depth > 1 else None
        self.apply_dev(_abi.ptr(Vd), s, s, _abi.ptr(Y), s, tmp)
        return Y.cpu().numpy() if host else Y

    def save(self, directory, stats_summary=None):
        """Persist the chain as ordered ``factor_NN.mtx`` files plus the
        ``preconditioner.json`` sidecar, in the reference's layout
        (spai.py:103-117) so either side can load the other's files."""
        directory = Path(directory)
        directory.mkdir(parents=True, exist_ok=True)
        files = []
        for i, F in enumerate(self.factors()):
            name = "factor_%02d.mtx" % i
            mmio.write_matrix_market(F.to_scipy(), directory / name)
            files.append(name)
        sidecar = {"kind": self.kind, "factors": files}
        if stats_summary:
            sidecar["stats"] = stats_summary
        with open(directory / "preconditioner.json", "w") as fh:
            json.dump(sidecar, fh, indent=2, sort_keys=True)
            fh.write("\n")

    @classmethod
    def load(cls, directory):
        """Rebuild the chain saved by ``save`` (here or by the reference,
        spai.py:119-128); factors go straight to the device."""
        directory = Path(directory)
        with open(directory / "preconditioner.json") as fh:
            sidecar = json.load(fh)
        mats = [mmio.read_matrix_market(directory / name) for name in sidecar["factors"]]
        pre = cls(matrix=mats[-1])
        for Q in reversed(mats[:-1]):
            pre = cls(q=Q, base=pre)
        return pre

    def materialize(self):
        """Explicit sparse matrix of the chain, on the host (diagnostics
        only, spai.py:91-95)."""
        mats = [F.to_scipy() for F in self.factors()]
        out = mats[-1]
        for M in reversed(mats[:-1]):
            out = M @ out
        out = sp.csr_matrix(out)
        out.eliminate_zeros()
        return out


def _block_to_dev(V):
    if torch.is_tensor(V):
        Vd = V.to(device=_dev(), dtype=torch.float64)
    else:
        arr = np.asarray(V)
        if np.iscomplexobj(arr):
            if np.any(arr.imag != 0):
                raise NotImplementedError("complex blocks are not supported by the B200 path yet")
            arr = arr.real
        Vd = torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64), device=_dev())
    if Vd.dim() == 1:
        Vd = Vd[:, None]
    if Vd.dim() != 2:
        raise ValueError("expected vector or 2-D block")
    return Vd.contiguous()


# ---------------------------------------------------------------------------
# least-squares planning (size tiers) -- host side, once per pattern
# ---------------------------------------------------------------------------

_TIERS = ((32, 0, 12 * 1024), (128, 0, 64 * 1024), (256, 0, 200 * 1024), (256, 1, None))


def _align16(b):
    return (b + 15) & ~15


def _team_bytes(lcap, mcap, ncap):
    d = mcap * (ncap + 1) + 4 * (ncap + 1) + 16
    i = lcap + 3 * (ncap + 1) + 1 + 16
    return _align16(8 * d) + _align16(4 * i)


def _pow2(v):
    v = np.maximum(np.asarray(v, dtype=np.int64), 1)

    def up(x):
        return (1 << np.ceil(np.log2(x)).astype(np.int64)).astype(np.int64)
    if v.ndim and v.size > 4096:
        vmax = int(v.max())
        if vmax <= (1 << 22):   # small integers: one table, one gather
            return up(np.maximum(np.arange(vmax + 1, dtype=np.int64), 1))[v]
    return up(v)


class _Tier:
    """One launch of pmp_ls_columns.  mode 3 = the semi-normal-equations
    kernel for columns whose dense block exceeds shared memory."""

    def __init__(self, team, glob, lcap, mcap, ncap, cols, mode=0, cols_dev=None):
        self.team, self.glob, self.mode = team, glob, mode
        self.lcap, self.mcap, self.ncap = int(lcap), int(mcap), int(ncap)
        self.cols_host = cols
        self.cols = i32(cols) if cols_dev is None else cols_dev
        self.ncols = int(cols.size)
        self.bytes = (_sne_bytes(self.lcap, self.mcap, self.ncap) if mode == 3
                      else _team_bytes(self.lcap, self.mcap, self.ncap))


def _sne_bytes(lcap, mcap, ncap):
    d = mcap + ncap * ncap + 5 * (ncap + 1) + 16
    i = lcap + 3 * (ncap + 1) + 1 + 16
    return _align16(8 * d) + _align16(4 * i)


def _split_tiers(cols, lcap, m, nI):
    """_split_tiers_direct, decided on the DISTINCT (list capacity, coarsened
    |I|, coarsened |J|) triples instead of on every column: the tier logic
    depends on a column only through that triple (and on the largest true
    |I| / |J| of a group), so for large column sets the triples are grouped
    on the device (torch.unique + scatter max: milliseconds at n = 2^21,
    where the per-column numpy sorts cost 0.25 s per plan), the tiers are
    formed on the few distinct triples, and every tier's column list is
    gathered on the device.  Same tiers, same column order."""
    n = cols.size
    if n < 65536:
        return _split_tiers_direct(cols, lcap, m, nI)
    cm, cn = _coarse(m), _coarse(nI)
    if max(int(lcap.max()), int(cm.max()), int(cn.max())) >= (1 << 21):
        return _split_tiers_direct(cols, lcap, m, nI)
    dev = _dev()
    key = torch.as_tensor((lcap << 42) | (cn << 21) | cm, device=dev)
    uk, inv = torch.unique(key, return_inverse=True)
    U = int(uk.numel())
    gm = torch.zeros(U, dtype=torch.int64, device=dev).scatter_reduce_(
        0, inv, torch.as_tensor(m, device=dev), "amax", include_self=False)
    gn = torch.zeros(U, dtype=torch.int64, device=dev).scatter_reduce_(
        0, inv, torch.as_tensor(nI, device=dev), "amax", include_self=False)
    rep = _split_tiers_direct(np.arange(U, dtype=np.int64), uk.cpu().numpy() >> 42,
                              gm.cpu().numpy(), gn.cpu().numpy())
    tier_of_key = np.zeros(U, dtype=np.int64)
    for ti, t in enumerate(rep):
        tier_of_key[t.cols_host] = ti
    tcol = torch.as_tensor(tier_of_key, device=dev)[inv]
    dcols = torch.as_tensor(cols, device=dev)
    out = []
    for ti, t in enumerate(rep):
        c = dcols[torch.nonzero(tcol == ti).flatten()]
        c = torch.sort(c).values
        out.append(_Tier(t.team, t.glob, t.lcap, t.mcap, t.ncap, c.cpu().numpy(), mode=t.mode,
                         cols_dev=c.to(torch.int32)))
    return out


def _split_tiers_direct(cols, lcap, m, nI):
    """Group columns into launch tiers by the team memory they need: dense
    pivoted-QR teams (warp / 128 / 256 threads, shared memory) while the
    dense block fits, the semi-normal-equations kernel (mode 3) beyond."""
    if cols.size == 0:
        return []
    b = _team_bytes(lcap, _coarse(m), _coarse(nI))   # classify on the padded dims
    cls = np.full(cols.size, len(_TIERS) - 1)
    for t in range(len(_TIERS) - 2, -1, -1):
        cls[b <= _TIERS[t][2]] = t
    tiers = []
    for t, (team, glob, limit) in enumerate(_TIERS):
        sel = np.flatnonzero(cls == t)
        if sel.size == 0:
            continue
        if limit is not None:
            tiers += _bucket_merge(sel, cols, lcap, m, nI, _team_bytes, limit, team, 0, 0)
            continue
        # beyond shared memory: semi-normal equations, in shared memory when
        # its much smaller footprint fits, else in global memory
        sb_ = _sne_bytes(lcap[sel], _coarse(m[sel]), _coarse(nI[sel]))
        small = sel[sb_ <= 200 * 1024]
        large = sel[sb_ > 200 * 1024]
        tiers += _bucket_merge(small, cols, lcap, m, nI, _sne_bytes, 200 * 1024, 256, 0, 3)
        if large.size:
            tiers.append(_tier_from(256, 1, cols, lcap, m, nI, large, mode=3))
    return tiers


def _bucket_merge(sel, cols, lcap, m, nI, bytes_fn, limit, team, glob, mode):
    """Bucket columns by coarsened dimensions (<= 25 % padding), then merge
    buckets in size order while the merged team still fits `limit`:
    O(n log n) and a handful of launches even for power-law sizes."""
    if sel.size == 0:
        return []
    # one int64 key per column (21 bits per coarsened dimension): a 1-D
    # unique is a plain sort, np.unique(axis=0) a lexicographic one that
    # took seconds at n = 2^21
    k0, k1, k2 = lcap[sel], _coarse(nI[sel]), _coarse(m[sel])
    if max(int(k0.max()), int(k1.max()), int(k2.max())) >= (1 << 21):
        key = np.stack([k0, k1, k2], axis=1)
        ukeys, inv = np.unique(key, axis=0, return_inverse=True)
        inv = inv.ravel()
    else:
        key1 = (k0 << 42) | (k1 << 21) | k2
        uk, inv = np.unique(key1, return_inverse=True)
        inv = inv.ravel()
        ukeys = np.stack([uk >> 42, (uk >> 21) & ((1 << 21) - 1), uk & ((1 << 21) - 1)], axis=1)
    gbytes = bytes_fn(ukeys[:, 0], ukeys[:, 2], ukeys[:, 1])
    order = np.argsort(gbytes, kind="stable")
    by_group = np.argsort(inv, kind="stable")
    bounds = np.searchsorted(inv[by_group], np.arange(len(ukeys) + 1))
    out, cur, dims = [], [], None
    for g in order:
        kd = ukeys[g]
        nd = kd if dims is None else np.maximum(dims, kd)
        if dims is not None and bytes_fn(nd[0], nd[2], nd[1]) > limit:
            out.append(_tier_from(team, glob, cols, lcap, m, nI, np.concatenate(cur), mode))
            cur, nd = [], kd
        cur.append(sel[by_group[bounds[g]:bounds[g + 1]]])
        dims = nd
    if cur:
        out.append(_tier_from(team, glob, cols, lcap, m, nI, np.concatenate(cur), mode))
    return out


def _coarse(v):
    """Round up to {1, 1.25, 1.5, 1.75} x 2^k (at least 8)."""
    v = np.maximum(np.asarray(v, dtype=np.int64), 8)

    def rnd(x):
        p = 1 << (np.floor(np.log2(x)).astype(np.int64) - 2)
        return ((x + p - 1) // p) * p
    vmax = int(v.max()) if v.size else 8
    if v.size > 4096 and vmax <= (1 << 22):
        # sizes are small integers: one table, one gather (log2 over millions
        # of columns was the largest item of the cold planning profile)
        lut = rnd(np.maximum(np.arange(vmax + 1, dtype=np.int64), 8))
        return lut[v]
    return rnd(v)


def _tier_from(team, glob, cols, lcap, m, nI, idx, mode=0):
    s = np.asarray(idx, dtype=np.int64)
    s = s[np.argsort(cols[s], kind="stable")]
    return _Tier(team, glob, lcap[s].max(), m[s].max(), nI[s].max(), cols[s], mode=mode)


def _plan(pattern, sys_colptr, sys_rowidx, t_colptr, t_rowidx, t_key, sys_key, cols_host=None):
    """Size tiers for solving the listed columns of ``pattern`` against the
    system (and target) structures; cached on the pattern when all columns
    are solved."""
    key = ("plan", sys_key, t_key) if cols_host is None else None
    if key is not None and key in pattern.cache:
        return pattern.cache[key]
    n = pattern.n
    st = _abi.stream()
    cols = np.arange(n, dtype=np.int64) if cols_host is None else np.asarray(cols_host, np.int64)
    ncols = cols.size
    if ncols == 0:
        return []
    dcols = None if cols_host is None else i32(cols)
    lsize = torch.empty(ncols, dtype=torch.int32, device=_dev())
    _abi.call("pmp_ls_bound", ncols, _abi.ptr(dcols), _abi.ptr(pattern.iptr),
              _abi.ptr(pattern.iidx), _abi.ptr(sys_colptr), _abi.ptr(t_colptr),
              _abi.ptr(lsize), st)
    L = lsize.cpu().numpy().astype(np.int64)
    iptr = pattern.iptr.cpu().numpy().astype(np.int64)
    nI = (iptr[cols + 1] - iptr[cols]).astype(np.int64)
    lcap = _pow2(L)
    # plan pass: |J_j| (mode 1) grouped by list capacity
    msize = torch.zeros(n, dtype=torch.int32, device=_dev())
    # (distinct capacities from a histogram of the small integer bounds: no
    # sort of the per-column array)
    Lc = np.maximum(L, 1)
    caps = np.unique(_pow2(np.flatnonzero(np.bincount(Lc)))) if ncols > 4096 else np.unique(lcap)
    for cap in caps:
        s = np.flatnonzero(lcap == cap)
        nc = int(nI[s].max())
        tb = _team_bytes(int(cap), 0, nc)
        team, glob = (32, 0) if tb <= 12 * 1024 else ((256, 0) if tb <= 200 * 1024 else (256, 1))
        dsel = i32(cols[s])
        ws = _ws_for(glob, tb, s.size)
        _abi.call("pmp_ls_columns", 1, team, glob, int(cap), 0, nc, int(s.size), _abi.ptr(dsel), n,
                  _abi.ptr(pattern.iptr), _abi.ptr(pattern.iidx), _abi.ptr(sys_colptr),
                  _abi.ptr(sys_rowidx), None, _abi.ptr(t_colptr), _abi.ptr(t_rowidx),
                  None, None, None, None, _abi.ptr(msize), None, None, _abi.ptr(ws),
                  ws.numel() if ws is not None else 0, st)
    m = msize.cpu().numpy().astype(np.int64)[cols]
    tiers = _split_tiers(cols, lcap, m, nI)
    # per-column sizes of a symbolic plan record (pmp_ls_columns_planned)
    # (position of every tier column in `cols`, vectorised: a Python dict over
    # the 2 M augmented columns of a level-1 build at c4 cost 0.6 s per system)
    order = scols = None
    if cols_host is not None:
        order = np.argsort(cols, kind="stable")
        scols = cols[order]
    for t in tiers:
        idx = (t.cols_host if order is None
               else order[np.searchsorted(scols, np.asarray(t.cols_host, dtype=np.int64))])
        t.plan_sizes = 4 + nI[idx] + 2 * L[idx]
    if key is not None:
        pattern.cache[key] = tiers
    return tiers


def _ws_for(glob, team_bytes, ncols):
    if not glob:
        return None
    grid = min(ncols, 2 * torch.cuda.get_device_properties(_dev()).multi_processor_count)
    # at most ~4 GB of team memory (the launcher shrinks the grid to fit)
    grid = max(1, min(grid, (4 << 30) // max(team_bytes, 1)))
    return scratch().get("ls_global", team_bytes * grid)


# ---------------------------------------------------------------------------
# column solves (spai.py:273-338)
# ---------------------------------------------------------------------------


def _csr_plan(pattern):
    """Transpose plan of a pattern (CSC supports -> CSR factor), cached."""
    plan = pattern.cache.get("csr")
    if plan is None:
        n, nnz = pattern.n, pattern.nnz
        rowptr = torch.empty(n + 1, dtype=torch.int32, device=_dev())
        colidx = torch.empty(max(nnz, 1), dtype=torch.int32, device=_dev())
        perm = torch.empty(max(nnz, 1), dtype=torch.int32, device=_dev())
        ws = scratch().get("transpose", _abi.lib().pmp_transpose_workspace(n, nnz))
        _abi.call("pmp_transpose", n, nnz, _abi.ptr(pattern.iptr), _abi.ptr(pattern.iidx), None,
                  0, _abi.ptr(rowptr), _abi.ptr(colidx), None, _abi.ptr(perm), _abi.ptr(ws),
                  ws.numel(), _abi.stream())
        st = Structure(n, rowptr, colidx[:nnz] if nnz else colidx[:0])
        plan = (st, perm[:nnz] if nnz else perm[:0])
        pattern.cache["csr"] = plan
    return plan


def _factor_from_columns(pattern, coef):
    st, perm = _csr_plan(pattern)
    vals = torch.empty(max(pattern.nnz, 1), dtype=torch.float64, device=_dev())[:pattern.nnz]
    if pattern.nnz:
        _abi.call("pmp_permute", pattern.nnz, _abi.ptr(perm), _abi.ptr(coef), _abi.ptr(vals),
                  _abi.stream())
    return DeviceCSR(st, vals, symmetric=False)


def _run_tiers(tiers, pattern, A_csc, T_csc, coef, resid, flags, mode=0, jptr=None, jidx=None):
    st = _abi.stream()
    acolptr, arowidx, avals = A_csc
    tcolptr, trowidx, tvals = T_csc if T_csc is not None else (None, None, None)
    sne = []
    for t in tiers:
        tmode = t.mode if mode == 0 else mode
        if tmode == 3:
            sne.append(t)
        tb = t.bytes if tmode == t.mode else _team_bytes(t.lcap, 0, t.ncap)
        glob = t.glob if tmode == t.mode else 0
        team = t.team
        ws = _ws_for(glob, tb, t.ncols)
        if tmode == 0 and _plan_ok(t):
            # record the symbolic work on the first solve of this tier, replay
            # it on every later one (same structures, new values)
            pmode = 5 if t.plan_ready else 4
            _abi.call("pmp_ls_columns_planned", pmode, team, glob, t.lcap, t.mcap, t.ncap,
                      t.ncols, _abi.ptr(t.cols), pattern.n, _abi.ptr(pattern.iptr),
                      _abi.ptr(pattern.iidx), _abi.ptr(acolptr), _abi.ptr(arowidx),
                      _abi.ptr(avals), _abi.ptr(tcolptr), _abi.ptr(trowidx), _abi.ptr(tvals),
                      _abi.ptr(coef), _abi.ptr(resid), _abi.ptr(flags), _abi.ptr(t.plan),
                      _abi.ptr(t.plan_ptr), _abi.ptr(ws), ws.numel() if ws is not None else 0,
                      st)
            t.plan_ready = True
            continue
        _abi.call("pmp_ls_columns", tmode, team, glob, t.lcap, t.mcap, t.ncap, t.ncols,
                  _abi.ptr(t.cols), pattern.n, _abi.ptr(pattern.iptr), _abi.ptr(pattern.iidx),
                  _abi.ptr(acolptr), _abi.ptr(arowidx), _abi.ptr(avals), _abi.ptr(tcolptr),
                  _abi.ptr(trowidx), _abi.ptr(tvals), _abi.ptr(coef), _abi.ptr(resid),
                  _abi.ptr(flags), None, _abi.ptr(jptr), _abi.ptr(jidx), _abi.ptr(ws),
                  ws.numel() if ws is not None else 0, st)
    if sne:
        # columns the semi-normal equations could not certify (near rank
        # deficient G, flags == 2): dense column-pivoted QR in global memory
        fl = flags.cpu().numpy()
        for t in sne:
            bad = t.cols_host[fl[t.cols_host] == 2]
            if bad.size == 0:
                continue
            d = _Tier(256, 1, t.lcap, t.mcap, t.ncap, bad)
            ws = _ws_for(1, d.bytes, d.ncols)
            _abi.call("pmp_ls_columns", 0, 256, 1, d.lcap, d.mcap, d.ncap, d.ncols,
                      _abi.ptr(d.cols), pattern.n, _abi.ptr(pattern.iptr),
                      _abi.ptr(pattern.iidx), _abi.ptr(acolptr), _abi.ptr(arowidx),
                      _abi.ptr(avals), _abi.ptr(tcolptr), _abi.ptr(trowidx), _abi.ptr(tvals),
                      _abi.ptr(coef), _abi.ptr(resid), _abi.ptr(flags), None, None, None,
                      _abi.ptr(ws), ws.numel(), st)


# symbolic plan records: per-column int32 records up to this many ints per tier
_PLAN_MAX_INTS = 1 << 30
USE_LS_PLANS = __import__("os").environ.get("PMP_LS_PLANS", "1") != "0"


def _plan_ok(t):
    """Allocate (once) the plan record of a dense-QR tier; False when the
    tier cannot use one (sizes beyond the record's 16-bit fields, too big)."""
    if not USE_LS_PLANS or t.mode != 0 or getattr(t, "plan_sizes", None) is None:
        return False
    if getattr(t, "plan", None) is not None:
        return True
    if t.mcap >= 65536 or t.ncap >= 32768:
        return False
    sizes = np.asarray(t.plan_sizes, dtype=np.int64)
    total = int(sizes.sum())
    if total <= 0 or total >= _PLAN_MAX_INTS:
        return False
    ptr = np.zeros(sizes.size, dtype=np.int64)
    ptr[1:] = np.cumsum(sizes)[:-1]
    t.plan_ptr = i32(ptr)
    t.plan = torch.empty(total, dtype=torch.int32, device=_dev())
    t.plan_ready = False
    return True


def _get_tiers(pattern, system, target, cols_host=None):
    acolptr, arowidx = system.csc_structure()
    tcolptr = trowidx = tkey = None
    if target is not None:
        tcolptr, trowidx = target.csc_structure()
        tkey = target.structure.key
    return _plan(pattern, acolptr, arowidx, tcolptr, trowidx, tkey, system.structure.key,
                 cols_host)


def _augment(system, base, cols_dev, ncols, max_fill):
    """Level-1 supports for the listed columns (spai.py:210-222): returns an
    n-column pattern whose column j is non-empty iff j was augmented."""
    n = base.n
    st = _abi.stream()
    acolptr, arowidx, avals = system.csc()
    lsize = torch.empty(ncols, dtype=torch.int32, device=_dev())
    _abi.call("pmp_ls_bound", ncols, _abi.ptr(cols_dev), _abi.ptr(base.iptr), _abi.ptr(base.iidx),
              _abi.ptr(acolptr), None, _abi.ptr(lsize), st)
    L = int(lsize.max().item())
    lcap = int(_pow2(L))
    tb = _abi.lib().pmp_augment_team_bytes(lcap)
    glob = 1 if tb > 200 * 1024 else 0
    ws = _ws_for(glob, tb, ncols)
    size = torch.zeros(n, dtype=torch.int32, device=_dev())
    args_tail = (_abi.ptr(ws), ws.numel() if ws is not None else 0, st)
    _abi.call("pmp_augment", 0, lcap, glob, ncols, _abi.ptr(cols_dev), int(max_fill),
              _abi.ptr(base.iptr), _abi.ptr(base.iidx), _abi.ptr(acolptr), _abi.ptr(arowidx),
              _abi.ptr(avals), _abi.ptr(size), None, None, *args_tail)
    aptr = torch.empty(n + 1, dtype=torch.int32, device=_dev())
    sws = scratch().get("scan", _abi.lib().pmp_scan_workspace(n))
    _abi.call("pmp_scan", n, _abi.ptr(size), _abi.ptr(aptr), _abi.ptr(sws), sws.numel(), st)
    nnz = int(aptr[n].item())
    aidx = torch.empty(max(nnz, 1), dtype=torch.int32, device=_dev())
    _abi.call("pmp_augment", 1, lcap, glob, ncols, _abi.ptr(cols_dev), int(max_fill),
              _abi.ptr(base.iptr), _abi.ptr(base.iidx), _abi.ptr(acolptr), _abi.ptr(arowidx),
              _abi.ptr(avals), None, _abi.ptr(aptr), _abi.ptr(aidx), *args_tail)
    return DevicePattern(n, aptr, aidx, nnz)


def solve_columns(system, target, pattern, cfg, events=True):
    """Device restatement of _run_column_solves + _build_columns
    (spai.py:273-338): returns (factor DeviceCSR, BuildStats, final pattern,
    coefficients in pattern order)."""
    n = system.n
    st = _abi.stream()
    ev0 = ev1 = None
    if events:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
    A_csc = system.csc()
    T_csc = target.csc() if target is not None else None
    tiers = _get_tiers(pattern, system, target)
    coef = torch.empty(max(pattern.nnz, 1), dtype=torch.float64, device=_dev())
    resid = torch.empty(n, dtype=torch.float64, device=_dev())
    flags = torch.zeros(n, dtype=torch.int32, device=_dev())
    _run_tiers(tiers, pattern, A_csc, T_csc, coef, resid, flags)
    final_pat, final_coef, n_aug = pattern, coef, 0
    if cfg.pattern_level >= 1 and n > 0 and system.cplx:
        final_pat, final_coef, n_aug = _augment_complex(system, target, pattern, coef, resid,
                                                        flags, cfg, A_csc, T_csc)
    elif cfg.pattern_level >= 1 and n > 0:
        sel = torch.empty(n, dtype=torch.int32, device=_dev())
        cnt = torch.zeros(1, dtype=torch.int32, device=_dev())
        ws = scratch().get("select", _abi.lib().pmp_select_workspace(n))
        _abi.call("pmp_select_gt", n, None, _abi.ptr(resid), float(cfg.ep), _abi.ptr(sel),
                  _abi.ptr(cnt), _abi.ptr(ws), ws.numel(), st)
        n_aug = int(cnt.item())
        if n_aug:
            cols_dev = sel[:n_aug]
            apat = _augment(system, pattern, cols_dev, n_aug, cfg.max_fill_per_column)
            atiers = _get_tiers(apat, system, target, cols_dev.cpu().numpy())
            acoef = torch.empty(max(apat.nnz, 1), dtype=torch.float64, device=_dev())
            _run_tiers(atiers, apat, A_csc, T_csc, acoef, resid, flags)
            final_pat, final_coef = _merge(pattern, coef, apat, acoef)
    if final_pat is pattern:
        P = _factor_from_columns(pattern, coef)
    else:
        P = _factor_from_columns(final_pat, final_coef)
    if events:
        ev1.record()
    if system.cplx:
        P.cplx = True
    stats = BuildStats(resid, flags, n_aug, (ev0, ev1) if events else None,
                       stride=2 if system.cplx else 1)
    return P, stats, final_pat, final_coef


def _augment_complex(system, target, pattern, coef, resid, flags, cfg, A_csc, T_csc):
    """Level-1 pass of a complex build on the real form (spai.py:285-289):
    complex column j (real columns 2j, 2j+1) is augmented when its residual
    -- that of real column 2j -- exceeds ep; the extra rows are ranked by the
    complex moduli |A| |A|[:, j] (spai.py:210-222) on the complex structure,
    realified, and both real columns re-solved."""
    from . import cplx as _cx
    n2 = system.n
    n = n2 // 2
    st = _abi.stream()
    even = torch.arange(0, n2, 2, dtype=torch.int32, device=_dev())
    sel = torch.empty(n, dtype=torch.int32, device=_dev())
    cnt = torch.zeros(1, dtype=torch.int32, device=_dev())
    ws = scratch().get("select", _abi.lib().pmp_select_workspace(n))
    _abi.call("pmp_select_gt", n, _abi.ptr(even), _abi.ptr(resid), float(cfg.ep), _abi.ptr(sel),
              _abi.ptr(cnt), _abi.ptr(ws), ws.numel(), st)
    n_aug = int(cnt.item())
    if not n_aug:
        return pattern, coef, 0
    jsel = (sel[:n_aug] // 2).to(torch.int32)
    absA = _cx.modulus_csr(system)
    base_c = level0_pattern(absA)
    apat_c = _augment(absA, base_c, jsel, n_aug, cfg.max_fill_per_column)
    apat = _cx.realify_pattern(apat_c)
    jh = jsel.cpu().numpy().astype(np.int64)
    cols = np.sort(np.concatenate([2 * jh, 2 * jh + 1]))
    atiers = _get_tiers(apat, system, target, cols)
    acoef = torch.empty(max(apat.nnz, 1), dtype=torch.float64, device=_dev())
    _run_tiers(atiers, apat, A_csc, T_csc, acoef, resid, flags)
    fp, fc = _merge(pattern, coef, apat, acoef)
    return fp, fc, n_aug


def _seg_tier(t):
    """Tier the library solves in the segmented register tier (several
    systems per launch): small dense blocks, warp teams, shared memory."""
    return t.mode == 0 and t.team == 32 and not t.glob and t.mcap <= 32 and t.ncap <= 15


def solve_columns_many(systems, target, pattern, cfg):
    """solve_columns for several systems that share one structure (the SPAI
    updates of a parameter sweep), level 0: every least-squares tier is ONE
    pmp_ls_columns_multi call -- the small-column tier solves every system
    in one launch -- so a window of updates costs a handful of launches and
    host calls instead of a few per system.  Bitwise the per-system result.
    Returns [(factor DeviceCSR, BuildStats)] in order."""
    systems = list(systems)
    if (cfg.pattern_level >= 1 or len(systems) < 2 or not USE_LS_PLANS
            or any(A.structure is not systems[0].structure for A in systems)):
        out = []
        for A in systems:
            P, stats, _, _ = solve_columns(A, target, pattern, cfg)
            out.append((P, stats))
        return out
    import ctypes
    n = systems[0].n
    k = len(systems)
    st = _abi.stream()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    A0 = systems[0]
    acolptr, arowidx, _ = A0.csc()
    tcolptr = trowidx = tvals = None
    if target is not None:
        tcolptr, trowidx, tvals = target.csc()
    tiers = _get_tiers(pattern, A0, target)
    # one [k, nnz] block: the factors leave it through one batched permute
    nz = -(-max(pattern.nnz, 1) // 32) * 32   # rows 256-byte aligned
    coef_block = torch.empty((k, nz), dtype=torch.float64, device=_dev())
    coefs = [coef_block[q] for q in range(k)]
    nr = -(-max(n, 1) // 64) * 64
    resid_block = torch.empty((k, nr), dtype=torch.float64, device=_dev())
    flag_block = torch.zeros((k, nr), dtype=torch.int32, device=_dev())  # one fill, not k
    resids = [resid_block[q, :n] for q in range(k)]
    flags = [flag_block[q, :n] for q in range(k)]
    csc_vals = [A.csc()[2] for A in systems]
    VP = ctypes.c_void_p * k
    h_avals = VP(*[v.data_ptr() for v in csc_vals])
    h_coef = VP(*[c.data_ptr() for c in coefs])
    h_resid = VP(*[r.data_ptr() for r in resids])
    h_flags = VP(*[f.data_ptr() for f in flags])
    for t in tiers:
        if t.mode != 0 or not _plan_ok(t):
            for q, A in enumerate(systems):
                _run_tiers([t], pattern, A.csc(), target.csc() if target is not None else None,
                           coefs[q], resids[q], flags[q])
            continue
        pmode = 5 if t.plan_ready else 4
        ws = _ws_for(t.glob, t.bytes, t.ncols)
        _abi.call("pmp_ls_columns_multi", pmode, t.team, t.glob, t.lcap, t.mcap, t.ncap,
                  t.ncols, _abi.ptr(t.cols), n, _abi.ptr(pattern.iptr), _abi.ptr(pattern.iidx),
                  _abi.ptr(acolptr), _abi.ptr(arowidx), k, h_avals, _abi.ptr(tcolptr),
                  _abi.ptr(trowidx), _abi.ptr(tvals), h_coef, h_resid, h_flags,
                  _abi.ptr(t.plan), _abi.ptr(t.plan_ptr), _abi.ptr(ws),
                  ws.numel() if ws is not None else 0, st)
        if _seg_tier(t) and _abi.lib_seg_enabled():
            first = 1 if pmode == 4 else 0
            extra = (2 if pmode == 4 else 0) + -(-(k - first) // 64)
        else:
            extra = k + (1 if pmode == 4 else 0)
        _abi.note_launches(extra - 1)
        t.plan_ready = True
    out = []
    csr, perm = _csr_plan(pattern)
    val_block = torch.empty((k, nz), dtype=torch.float64, device=_dev())
    if pattern.nnz:
        _abi.call("pmp_permute_batch", pattern.nnz, _abi.ptr(perm), k, _abi.ptr(coef_block), nz,
                  _abi.ptr(val_block), nz, st)
    for q in range(k):
        P = DeviceCSR(csr, val_block[q, :pattern.nnz], symmetric=False)
        P.cplx = systems[q].cplx
        out.append((P, (resids[q], flags[q])))
    ev1.record()
    stride = 2 if A0.cplx else 1
    return [(P, BuildStats(r, f, 0, (ev0, ev1), share=k, stride=stride)) for P, (r, f) in out]


def _merge(base, bcoef, apat, acoef):
    n = base.n
    st = _abi.stream()
    size = torch.empty(n, dtype=torch.int32, device=_dev())
    _abi.call("pmp_merge_sizes", n, _abi.ptr(base.iptr), _abi.ptr(apat.iptr), _abi.ptr(size), st)
    optr = torch.empty(n + 1, dtype=torch.int32, device=_dev())
    sws = scratch().get("scan", _abi.lib().pmp_scan_workspace(n))
    _abi.call("pmp_scan", n, _abi.ptr(size), _abi.ptr(optr), _abi.ptr(sws), sws.numel(), st)
    nnz = int(optr[n].item())
    oidx = torch.empty(max(nnz, 1), dtype=torch.int32, device=_dev())
    ocoef = torch.empty(max(nnz, 1), dtype=torch.float64, device=_dev())
    _abi.call("pmp_merge_columns", n, _abi.ptr(base.iptr), _abi.ptr(base.iidx), _abi.ptr(bcoef),
              _abi.ptr(apat.iptr), _abi.ptr(apat.iidx), _abi.ptr(acoef), _abi.ptr(optr),
              _abi.ptr(oidx), _abi.ptr(ocoef), st)
    return DevicePattern(n, optr, oidx, nnz), ocoef


# ---------------------------------------------------------------------------
# public API (spai.py:182-373)
# ---------------------------------------------------------------------------


class SparsityPattern:
    """Host mirror of sparsecore.SparsityPattern (sparsecore.py:76-99)."""

    def __init__(self, nrows, columns=()):
        self.nrows = nrows
        cleaned = []
        for idx in columns:
            arr = np.unique(np.asarray(idx, dtype=np.int64))
            if arr.size and (arr[0] < 0 or arr[-1] >= nrows):
                raise ValueError("pattern row index out of range [0, %d)" % nrows)
            cleaned.append(arr)
        self.columns = cleaned

    @property
    def ncols(self):
        return len(self.columns)

    def max_fill(self):
        return max((len(c) for c in self.columns), default=0)


def _to_device_pattern(pattern, n):
    if isinstance(pattern, DevicePattern):
        return pattern
    cols = pattern.columns if isinstance(pattern, SparsityPattern) else pattern
    if len(cols) != n:
        raise ValueError("pattern has %d columns, matrix has %d" % (len(cols), n))
    return DevicePattern.from_columns(n, [np.unique(np.asarray(c, dtype=np.int64)) for c in cols])


def spai_pattern(A, level=0, max_fill_per_column=80):
    """A-priori pattern (spai.py:182-207), computed on the device (complex
    matrices: on the complex structure, ranked by |A|)."""
    A = _as_dev_csr(A)
    if A.cplx:
        from .cplx import modulus_csr
        A = modulus_csr(A)
    base = level0_pattern(A)
    if level == 0:
        return SparsityPattern(A.n, base.columns())
    n = A.n
    cols = torch.arange(n, dtype=torch.int32, device=_dev())
    apat = _augment(A, base, cols, n, max_fill_per_column)
    return SparsityPattern(n, apat.columns())


def spai_column(A, i, pattern_i):
    """Least-squares column of the approximate inverse (spai.py:256-270)."""
    A = _as_dev_csr(A)
    support = np.unique(np.asarray(pattern_i, dtype=np.int64))
    if support.size == 0:
        raise ValueError("column pattern must be nonempty")
    if A.cplx:
        # real form: column 2i over rows {2k, 2k+1 : k in support}
        n = A.n
        cols = [np.zeros(0, dtype=np.int64)] * n
        cols[2 * int(i)] = np.sort(np.concatenate([2 * support, 2 * support + 1]))
        pat = DevicePattern.from_columns(n, cols)
        tiers = _get_tiers(pat, A, None, np.array([2 * int(i)]))
        coef = torch.empty(max(pat.nnz, 1), dtype=torch.float64, device=_dev())
        resid = torch.empty(n, dtype=torch.float64, device=_dev())
        flags = torch.zeros(n, dtype=torch.int32, device=_dev())
        _run_tiers(tiers, pat, A.csc(), None, coef, resid, flags)
        z = coef[:2 * support.size].cpu().numpy()
        return (support, z[0::2] + 1j * z[1::2], float(resid[2 * int(i)].item()),
                bool(flags[2 * int(i)].item()))
    n = A.n
    cols = [np.zeros(0, dtype=np.int64)] * n
    cols[int(i)] = support
    pat = DevicePattern.from_columns(n, cols)
    tiers = _get_tiers(pat, A, None, np.array([int(i)]))
    coef = torch.empty(max(pat.nnz, 1), dtype=torch.float64, device=_dev())
    resid = torch.empty(n, dtype=torch.float64, device=_dev())
    flags = torch.zeros(n, dtype=torch.int32, device=_dev())
    _run_tiers(tiers, pat, A.csc(), None, coef, resid, flags)
    return (support, coef[:support.size].cpu().numpy(), float(resid[int(i)].item()),
            bool(flags[int(i)].item()))


def spai_build(A, cfg=None, pattern=None, threads=1):
    """Explicit sparse approximate inverse of A (spai.py:341-364).
    ``threads`` is accepted for API compatibility (the device build is
    column-parallel regardless)."""
    A = _as_dev_csr(A)
    cfg = cfg or SpaiConfig()
    if pattern is None:
        pat = level0_pattern(A)   # (real form: the complex supports realified)
        eff = cfg
    else:
        if A.cplx:
            from .cplx import realify_pattern
            pat = realify_pattern(_to_device_pattern(pattern, A.complex_n))
        else:
            pat = _to_device_pattern(pattern, A.n)
        eff = SpaiConfig(ep=cfg.ep, pattern_level=0, max_fill_per_column=cfg.max_fill_per_column)
    P, stats, _, _ = solve_columns(A, None, pat, eff)
    return Preconditioner(matrix=P), stats


def spai_build_sharded(A, cfg=None, comm=None):
    """Base SPAI built across the ranks of ``comm``: every
    column is an independent least-squares problem (spai.py:273-292,
    SPEC "columns are independent"), so rank r solves the contiguous columns
    [b_r, b_{r+1}) of the level-0 pattern -- deterministic on every rank --
    and one grouped all-gather (pmp_nccl_allgatherv) replicates the
    coefficients (pattern order), residuals and flags; every rank then
    permutes its full copy to CSR.  Bitwise the single-rank build.

    Level >= 1 (augmented supports are only known after the first pass and
    differ per column): rank 0 builds, then its CSR structure -- nnz first --
    and values are broadcast, so every rank holds rank 0's exact factor.
    Returns (Preconditioner, BuildStats) on every rank."""
    from .comm import column_bounds, get_comm
    A = _as_dev_csr(A)
    cfg = cfg or SpaiConfig()
    comm = comm or get_comm()
    if comm.world <= 1:
        return spai_build(A, cfg)
    n = A.n
    dev = _dev()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    if cfg.pattern_level >= 1:
        meta = torch.zeros(2, dtype=torch.float64, device=dev)
        if comm.rank == 0:
            P0, st0 = spai_build(A, cfg)
            M = P0.matrix
            meta[0] = float(M.nnz)
            meta[1] = float(st0.augmented_columns)
        comm.bcast(meta, 0)
        nnz, n_aug = int(meta[0].item()), int(meta[1].item())
        if comm.rank == 0:
            rowptr, colidx, vals = M.structure.rowptr, M.structure.colidx, M.vals
            resid, flags = st0._resid, st0._flags
        else:
            rowptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
            colidx = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)[:nnz]
            vals = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)[:nnz]
            resid = torch.empty(n, dtype=torch.float64, device=dev)
            flags = torch.empty(n, dtype=torch.int32, device=dev)
        for t in (rowptr, colidx, vals, resid, flags):
            comm.bcast(t, 0)
        ev1.record()
        if comm.rank == 0:
            P = P0
        else:
            P = Preconditioner(matrix=DeviceCSR(Structure(n, rowptr, colidx), vals,
                                                symmetric=False))
        return P, BuildStats(resid, flags, n_aug, (ev0, ev1))
    pat = level0_pattern(A)
    b = column_bounds(n, comm.world)
    c0, c1 = b[comm.rank], b[comm.rank + 1]
    coef = torch.zeros(max(pat.nnz, 1), dtype=torch.float64, device=dev)
    resid = torch.zeros(n, dtype=torch.float64, device=dev)
    flags = torch.zeros(n, dtype=torch.int32, device=dev)
    if c1 > c0:
        tiers = _get_tiers(pat, A, None, np.arange(c0, c1, dtype=np.int64))
        _run_tiers(tiers, pat, A.csc(), None, coef, resid, flags)
    iptr = pat.iptr.cpu().numpy().astype(np.int64)
    comm.allgatherv(coef, [int(iptr[x]) for x in b])
    comm.allgatherv(resid, b)
    comm.allgatherv(flags, b)
    P = _factor_from_columns(pat, coef[:pat.nnz])
    ev1.record()
    return Preconditioner(matrix=P), BuildStats(resid, flags, 0, (ev0, ev1))


def quality(A, P):
    """||I - A P||_F (spai.py:367-373) on the device: the identity goes
    through the chain and A in 32-column slabs (SpMMs, never materialising
    P), each slab's squared norm is the trace of its Gram matrix (pmp_gram);
    one host read at the end.  Diagnostic only."""
    Pc = P if isinstance(P, Preconditioner) else Preconditioner(matrix=P)
    cx = _any_complex(A, Pc)
    A = _as_dev_csr(A, cplx=cx)
    if cx:
        Pc = Pc.as_complex()
    if Pc.dim != A.complex_n:
        raise ValueError("preconditioner does not conform with the matrix")
    # (complex: the real form R(I - A P) holds every entry twice -- columns
    # 2j and 2j+1 have equal norms -- hence the 1/sqrt(2) below)
    n, w = A.n, 32
    dev = _dev()
    E = torch.zeros((n, w), dtype=torch.float64, device=dev)
    Z = torch.empty_like(E)
    Y = torch.empty_like(E)
    tmp = [torch.empty_like(E), torch.empty_like(E)] if Pc.depth > 1 else None
    G = torch.empty((w, w), dtype=torch.float64, device=dev)
    L = _abi.lib()
    ws = scratch().get("quality_gram_ws", L.pmp_gram_workspace(n, w, w), zero=True)
    acc = torch.zeros(1, dtype=torch.float64, device=dev)
    ar = torch.arange(w, device=dev)
    for c0 in range(0, n, w):
        cw = min(w, n - c0)
        E.zero_()
        E[c0 + ar[:cw], ar[:cw]] = 1.0
        Pc.apply_dev(_abi.ptr(E), w, cw, _abi.ptr(Z), w, tmp)
        A.spmm(_abi.ptr(Z), w, cw, _abi.ptr(Y), w, alpha=-1.0, beta=1.0, Y0=_abi.ptr(E), ldy0=w)
        _abi.call("pmp_gram", n, cw, _abi.ptr(Y), w, cw, _abi.ptr(Y), w, _abi.ptr(G),
                  _abi.ptr(ws), ws.numel(), _abi.stream())
        acc += torch.diagonal(G.view(-1)[:cw * cw].view(cw, cw)).sum()
    q = float(np.sqrt(max(float(acc.item()), 0.0)))
    return q / np.sqrt(2.0) if cx else q
