"""Parametric system assembly on the B200 (kernel 1).

``SecondOrderModel.assemble(s, p)`` = (s^2 M(p) + s D(p)) + K(p)
(rpmor.py:92-107) and ``AffineFamily.evaluate(point)`` = A0 + sum c_j A_j
(affine.py:118-134) over a union pattern built once per model
(affine.py:97-116).  Term values are laid out once in HBM: a term whose
pattern is the diagonal is stored as an n-vector, every other term is
expanded onto the union pattern (one float64 per union entry), so one
streaming kernel evaluates every entry in the reference's exact operation
order (bit-identical values) and writes the CSR values -- plus the CSC copy
when the system is not symmetric -- in a single pass.
"""

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from . import _abi
from .device import DeviceCSR, Structure, _dev, f64, i32, scratch


def _canon(T):
    """as_csr (sparsecore.py:26-44): float64 when the imaginary part is zero,
    complex128 otherwise (complex terms run through the real form, cplx.py)."""
    T = sp.csr_matrix(T)
    cx = np.iscomplexobj(T.data) and T.nnz and np.any(T.data.imag != 0)
    if np.iscomplexobj(T.data) and not cx:
        T = sp.csr_matrix((T.data.real, T.indices, T.indptr), shape=T.shape)
    T = sp.csr_matrix(T, dtype=np.complex128 if cx else np.float64, copy=True)
    T.sum_duplicates()
    T.sort_indices()
    T.eliminate_zeros()
    return T


def _is_cx(c):
    return complex(c).imag != 0


def _block(a):
    """float64 unless the imaginary part is non-zero (then complex128)."""
    a = np.asarray(a)
    if np.iscomplexobj(a) and np.any(a.imag != 0):
        return a.astype(np.complex128)
    return np.asarray(a.real if np.iscomplexobj(a) else a, dtype=np.float64)


class _UnionTerms:
    """Union pattern of a list of terms and their device layout.  With
    ``with_diag`` (the complex path) the diagonal joins the union: the real
    form needs every diagonal block (cplx.py)."""

    def __init__(self, terms, with_diag=False):
        n = terms[0].shape[0]
        S = None
        for T in terms:
            ones = sp.csr_matrix((np.ones(T.nnz), T.indices, T.indptr), shape=T.shape)
            S = ones if S is None else S + ones
        S = sp.csr_matrix(S)
        self.n_added_diag = 0
        if with_diag:
            self.n_added_diag = int(n - np.count_nonzero(S.diagonal()))
            S = sp.csr_matrix(S + sp.identity(n, format="csr"))
        S.sort_indices()
        self.n = n
        self.symmetric = all(((T - T.T).nnz == 0) or not np.any((T - T.T).data) for T in terms)
        sym_pattern = (S - S.T).nnz == 0
        self.structure = Structure(n, i32(S.indptr), i32(S.indices),
                                   symmetric_pattern=sym_pattern or None)
        rows = np.repeat(np.arange(n), np.diff(S.indptr))
        self.vals = []
        self.ivals = []     # imaginary parts (None: real term)
        self.kinds = []
        for T in terms:
            Tc = T.tocoo()
            cx = np.iscomplexobj(T.data)
            if Tc.nnz and np.all(Tc.row == Tc.col):
                d = np.zeros(n, dtype=T.dtype)
                d[Tc.row] = Tc.data
                self.kinds.append(1)
            else:
                # slot of every term entry inside the union pattern: both
                # patterns are row-major sorted, so global (row, col) keys
                # are sorted and one searchsorted finds every slot
                skeys = rows.astype(np.int64) * n + S.indices
                tkeys = (np.repeat(np.arange(n, dtype=np.int64), np.diff(T.indptr)) * n
                         + T.indices)
                pos = np.searchsorted(skeys, tkeys)
                d = np.zeros(S.nnz, dtype=T.dtype)
                d[pos] = T.data
                self.kinds.append(0)
            self.vals.append(f64(d.real if cx else d))
            self.ivals.append(f64(d.imag) if cx else None)
        self.rowid = i32(rows) if 1 in self.kinds else None
        if not self.symmetric:
            self.structure.csc()

    def run(self, recipe, mode, s, zc=None):
        """recipe: list of (term index, group, first, coef).  With ``zc`` (a
        one-element int32 device slice, zeroed by the caller) the exact-zero
        count is left there and no host synchronisation happens: the caller
        checks it and calls ``finish``."""
        st = self.structure
        nt = len(recipe)
        ptrs = (ctypes_array_vp([self.vals[t].data_ptr() for t, _, _, _ in recipe]))
        kind = np.array([self.kinds[t] for t, _, _, _ in recipe], dtype=np.int32)
        group = np.array([g for _, g, _, _ in recipe], dtype=np.int32)
        first = np.array([f for _, _, f, _ in recipe], dtype=np.int32)
        coef = np.array([c for _, _, _, c in recipe], dtype=np.float64)
        out = torch.empty(max(st.nnz, 1), dtype=torch.float64, device=_dev())[:st.nnz]
        deferred = zc is not None
        if not deferred:
            zc = scratch().get("zero_count", 4, zero=False)[:4].view(torch.int32)
            zc.zero_()
        perm = out_perm = None
        if not self.symmetric:
            perm = st.csc()[2]
            out_perm = torch.empty_like(out)
        _abi.call("pmp_assemble", st.nnz, nt, ptrs, kind.ctypes.data, group.ctypes.data,
                  first.ctypes.data, coef.ctypes.data, mode, float(s), _abi.ptr(self.rowid),
                  _abi.ptr(st.colidx), _abi.ptr(out), _abi.ptr(perm), _abi.ptr(out_perm),
                  _abi.ptr(zc), _abi.stream())
        if deferred:
            return (out, out_perm)
        return self.finish((out, out_perm), int(zc.item()))

    def run_many(self, recipes, mode, svals, zc):
        """``run`` for several recipes of one shape (same terms, groups and
        opening terms) in one pmp_assemble_multi call; exact-zero counts go
        to zc[q] (device int32, zeroed by the caller).  Returns raw results
        for ``finish``."""
        import ctypes
        st = self.structure
        r0 = recipes[0]
        nt = len(r0)
        k = len(recipes)
        ptrs = ctypes_array_vp([self.vals[t].data_ptr() for t, _, _, _ in r0])
        kind = np.array([self.kinds[t] for t, _, _, _ in r0], dtype=np.int32)
        group = np.array([g for _, g, _, _ in r0], dtype=np.int32)
        first = np.array([f for _, _, f, _ in r0], dtype=np.int32)
        coef = np.array([[c for _, _, _, c in r] for r in recipes], dtype=np.float64)
        sv = np.asarray(svals, dtype=np.float64)
        # one [k, nnz] block per output (one allocation, not k): the window's
        # systems live and die together
        nz = -(-max(st.nnz, 1) // 32) * 32   # rows 256-byte aligned
        block = torch.empty((k, nz), dtype=torch.float64, device=_dev())
        outs = [block[q, :st.nnz] for q in range(k)]
        perm = None
        outs_perm = [None] * k
        if not self.symmetric:
            perm = st.csc()[2]
            pblock = torch.empty((k, nz), dtype=torch.float64, device=_dev())
            outs_perm = [pblock[q, :st.nnz] for q in range(k)]
        VP = ctypes.c_void_p * k
        h_out = VP(*[o.data_ptr() for o in outs])
        h_perm = VP(*[o.data_ptr() for o in outs_perm]) if perm is not None else None
        _abi.call("pmp_assemble_multi", st.nnz, nt, ptrs, kind.ctypes.data, group.ctypes.data,
                  first.ctypes.data, k, coef.ctypes.data, sv.ctypes.data, mode,
                  _abi.ptr(self.rowid), _abi.ptr(st.colidx), h_out, _abi.ptr(perm), h_perm,
                  _abi.ptr(zc), _abi.stream())
        _abi.note_launches(-(-k // 16) - 1)
        return list(zip(outs, outs_perm))

    def run_complex(self, recipe, mode, s):
        """Complex assembly (pmp_assemble_cplx): recipe entries (term, group,
        first, complex coef); s complex (mode 0).  Returns the real form."""
        st = self.structure
        nt = len(recipe)
        re_p = ctypes_array_vp([self.vals[t].data_ptr() for t, _, _, _ in recipe])
        im_p = ctypes_array_vp([self.ivals[t].data_ptr() if self.ivals[t] is not None else 0
                                for t, _, _, _ in recipe])
        kind = np.array([self.kinds[t] for t, _, _, _ in recipe], dtype=np.int32)
        group = np.array([g for _, g, _, _ in recipe], dtype=np.int32)
        first = np.array([f for _, _, f, _ in recipe], dtype=np.int32)
        cr = np.array([complex(c).real for _, _, _, c in recipe], dtype=np.float64)
        ci = np.array([complex(c).imag for _, _, _, c in recipe], dtype=np.float64)
        s = complex(s)
        s2 = s * s          # Python complex product, as the reference (rpmor.py:100)
        re = torch.empty(max(st.nnz, 1), dtype=torch.float64, device=_dev())[:st.nnz]
        im = torch.empty_like(re)
        zc = torch.zeros(1, dtype=torch.int32, device=_dev())
        rowid = self.rowid if self.rowid is not None else st.rowid()
        _abi.call("pmp_assemble_cplx", st.nnz, nt, re_p, im_p, kind.ctypes.data,
                  group.ctypes.data, first.ctypes.data, cr.ctypes.data, ci.ctypes.data, mode,
                  s.real, s.imag, s2.real, s2.imag, _abi.ptr(rowid), _abi.ptr(st.colidx),
                  _abi.ptr(re), _abi.ptr(im), _abi.ptr(zc), _abi.stream())
        return self.finish_complex(re, im, int(zc.item()))

    def finish_complex(self, re, im, zero_count):
        """Complex values on the union (+ diagonal) structure -> the real form
        (cplx.py).  Entries that came out exactly 0 + 0i beyond the diagonal
        positions the union added are dropped, as as_csr does: that rare
        case goes through the canonicalising host path."""
        from .cplx import realify_csr
        st = self.structure
        n = st.n
        if zero_count > self.n_added_diag:
            M = sp.csr_matrix((re.cpu().numpy() + 1j * im.cpu().numpy(), st.colidx.cpu().numpy(),
                               st.rowptr.cpu().numpy()), shape=(n, n))
            return realify_csr(M)
        if getattr(self, "real_struct", None) is None:
            rp2 = torch.empty(2 * n + 1, dtype=torch.int32, device=_dev())
            ci2 = torch.empty(max(4 * st.nnz, 1), dtype=torch.int32, device=_dev())
            v0 = torch.empty(max(4 * st.nnz, 1), dtype=torch.float64, device=_dev())
            _abi.call("pmp_realify", n, _abi.ptr(st.rowptr), _abi.ptr(st.colidx), None, None,
                      _abi.ptr(rp2), _abi.ptr(ci2), _abi.ptr(v0), _abi.stream())
            self.real_struct = Structure(2 * n, rp2, ci2[:4 * st.nnz],
                                         symmetric_pattern=st.symmetric_pattern)
        v2 = torch.empty(max(4 * st.nnz, 1), dtype=torch.float64, device=_dev())[:4 * st.nnz]
        _abi.call("pmp_realify", n, _abi.ptr(st.rowptr), _abi.ptr(st.colidx), _abi.ptr(re),
                  _abi.ptr(im), _abi.ptr(self.real_struct.rowptr), None, _abi.ptr(v2),
                  _abi.stream())
        A = DeviceCSR(self.real_struct, v2, symmetric=False)
        A.cplx = True
        A.cplx_struct = st
        A.cplx_re, A.cplx_im = re, im
        return A

    def finish(self, raw, zero_count):
        out, out_perm = raw
        if zero_count:
            return _compacted(self.structure, out)
        A = DeviceCSR(self.structure, out, symmetric=self.symmetric)
        if out_perm is not None:
            A._csc_vals = out_perm
        return A


def ctypes_array_vp(values):
    import ctypes
    arr = (ctypes.c_void_p * len(values))(*values)
    return ctypes.cast(arr, ctypes.c_void_p)


def _compacted(st, vals):
    """Drop exact zeros (as_csr, sparsecore.py:43): the system gets its own
    structure (rare path)."""
    n = st.n
    rowptr = torch.empty(n + 1, dtype=torch.int32, device=_dev())
    colidx = torch.empty(max(st.nnz, 1), dtype=torch.int32, device=_dev())
    v = torch.empty(max(st.nnz, 1), dtype=torch.float64, device=_dev())
    ws = scratch().get("compact", _abi.lib().pmp_compact_workspace(n))
    _abi.call("pmp_compact_zeros", n, _abi.ptr(st.rowptr), _abi.ptr(st.colidx), _abi.ptr(vals),
              _abi.ptr(rowptr), _abi.ptr(colidx), _abi.ptr(v), _abi.ptr(ws), ws.numel(),
              _abi.stream())
    nnz = int(rowptr[n].item())
    A = DeviceCSR(Structure(n, rowptr, colidx[:nnz]), v[:nnz], symmetric=False)
    M = A.to_scipy(drop_zeros=False)
    A.symmetric = (M - M.T).nnz == 0
    return A


@dataclass
class SecondOrderModel:
    """Second-order system s^2 M(p) + s D(p) + K(p) (rpmor.py:52-107), with
    term lists [T0, T1, ...] meaning T(p) = T0 + sum_i p_i T_i."""

    family: object = None
    mass_terms: list = None
    damping_terms: list = None
    stiffness_terms: list = None
    rhs: np.ndarray = None
    output: np.ndarray = None

    @classmethod
    def from_affine(cls, family):
        return cls(family=family, rhs=family.rhs, output=family.output)

    @classmethod
    def from_mdk(cls, mass_terms, damping_terms, stiffness_terms, rhs=None, output=None):
        def clean(ts):
            return None if ts is None else [_canon(T) for T in ts]
        m = cls(mass_terms=clean(mass_terms), damping_terms=clean(damping_terms),
                stiffness_terms=clean(stiffness_terms),
                rhs=None if rhs is None else np.atleast_2d(_block(rhs).T).T,
                output=None if output is None else _block(output))
        if m.mass_terms is None and m.damping_terms is None and m.stiffness_terms is None:
            raise ValueError("need at least one of mass/damping/stiffness terms")
        return m

    @property
    def dim(self):
        if self.family is not None:
            return self.family.dim
        for ts in (self.stiffness_terms, self.damping_terms, self.mass_terms):
            if ts is not None:
                return ts[0].shape[0]
        raise ValueError("empty model")

    def _union(self):
        u = getattr(self, "_u", None)
        if u is None:
            terms, groups = [], []
            for g, ts in enumerate((self.mass_terms, self.damping_terms, self.stiffness_terms)):
                for T in ts or []:
                    terms.append(T)
                    groups.append(g)
            u = _UnionTerms(terms)
            u.groups = groups
            self._u = u
        return u

    @property
    def structure(self):
        return self._union().structure

    @property
    def has_complex_terms(self):
        return any(np.iscomplexobj(T.data) for ts in
                   (self.mass_terms, self.damping_terms, self.stiffness_terms) for T in ts or [])

    def needs_complex(self, s, pvals):
        """Complex assembly: complex terms, shift or parameters."""
        return (self.has_complex_terms or _is_cx(s)
                or any(_is_cx(c) for c in np.atleast_1d(pvals)))

    def _union_c(self):
        u = getattr(self, "_uc", None)
        if u is None:
            terms, groups = [], []
            for g, ts in enumerate((self.mass_terms, self.damping_terms, self.stiffness_terms)):
                for T in ts or []:
                    terms.append(T)
                    groups.append(g)
            u = _UnionTerms(terms, with_diag=True)
            u.groups = groups
            self._uc = u
        return u

    def _assemble_complex(self, s, pvals):
        """(s^2 M(p) + s D(p)) + K(p) for complex s / p / terms, on the device,
        as its real form (rpmor.py:92-107 with the reference's complex
        arithmetic; cplx.py)."""
        u = self._union_c()
        pv = np.atleast_1d(np.asarray(pvals, dtype=np.complex128))
        recipe = []
        t = 0
        for g, ts in enumerate((self.mass_terms, self.damping_terms, self.stiffness_terms)):
            if ts is None:
                continue
            recipe.append((t, g, 1, 1.0))
            for i, c in enumerate(pv[:len(ts) - 1]):
                if c != 0:
                    recipe.append((t + i + 1, g, 0, complex(c)))
            t += len(ts)
        return u.run_complex(recipe, 0, complex(s))

    def reset_symbolic(self):
        """Drop every symbolic result derived from the model's sparsity
        structure -- the level-0 SPAI pattern, its CSR transpose plan, the
        least-squares size tiers and recorded symbolic plans, the CSC
        transpose -- so the next sequence recomputes them, exactly as a
        freshly constructed model would (the device term values are kept).
        Matrices assembled before the call keep the old structure."""
        u = self._union()
        st = u.structure
        u.structure = Structure(st.n, st.rowptr, st.colidx,
                                symmetric_pattern=st.symmetric_pattern)

    def assemble(self, s, pvals):
        """(s^2 M(p) + s D(p)) + K(p) as a device CSR, bit-identical to the
        reference's canonical CSR (rpmor.py:92-107)."""
        if self.family is None and self.needs_complex(s, pvals):
            return self._assemble_complex(s, pvals)
        u, recipe, s = self._recipe(s, pvals)
        return u.run(recipe, 0, s)

    def assemble_many(self, points, defer_zero_check=False):
        """assemble(s, p) for every (s, p) in ``points`` with ONE host
        synchronisation (the exact-zero counts of all systems are read
        together), so a window of systems is enqueued without stalling the
        device between them.

        ``defer_zero_check``: no synchronisation at all -- every system is
        returned on the union structure and the device tensor of exact-zero
        counts comes back too: ``(systems, counts)``.  The caller must check
        the counts before trusting the systems (a non-zero count means the
        reference's ``as_csr`` would drop entries: re-assemble without
        deferral)."""
        points = list(points)
        if not points:
            return ([], None) if defer_zero_check else []
        if any(self.needs_complex(s, p) for s, p in points):
            out = [self.assemble(s, p) for s, p in points]
            return (out, None) if defer_zero_check else out
        zc = torch.zeros(len(points), dtype=torch.int32, device=_dev())
        u = self._union()
        recs = [self._recipe(s, p) for s, p in points]
        raws = []
        i = 0
        while i < len(recs):
            # runs of one recipe shape (a term drops out when its parameter
            # is exactly 0) share one multi-system launch
            shape = [(t, g, f) for t, g, f, _ in recs[i][1]]
            j = i + 1
            while j < len(recs) and [(t, g, f) for t, g, f, _ in recs[j][1]] == shape:
                j += 1
            raws += u.run_many([r[1] for r in recs[i:j]], 0, [r[2] for r in recs[i:j]],
                               zc[i:j])
            i = j
        if defer_zero_check:
            return [u.finish(r, 0) for r in raws], zc
        counts = zc.cpu().numpy()
        return [u.finish(r, int(c)) for r, c in zip(raws, counts)]

    def _recipe(self, s, pvals):
        if self.family is not None:
            raise ValueError("affine-form models are evaluated at expansion points; "
                             "use family.evaluate")
        s = complex(s).real
        pv = [complex(c).real for c in np.atleast_1d(pvals)]
        u = self._union()
        recipe = []
        t = 0
        for g, ts in enumerate((self.mass_terms, self.damping_terms, self.stiffness_terms)):
            if ts is None:
                continue
            recipe.append((t, g, 1, 1.0))
            for i, c in enumerate(pv[:len(ts) - 1]):
                if c != 0:
                    recipe.append((t + i + 1, g, 0, c))
            t += len(ts)
        return u, recipe, s


class AffineFamily:
    """Affine family A0 + sum_j p_j A_j on the device (affine.py:60-134)."""

    def __init__(self, terms, rhs=None, output=None):
        terms = [_canon(T) for T in terms]
        if len(terms) < 2:
            raise ValueError("an affine family needs at least two terms")
        n = terms[0].shape[0]
        for T in terms:
            if T.shape != (n, n):
                raise ValueError("all terms must be square with equal dimension; got %s vs %s"
                                 % (T.shape, (n, n)))
        self.terms = terms
        self.rhs = None if rhs is None else _block(rhs).reshape(n, -1)
        self.output = None if output is None else _block(output)
        self._u = None

    @property
    def dim(self):
        return self.terms[0].shape[0]

    @property
    def n_params(self):
        return len(self.terms) - 1

    def evaluate(self, point):
        vals = getattr(point, "values", point)
        coeffs = [complex(c) for c in np.atleast_1d(vals)]
        if len(coeffs) != self.n_params:
            raise ValueError("point has %d components, family has %d parameters"
                             % (len(coeffs), self.n_params))
        if any(np.iscomplexobj(T.data) for T in self.terms) or any(c.imag != 0 for c in coeffs):
            if getattr(self, "_uc", None) is None:
                self._uc = _UnionTerms(self.terms, with_diag=True)
            recipe = [(0, 0, 1, 1.0)]
            for j, c in enumerate(coeffs):
                if c != 0:
                    recipe.append((j + 1, 0, 0, c))
            return self._uc.run_complex(recipe, 1, 0.0)
        coeffs = [c.real for c in coeffs]
        if self._u is None:
            self._u = _UnionTerms(self.terms)
        recipe = [(0, 0, 1, 1.0)]
        for j, c in enumerate(coeffs):
            if c != 0:
                recipe.append((j + 1, 0, 0, c))
        return self._u.run(recipe, 1, 0.0)


def evaluate(family, point):
    return family.evaluate(point)


def pmor_l_sequence(model, s_grid, p_grid):
    """All (A(s_k, p_j), B) systems, frequency grid outermost
    (zoo.py:268-284); matrices stay on the device."""
    s_grid, p_grid = list(s_grid), list(p_grid)
    if not s_grid or not p_grid:
        raise ValueError("both grids must be nonempty")
    if model.rhs is None:
        raise ValueError("model has no right-hand side")
    return [(model.assemble(s, np.atleast_1d(p)), model.rhs) for s in s_grid for p in p_grid]
