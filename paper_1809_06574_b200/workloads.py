"""Seeded synthetic generators for the BASELINE.json configurations c1-c5.

The reference ships no generator for these configurations (its ``zoo.py``
only builds the gyroscope / Penzl / heat families), so this module is the
single source of inputs for BOTH the oracle (``oracle/``) and the device
path: generator choices can therefore never affect parity.  The seeds,
draw orders and the unspecified details (boundary treatment, c5 shifts)
follow SURVEY.md section 8.1 and are restated in DESIGN.md.

Every generator returns a :class:`Workload` holding the mass / damping /
stiffness term lists in the form the reference's
``SecondOrderModel.from_mdk`` takes (``rpmor.py:72-81``), the (sigma, p)
grids enumerated in ``pmor_l_sequence`` order (``zoo.py:268-284``: sigma
outermost) and the right-hand-side block B.

This is host-side input generation (numpy / scipy); it is not on the
timed path.
"""

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp


@dataclass
class Workload:
    name: str
    n: int
    mass_terms: list
    damping_terms: list
    stiffness_terms: list
    s_grid: list
    p_grid: list            # list of parameter tuples (one entry per p sample)
    rhs: np.ndarray
    pattern_level: int = 0
    notes: dict = field(default_factory=dict)

    @property
    def n_systems(self):
        return len(self.s_grid) * len(self.p_grid)

    def points(self):
        """(sigma, pvals) in pmor_l_sequence order (zoo.py:280-283)."""
        return [(s, np.atleast_1d(np.asarray(p, dtype=np.float64)))
                for s in self.s_grid for p in self.p_grid]


# ---------------------------------------------------------------------------
# grid Laplacians
# ---------------------------------------------------------------------------

def _offsets(dim, kind):
    """Undirected neighbour offsets (x, y[, z]) of a stencil, one per edge
    direction: 'star' = 5-pt (2D) / 7-pt (3D); 'box' = 9-pt / 27-pt.
    Only the half whose first nonzero component, scanning from the slowest
    axis, is positive is kept."""
    import itertools
    offs = []
    for o in itertools.product((-1, 0, 1), repeat=dim):
        o = tuple(reversed(o))              # (x, y, z) with x fastest
        nz = [v for v in reversed(o) if v != 0]
        if not nz or nz[0] < 0:
            continue
        if kind == "star" and sum(abs(v) for v in o) != 1:
            continue
        offs.append(o)
    if kind not in ("star", "box"):
        raise ValueError(kind)
    return offs


def grid_laplacian(shape, kind, rng, sigma_ln, unit=False):
    """Weighted graph Laplacian K = sum_e w_e (e_a - e_b)(e_a - e_b)^T plus a
    Dirichlet ghost weight on the diagonal of every boundary node.

    shape: (nx, ny[, nz]); node index x + nx*(y + ny*z).  Edge weights are
    drawn direction by direction, then by source node id; the boundary ghost
    weights are drawn afterwards in node order.
    """
    dim = len(shape)
    shape = np.asarray(shape, dtype=np.int64)
    n = int(np.prod(shape))
    ids = np.arange(n, dtype=np.int64)
    strides = np.concatenate([[1], np.cumprod(shape[:-1])])
    coords = np.stack([(ids // strides[d]) % shape[d] for d in range(dim)], axis=1)
    rows, cols, vals = [], [], []
    diag = np.zeros(n)
    deg = np.zeros(n, dtype=np.int64)
    offs = _offsets(dim, kind)
    for off in offs:
        tgt = coords + np.asarray(off)
        ok = np.all((tgt >= 0) & (tgt < shape), axis=1)
        a = ids[ok]
        b = tgt[ok] @ strides
        w = np.ones(a.size) if unit else rng.lognormal(0.0, sigma_ln, a.size)
        rows += [a, b]
        cols += [b, a]
        vals += [-w, -w]
        np.add.at(diag, a, w)
        np.add.at(diag, b, w)
        np.add.at(deg, a, 1)
        np.add.at(deg, b, 1)
    boundary = np.flatnonzero(deg < 2 * len(offs))
    g = np.ones(boundary.size) if unit else rng.lognormal(0.0, sigma_ln, boundary.size)
    diag[boundary] += g
    rows.append(ids)
    cols.append(ids)
    vals.append(diag)
    K = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    K.sum_duplicates()
    K.sort_indices()
    return K


def _mdk_rayleigh(K_terms, Mdiag, u=None):
    """M, D = 0.1 M + 1e-3 K(p), K(p) term lists (SURVEY.md 8.1 'MDK form')."""
    M = sp.diags(Mdiag).tocsr()
    D0 = (0.1 * M + 1e-3 * K_terms[0]).tocsr()
    damping = [D0] + [(1e-3 * T).tocsr() for T in K_terms[1:]]
    for T in damping:
        T.sort_indices()
    return [M], damping, list(K_terms)


def make_config(cfg, scale=None):
    """Generator for BASELINE configs 1..5.

    ``scale`` optionally shrinks the grid (for CPU-sized parity tests) while
    keeping the stencil, distributions and draw order of the config.
    """
    if cfg == 1:
        rng = np.random.default_rng(1)
        nx = scale or 64
        K0 = grid_laplacian((nx, nx), "star", rng, 0.5)
        n = K0.shape[0]
        u = rng.uniform(0.0, 1.0, n)
        m = rng.uniform(1.0, 2.0, n)
        K1 = sp.diags(u).tocsr()
        Mt, Dt, Kt = _mdk_rayleigh([K0, K1], m)
        B = rng.standard_normal((n, 4))
        return Workload("c1", n, Mt, Dt, Kt, [0.1, 1.0, 10.0], [(0.5,), (1.0,)], B,
                        pattern_level=0)
    if cfg in (2, 4):
        seed = 2 if cfg == 2 else 4
        rng = np.random.default_rng(seed)
        nx = scale or (32 if cfg == 2 else 128)
        K0 = grid_laplacian((nx, nx, nx), "star", rng, 0.5)
        n = K0.shape[0]
        u = rng.uniform(0.0, 1.0, n)
        m = rng.uniform(1.0, 2.0, n)
        n_p = 10 if cfg == 2 else 64
        n_s = 4 if cfg == 2 else 8
        ps = rng.uniform(0.5, 2.0, n_p)
        K1 = sp.diags(u).tocsr()
        Mt, Dt, Kt = _mdk_rayleigh([K0, K1], m)
        B = rng.standard_normal((n, 8))
        return Workload("c%d" % cfg, n, Mt, Dt, Kt, list(np.logspace(-1, 1, n_s)),
                        [(float(p),) for p in ps], B, pattern_level=0)
    if cfg == 3:
        rng = np.random.default_rng(3)
        nx = scale or 64
        K0 = grid_laplacian((nx, nx, nx), "box", rng, 1.0)
        K1 = grid_laplacian((nx, nx, nx), "star", rng, 0.0, unit=True)
        n = K0.shape[0]
        u = rng.uniform(0.0, 1.0, n)
        m = rng.uniform(1.0, 2.0, n)
        pq = rng.uniform(0.5, 2.0, (32, 2))
        U = sp.diags(u).tocsr()
        Mt, Dt, Kt = _mdk_rayleigh([K0, K1, U], m)
        B = rng.standard_normal((n, 16))
        return Workload("c3", n, Mt, Dt, Kt, list(np.logspace(-1, 1, 4)),
                        [(float(a), float(b)) for a, b in pq], B, pattern_level=0)
    if cfg == 5:
        rng = np.random.default_rng(5)
        n = scale or (1 << 20)
        alpha = 0.98
        L = np.clip(np.floor(4.0 * rng.uniform(0.0, 1.0, n) ** (-1.0 / alpha)), 4, 200)
        L = L.astype(np.int64)
        rows = np.repeat(np.arange(n), L)
        cols = rng.integers(0, n, rows.size)
        vals = rng.standard_normal(rows.size)
        A = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
        A.sum_duplicates()
        K0 = ((A + A.T) * 0.5).tocsr()
        K0.setdiag(0.0)
        K0.eliminate_zeros()
        rowsum = np.asarray(abs(K0).sum(axis=1)).ravel()
        K0 = (K0 + sp.diags(1.1 * rowsum + (rowsum == 0))).tocsr()
        K0.sort_indices()
        u = rng.uniform(0.0, 1.0, n)
        m = rng.uniform(1.0, 2.0, n)
        ps = rng.uniform(0.5, 2.0, 16)
        M = sp.diags(m).tocsr()
        Mt = [M]
        Dt = [(0.05 * M).tocsr()]
        Kt = [K0, sp.diags(u).tocsr()]
        B = rng.standard_normal((n, 8))
        return Workload("c5", n, Mt, Dt, Kt, list(np.logspace(-1, 1, 4)),
                        [(float(p),) for p in ps], B, pattern_level=0,
                        notes={"shifts": "unspecified in BASELINE; logspace(-1,1,4)"})
    raise ValueError("unknown config %r" % (cfg,))
