"""CPU ORACLE — test infrastructure only, never the product path.

A plain numpy/scipy restatement, in real float64, of the reference
``pmorprec`` algorithms on the SPAI / SPAI-update / block-GCRO hot path
(reference at ``/root/reference/pkg/src/pmorprec``; citations are
``file:line`` there).  The reference computes in complex128 throughout
(``sparsecore.py:26-44``); on the all-real BASELINE inputs every imaginary
part it produces is exactly 0.0, so a real restatement
is the same computation.

Who may use this module: ``tests/`` (as the checker), ``__graft_entry__.smoke``
(as the checker) and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs (as the timed CPU baseline, kind "port").  The package
``paper_1809_06574_b200`` never imports it.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference in
the survey container on seeded inputs and commits the outputs as
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this module
against them (bit-exact for patterns / assembly, tolerance for values).
"""

import numpy as np
import scipy.linalg
import scipy.sparse as sp


# ---------------------------------------------------------------------------
# canonical sparse form (sparsecore.py:26-44)
# ---------------------------------------------------------------------------

def canon(A):
    """Real canonical CSR: duplicates summed, indices sorted, explicit zeros
    removed (sparsecore.py:26-44, restated for float64)."""
    M = sp.csr_matrix(A, dtype=np.float64, copy=True)
    M.sum_duplicates()
    M.sort_indices()
    M.eliminate_zeros()
    return M


# ---------------------------------------------------------------------------
# assembly (rpmor.py:41-49, 92-107; affine.py:97-134)
# ---------------------------------------------------------------------------

def _term_sum(terms, pvals):
    # rpmor.py:41-49: T0 + sum_{c != 0} c * T_{i+1}, scipy sparse adds
    if terms is None:
        return None
    out = terms[0].copy()
    for c, T in zip(list(pvals)[:len(terms) - 1], terms[1:]):
        if c != 0:
            out = out + c * T
    return canon(out)


def assemble_mdk(mass_terms, damping_terms, stiffness_terms, s, pvals):
    """(s^2 M(p) + s D(p)) + K(p) as canonical CSR (rpmor.py:92-107)."""
    pvals = np.atleast_1d(np.asarray(pvals, dtype=np.float64))
    s = float(s)
    acc = None
    for coef, terms in ((s * s, mass_terms), (s, damping_terms), (1.0, stiffness_terms)):
        part = _term_sum(None if terms is None else [canon(T) for T in terms], pvals)
        if part is None:
            continue
        part = coef * part
        acc = part if acc is None else acc + part
    return canon(acc)


def affine_evaluate(terms, coeffs):
    """A0 + sum_j c_j A_j over the union pattern, np.add.at in term order,
    |v| < 1e-300 pruned (affine.py:97-134)."""
    terms = [canon(T) for T in terms]
    n = terms[0].shape[0]
    S = None
    for T in terms:
        ones = sp.csr_matrix((np.ones(T.nnz), T.indices, T.indptr), shape=T.shape)
        S = ones if S is None else S + ones
    S.sort_indices()
    data = np.zeros(S.nnz)
    for j, T in enumerate(terms):
        c = 1.0 if j == 0 else float(coeffs[j - 1])
        if j > 0 and c == 0:
            continue
        Tcoo = T.tocoo()
        pos = np.empty(T.nnz, dtype=np.int64)
        for i in range(n):
            lo, hi = S.indptr[i], S.indptr[i + 1]
            tlo, thi = T.indptr[i], T.indptr[i + 1]
            pos[tlo:thi] = lo + np.searchsorted(S.indices[lo:hi], T.indices[tlo:thi])
        np.add.at(data, pos, T.data if j == 0 else c * T.data)
        del Tcoo
    A = sp.csr_matrix((data, S.indices.copy(), S.indptr.copy()), shape=(n, n))
    A.data[np.abs(A.data) < 1e-300] = 0
    A.eliminate_zeros()
    return A


# ---------------------------------------------------------------------------
# SPAI patterns (spai.py:178-222)
# ---------------------------------------------------------------------------

def col_rows(A_csc, k):
    return A_csc.indices[A_csc.indptr[k]:A_csc.indptr[k + 1]]


def level0_support(A_csc, j):
    """rows(A(:, j)) union {j} (spai.py:201-204)."""
    return np.union1d(col_rows(A_csc, j), [j]).astype(np.int64)


def level0_pattern(A):
    A_csc = canon(A).tocsc()
    return [level0_support(A_csc, j) for j in range(A_csc.shape[0])]


def abs_csc_of(A_csc):
    return sp.csc_matrix((np.abs(A_csc.data), A_csc.indices.copy(), A_csc.indptr.copy()),
                         shape=A_csc.shape)


def level1_weights(abs_csc, j):
    """|A| @ |A|[:, j] -- the same scipy sparse product the reference uses
    (spai.py:212).  Returns (rows, weights)."""
    w = (abs_csc @ abs_csc[:, [j]]).tocoo()
    return w.row.astype(np.int64), w.data


def level1_weights_ordered(abs_csc, j):
    """Explicit restatement of the product above: w_r = sum over k ascending
    of |a_rk| * |a_kj|, left to right, each product and sum rounded (no
    FMA), exact zeros dropped.  SURVEY.md 8.3 #3 measured scipy to follow
    exactly this order; tests check the two agree bit for bit."""
    acc = {}
    for k, akj in zip(col_rows(abs_csc, j), abs_csc.data[abs_csc.indptr[j]:abs_csc.indptr[j + 1]]):
        lo, hi = abs_csc.indptr[k], abs_csc.indptr[k + 1]
        for r, ark in zip(abs_csc.indices[lo:hi], abs_csc.data[lo:hi]):
            acc[r] = acc.get(r, 0.0) + ark * akj
    rows = np.array(sorted(r for r, v in acc.items() if v != 0), dtype=np.int64)
    return rows, np.array([acc[r] for r in rows])


def augment_support(abs_csc, j, base, max_fill):
    """Level-1 support: base union the top max(max_fill-|base|, 0) extra
    rows by (weight desc, row asc) (spai.py:210-222)."""
    rows, w = level1_weights(abs_csc, j)
    keep = ~np.isin(rows, base)
    rows, w = rows[keep], w[keep]
    room = max(max_fill - base.size, 0)
    if rows.size > room:
        rows = rows[np.lexsort((rows, -w))[:room]]
    return np.union1d(base, rows).astype(np.int64)


def level1_pattern(A, max_fill=80):
    A_csc = canon(A).tocsc()
    ab = abs_csc_of(A_csc)
    return [augment_support(ab, j, level0_support(A_csc, j), max_fill)
            for j in range(A_csc.shape[0])]


# ---------------------------------------------------------------------------
# column least squares (spai.py:229-292)
# ---------------------------------------------------------------------------

def touched_rows(A_csc, support, t_rows):
    """J = unique(target rows U rows of A(:, k) for k in support)
    (spai.py:237-240)."""
    parts = [np.asarray(t_rows, dtype=np.int64)]
    parts += [col_rows(A_csc, k) for k in support]
    return np.unique(np.concatenate(parts)).astype(np.int64)


def ls_column(A_csc, support, t_rows, t_vals):
    """min ||t - A z|| over supp(z) = support on the touched rows; LAPACK
    gelsy (rcond = eps) exactly as spai.py:243-253.  Returns (coef, resid,
    rank_deficient)."""
    J = touched_rows(A_csc, support, t_rows)
    if support.size == 0 or J.size == 0:
        return np.zeros(0), float(np.linalg.norm(t_vals)), False
    M = np.zeros((J.size, support.size))
    for c, k in enumerate(support):
        lo, hi = A_csc.indptr[k], A_csc.indptr[k + 1]
        M[np.searchsorted(J, A_csc.indices[lo:hi]), c] = A_csc.data[lo:hi]
    rhs = np.zeros(J.size)
    rhs[np.searchsorted(J, t_rows)] = t_vals
    coef, _, rank, _ = scipy.linalg.lstsq(M, rhs, lapack_driver="gelsy", check_finite=False)
    return coef, float(np.linalg.norm(rhs - M @ coef)), rank < support.size


def solve_columns(sys_csc, tgt_csc, pattern, ep, level, max_fill, columns, abs_csc=None):
    """Per-column solve + single augmentation pass (spai.py:273-292).
    Returns a list of (j, support, coef, resid, deficient, augmented)."""
    if level >= 1 and abs_csc is None:
        abs_csc = abs_csc_of(sys_csc)
    out = []
    for j in columns:
        sup = pattern[j]
        t_rows = col_rows(tgt_csc, j)
        t_vals = tgt_csc.data[tgt_csc.indptr[j]:tgt_csc.indptr[j + 1]]
        coef, resid, dfc = ls_column(sys_csc, sup, t_rows, t_vals)
        aug = False
        if resid > ep and level >= 1:
            sup = augment_support(abs_csc, j, sup, max_fill)
            coef, resid, dfc = ls_column(sys_csc, sup, t_rows, t_vals)
            aug = True
        out.append((j, sup, coef, resid, dfc, aug))
    return out


def assemble_columns(n, results):
    """COO(support, j, coef) -> canonical CSR + stats (spai.py:295-315)."""
    results = sorted(results, key=lambda r: r[0])
    resid = np.zeros(n)
    rows, cols, vals = [], [], []
    n_aug = n_def = 0
    for j, sup, coef, r, dfc, aug in results:
        rows.append(sup)
        cols.append(np.full(sup.size, j, dtype=np.int64))
        vals.append(coef)
        resid[j] = r
        n_aug += aug
        n_def += dfc
    P = canon(sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                            shape=(n, n)))
    return P, {"residuals": resid, "augmented_columns": n_aug,
               "rank_deficient_columns": n_def}


def spai_build(A, ep=1e-4, pattern_level=1, max_fill=80, pattern=None, columns=None):
    """Explicit SPAI (spai.py:341-364): level-0 pattern, optional single
    augmentation; an explicit pattern disables augmentation."""
    A = canon(A)
    n = A.shape[0]
    level = pattern_level if pattern is None else 0
    A_csc = A.tocsc()
    pat = pattern if pattern is not None else [level0_support(A_csc, j) for j in range(n)]
    eye = sp.identity(n, format="csc")
    res = solve_columns(A_csc, eye, pat, ep, level, max_fill,
                        range(n) if columns is None else columns)
    return assemble_columns(n, res) if columns is None else res


def update_factor(reference, system, ep=1e-4, pattern_level=1, max_fill=80,
                  pattern_source="system", columns=None):
    """Q = argmin ||reference - system Q||_F (update.py:66-75)."""
    reference, system = canon(reference), canon(system)
    src = system if pattern_source == "system" else reference
    src_csc = src.tocsc()
    n = system.shape[0]
    pat = [level0_support(src_csc, j) for j in range(n)]
    res = solve_columns(system.tocsc(), reference.tocsc(), pat, ep, pattern_level, max_fill,
                        range(n) if columns is None else columns)
    return assemble_columns(n, res) if columns is None else res


class Chain:
    """Factored preconditioner P = F0 @ F1 @ ... applied right to left
    (spai.py:82-89)."""

    def __init__(self, factors):
        self.factors = list(factors)

    def apply(self, V):
        for F in reversed(self.factors):
            V = F @ V
        return V

    @property
    def depth(self):
        return len(self.factors)


# ---------------------------------------------------------------------------
# block GCRO (krylov.py:79-275)
# ---------------------------------------------------------------------------

class Breakdown(RuntimeError):
    pass


def qr_deflate(Z, tol):
    """Pivoted QR with relative R-diagonal deflation (krylov.py:79-95)."""
    n, m = Z.shape
    if m == 0:
        return np.zeros((n, 0)), np.zeros((0, 0))
    Q, R, piv = scipy.linalg.qr(Z, mode="economic", pivoting=True)
    d = np.abs(np.diag(R))
    if d.size == 0 or d[0] == 0.0:
        return np.zeros((n, 0)), np.zeros((0, m))
    r = int(np.sum(d > tol * d[0]))
    inv = np.empty_like(piv)
    inv[piv] = np.arange(piv.size)
    return Q[:, :r].copy(), R[:r][:, inv].copy()


def _rel(norms, refs):
    out = np.zeros_like(norms)
    nz = refs > 0
    out[nz] = norms[nz] / refs[nz]
    return out


def block_gcro(A, B, P=None, tol=1e-10, max_iters=1000, outer_space_dim=10,
               inner_restart=50, deflation_tol=1e-12):
    """Right-preconditioned block GCRO restated from krylov.py:105-275.
    Returns (X, info dict with iterations / converged / residual_history /
    matvec_count / precond_apply_count)."""
    A = canon(A)
    n = A.shape[0]
    B = np.asarray(B, dtype=np.float64)
    if B.ndim == 1:
        B = B[:, None]
    s = B.shape[1]
    info = {"iterations": 0, "converged": False, "residual_history": [],
            "matvec_count": 0, "precond_apply_count": 0}
    bn = np.linalg.norm(B, axis=0)
    X = np.zeros((n, s))
    Xt = np.zeros((n, s))
    R = B.copy()
    last = np.where(bn > 0, 1.0, 0.0)
    info["residual_history"].append(last.copy())
    active = np.flatnonzero(bn > 0)

    def op(V):
        if P is not None:
            V = P.apply(V)
            info["precond_apply_count"] += V.shape[1]
        info["matvec_count"] += V.shape[1]
        return A @ V

    U = C = None
    cap = inner_restart + 2 * s + 2
    while active.size and info["iterations"] < max_iters:
        na = active.size
        Ra = R[:, active]
        start = _rel(np.linalg.norm(Ra, axis=0), bn[active])
        k = 0 if C is None else C.shape[1]
        if k:
            rhs_c = C.T @ Ra
            Z0 = Ra - C @ rhs_c
        else:
            rhs_c = np.zeros((0, na))
            Z0 = Ra
        V1, S0 = qr_deflate(Z0, deflation_tol)
        bs = V1.shape[1]
        if bs == 0:
            raise Breakdown("projected residual block vanished")
        V = np.zeros((n, cap))
        V[:, :bs] = V1
        H = np.zeros((cap, cap))
        Bm = np.zeros((k, cap))
        rv = np.zeros((cap, na))
        rv[:bs] = S0
        m, total, Y = 0, bs, None
        exhausted = done = False
        while info["iterations"] < max_iters and not done and not exhausted and m < inner_restart:
            q0, q1 = m, total
            W = op(V[:, q0:q1])
            info["iterations"] += 1
            if k:
                Bb = C.T @ W
                Bm[:, q0:q1] = Bb
                W = W - C @ Bb
            for _ in range(2):
                Hc = V[:, :total].T @ W
                W = W - V[:, :total] @ Hc
                H[:total, q0:q1] += Hc
            Qn, Rn = qr_deflate(W, deflation_tol)
            bn_next = Qn.shape[1]
            V[:, total:total + bn_next] = Qn
            H[total:total + bn_next, q0:q1] = Rn
            m = total
            total += bn_next
            G = np.zeros((k + total, k + m))
            if k:
                G[:k, :k] = np.eye(k)
                G[:k, k:] = Bm[:, :m]
            G[k:, k:] = H[:total, :m]
            rhs = np.vstack([rhs_c, rv[:total]])
            Y = np.linalg.lstsq(G, rhs, rcond=None)[0]
            est = _rel(np.linalg.norm(rhs - G @ Y, axis=0), bn[active])
            last[active] = est
            info["residual_history"].append(last.copy())
            done = bool(np.all(est <= tol))
            exhausted = bn_next == 0
        if Y is None:
            break
        dXt = V[:, :m] @ Y[k:]
        if k:
            dXt += U @ Y[:k]
        Xt[:, active] += dXt
        if P is not None:
            Xa = P.apply(Xt[:, active])
            info["precond_apply_count"] += na
        else:
            Xa = Xt[:, active]
        X[:, active] = Xa
        Rt = B[:, active] - A @ Xa
        info["matvec_count"] += na
        R[:, active] = Rt
        true = _rel(np.linalg.norm(Rt, axis=0), bn[active])
        last[active] = true
        info["residual_history"].append(last.copy())
        still = true > tol
        if exhausted and np.all(still) and np.all(true >= start * (1 - 1e-10)):
            raise Breakdown("Krylov subspace exhausted without residual reduction")
        img = G @ Y
        images = V[:, :total] @ img[k:]
        if k:
            images += C @ img[:k]
        for col in range(na):
            w = images[:, col].copy()
            z = dXt[:, col].copy()
            w0 = np.linalg.norm(w)
            if w0 == 0.0:
                continue
            if C is not None:
                for _ in range(2):
                    h = C.T @ w
                    w -= C @ h
                    z -= U @ h
            nw = np.linalg.norm(w)
            if nw <= 1e-10 * w0:
                continue
            C = (w / nw)[:, None] if C is None else np.hstack([C, (w / nw)[:, None]])
            U = (z / nw)[:, None] if U is None else np.hstack([U, (z / nw)[:, None]])
        if C is not None and C.shape[1] > outer_space_dim:
            C = C[:, -outer_space_dim:].copy()
            U = U[:, -outer_space_dim:].copy()
        active = active[still]
    info["converged"] = active.size == 0
    return X, info


# ---------------------------------------------------------------------------
# sequence composition (rpmor.py:199-218, zoo.py:268-284)
# ---------------------------------------------------------------------------

def run_sequence(workload, kind="spai-update-first", level=0, tol=1e-8, systems=None,
                 ep=1e-4, max_fill=80):
    """assemble -> SPAI (first system) / update -> block GCRO for each
    (sigma, p) system in pmor_l_sequence order.  ``systems`` restricts the
    solved systems (the base SPAI is always built)."""
    pts = workload.points()
    A1 = P1 = Aprev = Pprev = None
    out = []
    for idx, (s, p) in enumerate(pts):
        if (systems is not None and idx not in systems and idx > 0
                and kind == "spai-update-first"):
            continue        # independent of (A1, P1) only: nothing to carry
        A = assemble_mdk(workload.mass_terms, workload.damping_terms,
                         workload.stiffness_terms, s, p)
        if idx == 0 or kind == "spai":
            Pm, st = spai_build(A, ep=ep, pattern_level=level, max_fill=max_fill)
            P = Chain([Pm])
        elif kind == "spai-update-first":
            Q, st = update_factor(A1, A, ep=ep, pattern_level=level, max_fill=max_fill)
            P = Chain([Q] + P1.factors)
        else:
            Q, st = update_factor(Aprev, A, ep=ep, pattern_level=level, max_fill=max_fill)
            P = Chain([Q] + Pprev.factors)
        if idx == 0:
            A1, P1 = A, P
        Aprev, Pprev = A, P
        if systems is None or idx in systems:
            X, info = block_gcro(A, workload.rhs, P, tol=tol)
            out.append((idx, X, info, st))
    return out


# ---------------------------------------------------------------------------
# moment pipeline (rpmor.py:271-362, sparsecore.py:176-204)
# ---------------------------------------------------------------------------

def extend_orthonormal_basis(Q, X, tol_drop=1e-10):
    """Modified Gram-Schmidt, two passes, relative drop test
    (sparsecore.py:176-204)."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    kept = [] if Q is None else [np.ascontiguousarray(Q[:, j]) for j in range(Q.shape[1])]
    for j in range(X.shape[1]):
        v = X[:, j].copy()
        norm0 = np.linalg.norm(v)
        if norm0 == 0.0:
            continue
        for _ in range(2):
            for q in kept:
                v -= q * np.dot(q, v)
        nrm = np.linalg.norm(v)
        if nrm <= tol_drop * norm0:
            continue
        kept.append(v / nrm)
    return np.column_stack(kept) if kept else np.zeros((n, 0))


def rpmor_reduce(terms, B, C, points, levels=1, tol=1e-10, kind="spai-update-first",
                 pattern_level=0, drop_tol=1e-10):
    """rpmor.py:307-362 with the SequencePreconditioner of rpmor.py:189-218
    (kind "none", "spai" or "spai-update-first").  Returns (reduced terms,
    reduced rhs, reduced output, basis, per-call iteration counts)."""
    terms = [canon(T) for T in terms]
    V, iters = None, []
    A1 = P1 = None
    for pt in points:
        A = affine_evaluate(terms, list(pt))
        if kind == "none":
            P = None
        elif kind == "spai" or P1 is None:
            P, _ = spai_build(A, pattern_level=pattern_level)
            P = Chain([P])
            if A1 is None:
                A1, P1 = A, P
        else:
            Q, _ = update_factor(A1, A, pattern_level=pattern_level)
            P = Chain([Q] + P1.factors)
        X0, info = block_gcro(A, B, P, tol=tol)
        iters.append(info["iterations"])
        V = extend_orthonormal_basis(V, X0, drop_tol)
        parents = X0
        for _ in range(levels):
            blocks = []
            for c in range(parents.shape[1]):
                rhs = np.hstack([T @ parents[:, [c]] for T in terms[1:]])
                Xh, info = block_gcro(A, rhs, P, tol=tol)
                iters.append(info["iterations"])
                V = extend_orthonormal_basis(V, Xh, drop_tol)
                blocks.append(Xh)
            parents = np.hstack(blocks)
    red = [V.T @ (T @ V) for T in terms]
    return red, V.T @ B, C.T @ V, V, iters
