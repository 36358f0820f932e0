"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference's LOBPCG hot
path (/root/reference/proj/src), used as the CPU checker. Every function cites
the reference code it restates. Pinned against the compiled reference via the
golden fixtures in tests/golden (make_golden.py); where this port is bitwise
faithful (spmm, block_inner, linear_combination, random_block, choose_shifts,
the generator) the tests compare bitwise, elsewhere within the tolerance the
tests state (LAPACK factorizations stand in for Eigen's).

Never imported by the product path (paper_1609_01689_b200/).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

M64 = (1 << 64) - 1
K_PANEL_ROWS = 256  # block_vectors.hpp:57
K_TINY_DIAG = 1e-300  # lobpcg.cpp:14


# ----------------------------------------------------------------- rng.hpp

def mix64(x):
    """splitmix64 finalizer (rng.hpp:13-20), vectorised over uint64 arrays."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint64(30))
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x = x ^ (x >> np.uint64(27))
        x = x * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def hash3(seed, i, j):
    """rng.hpp:23-28."""
    with np.errstate(over="ignore"):
        h = mix64(np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15))
        h = mix64(h ^ (np.asarray(i, dtype=np.uint64) + np.uint64(0xD1B54A32D192ED03)))
        h = mix64(h ^ (np.asarray(j, dtype=np.uint64) + np.uint64(0x8CB92BA72F3D8DD7)))
    return h


def unit_double(h):
    """rng.hpp:31-33."""
    return (np.asarray(h, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def random_block(dim, width, seed):
    """block_vectors.cpp:162-174: entry (i, j) = 2 unit(hash3(seed, i, j)) - 1."""
    i = np.arange(dim, dtype=np.uint64)[:, None]
    j = np.arange(width, dtype=np.uint64)[None, :]
    return 2.0 * unit_double(hash3(seed, i, j)) - 1.0


# ---------------------------------------------------- generator (new code)
# Restatement of paper_1609_01689_b200/csrc/generator.cpp + gen_common.h (the
# BASELINE sector generator has no reference counterpart).

def _portable_log(x):
    m, e = np.frexp(x)
    small = m < 0.70710678118654752440
    m = np.where(small, m * 2.0, m)
    e = np.where(small, e - 1, e)
    s = (m - 1.0) / (m + 1.0)
    s2 = s * s
    coeffs = [2.0 / 23.0, 2.0 / 21.0, 2.0 / 19.0, 2.0 / 17.0, 2.0 / 15.0, 2.0 / 13.0, 2.0 / 11.0, 2.0 / 9.0,
              2.0 / 7.0, 2.0 / 5.0, 2.0 / 3.0, 2.0]
    p = np.full_like(s, coeffs[0])
    for c in coeffs[1:]:
        p = _fma(p, s2, c)
    lnm = p * s
    de = e.astype(np.float64)
    return _fma(de, 6.93147180369123816490e-01, _fma(de, 1.90821492927058770002e-10, lnm))


def _fma(a, b, c):
    """Correctly rounded a*b+c (numpy has no fma; exact via fractions for the
    generator's small pinning cases)."""
    a, b, c = np.broadcast_arrays(np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64),
                                  np.asarray(c, dtype=np.float64))
    out = np.empty(a.shape)
    from fractions import Fraction

    fa, fb, fc = a.ravel(), b.ravel(), c.ravel()
    o = out.ravel()
    for k in range(fa.size):
        o[k] = float(Fraction(float(fa[k])) * Fraction(float(fb[k])) + Fraction(float(fc[k])))
    return out


def _sin_poly(r):
    r2 = r * r
    p = np.full_like(r, -1.0 / 1307674368000.0)
    for c in (1.0 / 6227020800.0, -1.0 / 39916800.0, 1.0 / 362880.0, -1.0 / 5040.0, 1.0 / 120.0, -1.0 / 6.0):
        p = _fma(p, r2, c)
    return _fma(p * r2, r, r)


def _cos_poly(r):
    r2 = r * r
    p = np.full_like(r, 1.0 / 20922789888000.0)
    for c in (-1.0 / 87178291200.0, 1.0 / 479001600.0, -1.0 / 3628800.0, 1.0 / 40320.0, -1.0 / 720.0, 1.0 / 24.0,
              -0.5):
        p = _fma(p, r2, c)
    return _fma(p, r2, 1.0)


def _cos_2pi(u):
    v = u - np.where(u >= 0.5, 1.0, 0.0)
    w = 4.0 * v
    k = np.where(w >= 0.0, np.floor(w + 0.5), -np.floor(-w + 0.5))
    r = (w - k) * 1.57079632679489661923
    q = k.astype(np.int64) & 3
    return np.select([q == 0, q == 1, q == 2], [_cos_poly(r), -_sin_poly(r), -_cos_poly(r)], _sin_poly(r))


def _normal(h1, h2):
    u1 = unit_double(h1)
    u2 = unit_double(h2)
    return np.sqrt(-2.0 * _portable_log(1.0 - u1)) * _cos_2pi(u2)


@dataclasses.dataclass
class OracleCsb:
    dim: int
    precision: int
    block_boundaries: np.ndarray
    entry_offsets: np.ndarray
    rows: np.ndarray
    cols: np.ndarray
    values: np.ndarray
    groups: np.ndarray


def generate(n, sectors, tile, p, q, seed, precision, beta=2000, band=2) -> OracleCsb:
    """Slow, small-size restatement of generator.cpp (pinning only)."""
    seeds = [int(hash3(seed, k, 0)) for k in (1, 2, 3, 4, 5)]
    s_tile, s_q, s_v1, s_v2, s_d = seeds
    ss = [(n * s) // sectors for s in range(sectors + 1)]
    starts, sec = [], []
    for s in range(sectors):
        for r in range(ss[s], ss[s + 1], tile):
            starts.append(r)
            sec.append(s)
    starts.append(n)
    nt = len(sec)
    # expectation -> value scale
    diag_off, cand = 0.0, 0.0
    rows_s = np.zeros(sectors)
    t2 = np.zeros(sectors)
    for t in range(nt):
        sz = starts[t + 1] - starts[t]
        diag_off += q * sz * (sz - 1.0) / 2.0
        t2[sec[t]] += sz * sz
        rows_s[sec[t]] += sz
    for s in range(sectors):
        cand += (rows_s[s] * rows_s[s] - t2[s]) / 2.0
        for s2 in range(max(0, s - band), s):
            cand += rows_s[s] * rows_s[s2]
    avg = 2.0 * (diag_off + p * q * cand) / n
    scale = 1.0 / math.sqrt(avg) if avg > 0 else 0.0
    kept = []
    for I in range(nt):
        lo = max(0, sec[I] - band)
        J0 = next(t for t in range(nt) if starts[t] >= ss[lo])
        row = [J for J in range(J0, I) if unit_double(hash3(s_tile, I, J)) < p]
        kept.append(row + [I])
    # CSB blocks
    bb = [0]
    tile_block = []
    for t in range(nt):
        s, e = starts[t], starts[t + 1]
        stratum = s != 0 and ss[sec[t]] == s
        if s > bb[-1] and (stratum or e - bb[-1] > beta):
            bb.append(s)
        tile_block.append(len(bb) - 1)
    bb.append(n)
    nb = len(bb) - 1
    blocks = {}
    for I in range(nt):
        for a in range(starts[I], starts[I + 1]):
            for J in kept[I]:
                BJ = tile_block[J]
                ce = a if J == I else starts[J + 1]
                bs = np.arange(starts[J], ce, dtype=np.uint64)
                if bs.size:
                    keep = unit_double(hash3(s_q, a, bs)) < q
                    bs = bs[keep]
                    if bs.size:
                        z = _normal(hash3(s_v1, a, bs), hash3(s_v2, a, bs)) * scale
                        lst = blocks.setdefault((tile_block[I], BJ), [])
                        lst.extend(zip([a] * bs.size, bs.tolist(), z.tolist()))
                if J == I:
                    u = float(unit_double(hash3(s_d, a, a)))
                    blocks.setdefault((tile_block[I], BJ), []).append((a, a, 10.0 * sec[I] + 4.0 * u - 2.0))
    offs = [0]
    R, Cc, V = [], [], []
    for BI in range(nb):
        for BJ in range(BI + 1):
            lst = blocks.get((BI, BJ), [])
            for a, b, v in lst:
                R.append(a - bb[BI])
                Cc.append(b - bb[BJ])
                V.append(v)
            offs.append(offs[-1] + len(lst))
    vals = np.array(V, dtype=np.float64)
    return OracleCsb(n, precision, np.array(bb, np.uint32), np.array(offs, np.uint64), np.array(R, np.uint16),
                     np.array(Cc, np.uint16), vals.astype(np.float32) if precision == 0 else vals,
                     np.array(starts, np.uint32))


# ----------------------------------------------------------------- csb.cpp

def _global_entries(h):
    nb = len(h.block_boundaries) - 1
    counts = np.diff(np.asarray(h.entry_offsets, dtype=np.int64))
    bi = np.concatenate([np.full(i + 1, i) for i in range(nb)])
    bj = np.concatenate([np.arange(i + 1) for i in range(nb)])
    bb = np.asarray(h.block_boundaries, dtype=np.int64)
    ei = np.repeat(bi, counts)
    ej = np.repeat(bj, counts)
    r = bb[ei] + np.asarray(h.rows, dtype=np.int64)
    c = bb[ej] + np.asarray(h.cols, dtype=np.int64)
    return r, c, np.asarray(h.values).astype(np.float64), ei, ej


def spmm(h, x):
    """spmm_serial (csb.cpp:195-201): phase one walks block rows in order
    (apply_block, :118-128), phase two walks block columns (apply_block_
    transposed, :130-141) skipping the diagonal of diagonal blocks; each product
    is formed in fp64 and added sequentially -- np.add.at is unbuffered and
    ordered, so this is bitwise the reference's serial accumulation."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape[0] != h.dim:
        raise ValueError("DimensionMismatch: spmm: vector dim != matrix dim")
    r, c, v, ei, ej = _global_entries(h)
    u = np.zeros_like(x)
    np.add.at(u, r, v[:, None] * x[c])
    # phase two order: block column j ascending, block row i >= j ascending, entries in order
    nb = len(h.block_boundaries) - 1
    order_blocks = sorted(((j, i) for i in range(nb) for j in range(i + 1)))
    offs = np.asarray(h.entry_offsets, dtype=np.int64)
    idx = []
    for j, i in order_blocks:
        b = i * (i + 1) // 2 + j
        e = np.arange(offs[b], offs[b + 1])
        if i == j:
            e = e[r[e] != c[e]]
        idx.append(e)
    idx = np.concatenate(idx) if idx else np.zeros(0, np.int64)
    np.add.at(u, c[idx], v[idx, None] * x[r[idx]])
    return u


def to_dense(h):
    """csb.cpp:220-237."""
    r, c, v, _, _ = _global_entries(h)
    m = np.zeros((h.dim, h.dim))
    m[r, c] = v
    m[c, r] = v
    return m


# --------------------------------------------------------- block_vectors.cpp

def block_inner(x, y):
    """block_vectors.cpp:57-97: 256-row panels, rows accumulated in order
    within a panel (cumsum is sequential), panels summed in panel order."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    n = x.shape[0]
    res = np.zeros((x.shape[1], y.shape[1]))
    for lo in range(0, n, K_PANEL_ROWS):
        prod = x[lo:lo + K_PANEL_ROWS, :, None] * y[lo:lo + K_PANEL_ROWS, None, :]
        res = res + np.cumsum(prod, axis=0)[-1]
    return res


def linear_combination(y, g):
    """block_vectors.cpp:101-129: out[i][c] = sum_t y[i][t] g[t][c], t in order."""
    y = np.asarray(y, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    if g.shape[0] != y.shape[1]:
        raise ValueError("DimensionMismatch: linear_combination: G rows != block width")
    if y.shape[1] == 0:
        return np.zeros((y.shape[0], g.shape[1]))
    return np.cumsum(y[:, :, None] * g[None, :, :], axis=1)[:, -1, :]


def add_linear_combination(y, x, g):
    """block_vectors.cpp:139-160 (returns the updated copy)."""
    return np.asarray(y, dtype=np.float64) + linear_combination(x, g)


def column_norms(x):
    return np.sqrt(np.diag(block_inner(x, x)))


# -------------------------------------------------------------- precond.cpp

@dataclasses.dataclass
class PrecondConfig:
    inner_iters: int = 3
    small_block_cutoff: int = 64
    engage_after: int = 3
    relres_gate: float = 1e-1
    near_converged_factor: float = 10.0
    far_threshold: float = 1e-2
    column_floor_factor: float = 100.0


def choose_shifts(theta, res_norm, x_norm, relres, iteration, tol, cfg=PrecondConfig()):
    """precond.cpp:13-55."""
    k = len(theta)
    mu = list(map(float, theta))
    engage = [True] * k
    if iteration <= cfg.engage_after:
        engage = [False] * k
    elif k and relres[0] > cfg.relres_gate:
        engage = [False] * k
    else:
        for j in range(k):
            if relres[j] <= cfg.column_floor_factor * tol:
                engage[j] = False
    for j in range(k):
        backed = theta[j] - 2.0 * res_norm[j] / x_norm[j]
        mu[j] = backed if j == 0 else min(backed, mu[0])
    first_far = k
    for i in range(k):
        if relres[i] > cfg.far_threshold:
            first_far = i
            break
    if first_far < k:
        carried = mu[first_far - 1 if first_far > 0 else 0]
        for t in range(first_far, k):
            mu[t] = carried
    return np.array(mu), np.array(engage)


def _lu_factor(a):
    import scipy.linalg

    return scipy.linalg.lu_factor(a, check_finite=False)


def direct_solve(block, mu, rhs):
    """precond.cpp:61-83: LU of (block - mu I), singular test |U_ii| <= 1e-14
    max|U_ii|, one perturbation, else pass-through."""
    import scipy.linalg

    n = block.shape[0]
    for shift in (mu, mu + 1e-8 * (1.0 + abs(mu))):
        lu = _lu_factor(block - shift * np.eye(n))
        d = np.abs(np.diag(lu[0]))
        if d.min() > 1e-14 * max(d.max(), 1e-300):
            return scipy.linalg.lu_solve(lu, rhs, check_finite=False), True
    return rhs, False


def fom_solve(block, mu, rhs, iters):
    """precond.cpp:87-158 (fused multi-RHS FOM, 2-pass MGS, lucky breakdown)."""
    if iters < 1:
        raise ValueError("ConfigError: fom_solve: iters must be >= 1")
    n, k = rhs.shape
    m_max = min(iters, n)
    x = np.zeros((n, k))
    basis = [None] * k
    hess = [None] * k
    beta = np.zeros(k)
    steps = [0] * k
    active = [False] * k
    for j in range(k):
        beta[j] = np.linalg.norm(rhs[:, j])
        if beta[j] == 0.0:
            continue
        basis[j] = np.zeros((n, m_max + 1))
        hess[j] = np.zeros((m_max + 1, m_max))
        basis[j][:, 0] = rhs[:, j] / beta[j]
        active[j] = True

    def finish(j, m):
        hm = hess[j][:m, :m]
        e1 = np.zeros(m)
        e1[0] = beta[j]
        y = np.linalg.solve(hm, e1)
        x[:, j] = basis[j][:, :m] @ y
        active[j] = False

    for m in range(m_max):
        cols = [j for j in range(k) if active[j]]
        if not cols:
            break
        vm = np.stack([basis[j][:, m] for j in cols], axis=1)
        z = block @ vm
        for c, j in enumerate(cols):
            w = z[:, c] - mu[j] * vm[:, c]
            scale = max(beta[j], np.linalg.norm(w))
            for p in range(2):
                for i in range(m + 1):
                    hij = basis[j][:, i] @ w
                    hess[j][i, m] = hij if p == 0 else hess[j][i, m] + hij
                    w = w - hij * basis[j][:, i]
            norm = np.linalg.norm(w)
            steps[j] = m + 1
            if norm <= 1e-12 * max(scale, 1.0):
                hess[j][m + 1, m] = 0.0
                finish(j, m + 1)
                continue
            hess[j][m + 1, m] = norm
            basis[j][:, m + 1] = w / norm
    for j in range(k):
        if active[j]:
            finish(j, steps[j])
    return x


def extract_tile_diagonal(h, groups):
    """hamiltonian.cpp:178-203."""
    d = to_dense(h) if h.dim <= 20000 else None
    out = []
    for g in range(len(groups) - 1):
        s, e = int(groups[g]), int(groups[g + 1])
        if d is not None:
            out.append(d[s:e, s:e].copy())
    return out


def apply_preconditioner(blocks, bounds, r, mu, engage, cfg=PrecondConfig()):
    """precond.cpp:160-207."""
    w = np.array(r, dtype=np.float64, copy=True)
    eng = [j for j in range(r.shape[1]) if engage[j]]
    if not eng:
        return w
    for g, blk in enumerate(blocks):
        s, e = int(bounds[g]), int(bounds[g + 1])
        n = e - s
        rhs = r[s:e][:, eng].copy()
        if n <= cfg.small_block_cutoff:
            by = {}
            for c, j in enumerate(eng):
                by.setdefault(float(mu[j]), []).append(c)
            for shift in sorted(by):
                cols = by[shift]
                sol, _ = direct_solve(blk, shift, rhs[:, cols])
                rhs[:, cols] = sol
        else:
            rhs = fom_solve(blk, [mu[j] for j in eng], rhs, cfg.inner_iters)
        w[s:e, eng] = rhs
    return w


# --------------------------------------------------------------- lobpcg.cpp

def _rank_revealing_select(gram, orig_sq, drop_tol):
    """lobpcg.cpp:20-51."""
    gram = np.array(gram, dtype=np.float64, copy=True)
    m = gram.shape[0]
    active = [True] * m
    kept = []
    for _ in range(m):
        pivot, best = -1, -1.0
        for j in range(m):
            if active[j] and gram[j, j] > best:
                best, pivot = gram[j, j], j
        if pivot < 0:
            break
        active[pivot] = False
        thr = max(drop_tol * drop_tol * orig_sq[pivot], K_TINY_DIAG)
        if not gram[pivot, pivot] > thr:
            continue
        kept.append(pivot)
        d = gram[pivot, pivot]
        for a in range(m):
            if not active[a]:
                continue
            for b in range(m):
                if not active[b] and b != a:
                    continue
                gram[a, b] -= gram[a, pivot] * gram[b, pivot] / d
    return sorted(kept)


def _llt_rinv(a):
    try:
        L = np.linalg.cholesky(a)
    except np.linalg.LinAlgError:
        return None
    import scipy.linalg

    return scipy.linalg.solve_triangular(L.T, np.eye(a.shape[0]), lower=False)


def orthonormalize(y, drop_tol=1e-8, against=None, inner=block_inner):
    """lobpcg.cpp:89-119. `inner` computes X^T Y (a sharded run passes a
    local-partial + all-reduce)."""
    v = np.array(y, dtype=np.float64, copy=True)
    if v.shape[1] == 0:
        return v
    orig_sq = np.diag(inner(y, y)).copy()
    if against is not None and against.shape[1] > 0:
        for _ in range(2):
            c = inner(against, v)
            v = add_linear_combination(v, against, -c)
    gram = inner(v, v)
    kept = _rank_revealing_select(gram, orig_sq, drop_tol)
    while kept:
        q = v[:, kept]
        rinv = _llt_rinv(gram[np.ix_(kept, kept)])
        if rinv is not None:
            q = linear_combination(q, rinv)
            r2 = _llt_rinv(inner(q, q))
            if r2 is not None:
                q = linear_combination(q, r2)
            return q
        kept.pop()
    return np.zeros((y.shape[0], 0))


def _eig_sym(a):
    return np.linalg.eigh(0.5 * (a + a.T))


@dataclasses.dataclass
class Report:
    eigenvalues: np.ndarray
    trial_vectors: np.ndarray
    history: list
    counters: list
    converged: bool
    iterations: int
    norm_estimate: float
    active_sets: list


def lobpcg_solve(h, x0, k_want, tol, max_iter=500, tiles=None, bounds=None, cfg=PrecondConfig(), matvec=None,
                 inner=block_inner):
    """lobpcg.cpp:216-387, verbatim control flow. `tiles`/`bounds` give the
    dense tile diagonal (None = unpreconditioned); `matvec` overrides the SpMM;
    `inner` overrides X^T Y -- together they run the same loop on a row shard
    (local rows, all-gathered SpMM input, all-reduced Grams)."""
    block_inner = inner  # noqa: N806 -- every Gram below goes through the hook
    if x0.shape[1] < k_want:
        raise ValueError("ConfigError: lobpcg: trial width below k_want")
    apply = matvec or (lambda v: spmm(h, v))
    counters = [0, 0, 0, 0]
    drop_tol = 1e-8
    x = orthonormalize(x0, drop_tol, inner=inner)
    counters[3] += 1
    if x.shape[1] < k_want:
        raise ValueError("SubspaceCollapse: initial block has fewer than k_want independent columns")
    kt = x.shape[1]

    def apply_h(v):
        counters[0] += 1
        counters[1] += v.shape[1]
        return apply(v)

    hx = apply_h(x)
    ev, vec = _eig_sym(block_inner(x, hx))
    theta = ev[:kt].copy()
    x = linear_combination(x, vec)
    hx = linear_combination(hx, vec)
    norm_est = max(abs(theta[0]), abs(theta[-1]))
    n = x.shape[0]
    p = np.zeros((n, 0))
    hp = np.zeros((n, 0))
    history, active_sets = [], []
    converged, iterations = False, 0
    it = 0
    while True:
        r = hx - x * theta[None, :]
        res_norm = np.sqrt(np.diag(block_inner(r, r)))
        relres = res_norm / max(norm_est, K_TINY_DIAG)
        for j in range(kt):
            history.append((it, j, float(relres[j]), float(theta[j])))
        iterations = it
        if all(relres[j] <= tol for j in range(k_want)):
            converged = True
            break
        if it >= max_iter:
            break
        if tiles is not None:
            mu, engage = choose_shifts(theta, res_norm, np.ones(kt), relres, it + 1, tol, cfg)
            wsrc = apply_preconditioner(tiles, bounds, r, mu, engage, cfg)
            if engage.any():
                counters[2] += 1
        else:
            wsrc = r
        active = [j for j in range(kt) if relres[j] > tol]
        active_sets.append(active)
        w = orthonormalize(wsrc[:, active], drop_tol, np.hstack([x, p]), inner=inner)
        counters[3] += 1
        if w.shape[1] == 0:
            break
        hw = apply_h(w)
        kw = w.shape[1]
        y = np.hstack([x, w, p])
        hy = np.hstack([hx, hw, hp])
        ok = True
        overlap = block_inner(y, y)
        if np.abs(overlap - np.eye(y.shape[1])).max() > 1e-8:
            ok = False
        else:
            try:
                ev, vec = _eig_sym(block_inner(y, hy))
            except np.linalg.LinAlgError:
                ok = False
        if not ok:
            p = np.zeros((n, 0))
            hp = np.zeros((n, 0))
            y = np.hstack([x, w])
            hy = np.hstack([hx, hw])
            ev, vec = _eig_sym(block_inner(y, hy))
        m = y.shape[1]
        kp = m - kt - kw
        theta = ev[:kt].copy()
        norm_est = max(norm_est, abs(ev[0]), abs(ev[m - 1]))
        g = vec[:, :kt]
        g1, g2, g3 = g[:kt], g[kt:kt + kw], g[kt + kw:]
        xn = add_linear_combination(linear_combination(x, g1), w, g2)
        hxn = add_linear_combination(linear_combination(hx, g1), hw, g2)
        pn = linear_combination(w, g2)
        hpn = linear_combination(hw, g2)
        if kp > 0:
            xn = add_linear_combination(xn, p, g3)
            hxn = add_linear_combination(hxn, hp, g3)
            pn = add_linear_combination(pn, p, g3)
            hpn = add_linear_combination(hpn, hp, g3)
        x, hx, p, hp = xn, hxn, pn, hpn
        xg = block_inner(x, x)
        if np.abs(xg - np.eye(kt)).max() > 1e-12:
            rinv = _llt_rinv(xg)
            if rinv is not None:
                x = linear_combination(x, rinv)
                hx = linear_combination(hx, rinv)
                counters[3] += 1
        # clean_p_block (lobpcg.cpp:180-212)
        if p.shape[1] > 0:
            for _ in range(2):
                c = block_inner(x, p)
                p = add_linear_combination(p, x, -c)
                hp = add_linear_combination(hp, hx, -c)
            gram = block_inner(p, p)
            kept = _rank_revealing_select(gram, np.diag(gram).copy(), drop_tol)
            if not kept:
                p, hp = np.zeros((n, 0)), np.zeros((n, 0))
            else:
                rinv = _llt_rinv(gram[np.ix_(kept, kept)])
                if rinv is None:
                    p, hp = np.zeros((n, 0)), np.zeros((n, 0))
                else:
                    p = linear_combination(p[:, kept], rinv)
                    hp = linear_combination(hp[:, kept], rinv)
        counters[3] += 1
        it += 1
    return Report(theta[:k_want].copy(), x, history, counters, converged, iterations, norm_est, active_sets)


# ------------------------------------------------------------- lanczos.cpp

def lanczos_checkpoint(m):
    """lanczos.cpp:11-15: every 10 steps to 100, every 20 to 200, then 40."""
    if m <= 100:
        return m % 10 == 0
    if m <= 200:
        return m % 20 == 0
    return m % 40 == 0


def symmetric_double(seed, i, j):
    """rng.hpp:33-36."""
    return 2.0 * unit_double(hash3(seed, i, j)) - 1.0


def lanczos_solve(matvec, v0, k_want, tol, max_iter=500):
    """lanczos.cpp:24-136: Lanczos with two-pass full reorthogonalisation,
    seeded random restart on breakdown, Ritz analysis on the checkpoint grid.
    `matvec(v)` applies H to an (n, 1) block (spmm with m = 1). numpy's
    LAPACK eigh stands in for Eigen's tridiagonal QL (tolerance-level)."""
    v0 = np.asarray(v0, dtype=np.float64).reshape(-1)
    dim = v0.shape[0]
    nrm0 = np.linalg.norm(v0)
    if nrm0 == 0.0:
        raise ValueError("lanczos: v0 must be nonzero")
    max_steps = min(max_iter, dim)
    basis = np.zeros((dim, max_steps + 1))
    basis[:, 0] = v0 / nrm0  # :36
    alpha, beta = [], []
    counters = [0, 0, 0, 0]
    history = []
    norm_est = 0.0
    ritz = ritz_vecs = None
    factorized = 0
    converged = False
    iterations = 0

    def factorize(m):  # :54-63
        t = np.diag(np.array(alpha[:m])) + np.diag(np.array(beta[: m - 1]), -1) + np.diag(np.array(beta[: m - 1]), 1)
        w, z = np.linalg.eigh(t)
        return w, z, m

    restart_counter = 0
    for m in range(1, max_steps + 1):
        w = matvec(basis[:, m - 1 : m]).reshape(-1)  # :67
        counters[0] += 1
        counters[1] += 1
        a = float(basis[:, m - 1] @ w)  # :68
        alpha.append(a)
        w = w - a * basis[:, m - 1]  # :70
        if m >= 2:
            w = w - beta[m - 2] * basis[:, m - 2]  # :71
        for _ in range(2):  # :73-76
            coeff = basis[:, :m].T @ w
            w = w - basis[:, :m] @ coeff
        counters[3] += 1
        b = float(np.linalg.norm(w))
        scale = max(abs(a), 1.0)
        if b <= 1e-13 * scale:  # :81-96
            r = np.array([symmetric_double(0x4C414E43 + restart_counter, i, m) for i in range(dim)])
            restart_counter += 1
            for _ in range(2):
                coeff = basis[:, :m].T @ r
                r = r - basis[:, :m] @ coeff
            rn = float(np.linalg.norm(r))
            if rn == 0.0:
                break
            basis[:, m] = r / rn
            beta.append(0.0)
        else:
            basis[:, m] = w / b
            beta.append(b)
        last = m == max_steps
        if not lanczos_checkpoint(m) and not last:  # :102-103
            continue
        ritz, ritz_vecs, factorized = factorize(m)
        norm_est = max(norm_est, abs(ritz[0]), abs(ritz[m - 1]))  # :106-107
        k = min(k_want, m)
        all_conv = k >= k_want
        for j in range(k):  # :111-118
            res = abs(beta[m - 1]) * abs(ritz_vecs[m - 1, j])
            relres = res / max(norm_est, 1e-300)
            history.append((m, j, relres, ritz[j]))
            if relres > tol:
                all_conv = False
        iterations = m
        if all_conv:
            converged = True
            break
    if factorized == 0:
        ritz, ritz_vecs, factorized = factorize(len(alpha))
    k = min(k_want, factorized)
    x = basis[:, :factorized] @ ritz_vecs[:, :k]  # :131-132
    return Report(ritz[:k].copy(), x, history, counters, converged, iterations, norm_est, [])


# ------------------------------------------------------- lobpcg.cpp helpers

def rayleigh_ritz(y_basis, hy, k_trial):
    """lobpcg.cpp:121-145: overlap check (1e-6), eig_sym of Y^T HY, leading
    k_trial eigenpairs."""
    m = y_basis.shape[1]
    if k_trial > m:
        raise ValueError("DimensionMismatch: rayleigh_ritz: k_trial exceeds basis width")
    overlap = block_inner(y_basis, y_basis)
    dev = np.abs(overlap - np.eye(m)).max()
    if dev > 1e-6:
        raise ValueError(f"IndefiniteGram: basis overlap deviates from identity by {dev}")
    evals, evecs = _eig_sym(block_inner(y_basis, hy))
    return evals[:k_trial].copy(), evecs[:, :k_trial].copy()


def residual_norms(h, x, theta, norm_est=None):
    """lobpcg.cpp:147-169."""
    r = spmm(h, x) - x * np.asarray(theta)[None, :]
    rn = column_norms(r)
    xn = column_norms(x)
    est = norm_est if norm_est is not None else 0.0
    if not est > 0.0:
        est = max([0.0] + [abs(t) for t in theta])
    return [rn[j] / max(est * xn[j], K_TINY_DIAG) for j in range(x.shape[1])]


# ---------------------------------------------------------------- guess.cpp

def pad_from_subspace(x1, dim):
    """guess.cpp:14-23."""
    out = np.zeros((dim, x1.shape[1]))
    out[: x1.shape[0]] = x1
    return out


def _widen_to(x, k_trial, seed):
    """guess.cpp:57-62."""
    if x.shape[1] >= k_trial:
        return x
    extra = random_block(x.shape[0], k_trial - x.shape[1], (int(mix64(np.uint64(seed))) + 1) & M64)
    extra = orthonormalize(extra, 1e-8, against=x)
    return np.hstack([x, extra])


def multilevel_guess(h, level_dims, k_want=8, k_trial=12, tol=1e-6, max_iter=500, seed=1):
    """guess.cpp:66-117 with the truncated problems taken as the leading
    blocks H[0:d, 0:d] (d in level_dims): random orthonormal start at the
    smallest level, unpreconditioned LOBPCG per level, zero-pad + widen_to
    into the next space. Returns (guess, [(dim, iterations, converged)])."""
    n = h.dim
    levels = len(level_dims) + 1
    if levels == 1:
        return orthonormalize(random_block(n, k_trial, seed)), []
    carried = None
    reports = []
    for level, d in enumerate(level_dims):
        width = min(k_trial, d)
        if level == 0:
            x0 = orthonormalize(random_block(d, width, seed))
        else:
            x0 = _widen_to(pad_from_subspace(carried, d), width, seed + level)
        if x0.shape[1] < k_want:
            raise ValueError("SubspaceCollapse: level guess lost too many columns")
        r = lobpcg_solve(h, x0, k_want, tol, max_iter,
                         matvec=lambda v, d=d: spmm(h, pad_from_subspace(v, n))[:d])
        carried = r.trial_vectors
        reports.append((d, r.iterations, r.converged))
    return _widen_to(pad_from_subspace(carried, n), k_trial, seed + levels), reports
