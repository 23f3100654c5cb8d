"""CPU oracle for the sketched Tucker-ALS hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it.  The product path
(``paper_2104_01101_b200``) never imports anything under ``oracle/``.

It restates, in numpy/scipy, the algorithm of the reference package
``sketchals`` (``/root/reference/pkg/src/sketchals``; cited below as
``src/<file>:<line>``) for the path named by BASELINE.json's north star:
sketched Tucker-ALS (TensorSketch or leverage-score sampling), randomized
range-finder initialisation, and CP via Tucker compression.  The same numpy
primitives are used in the same order as the reference so that the oracle is
bit-identical to it in practice; tests/test_oracle_golden.py pins it against
fixtures produced by running the reference itself (tests/golden/make_golden.py).

Arithmetic third-party dependencies (not vendored under /root/reference):
numpy 2.3.5 (Philox/SeedSequence/Lemire/ziggurat, pocketfft, LAPACK via
scipy-openblas 0.3.30, ufunc.at) and scipy 1.18.1 (sparsetools,
solve_triangular).  The RNG stream part is independently restated in C in
oracle/rngref.c.

Data conventions (src/tensors.py:7-13): the mode-n unfolding is s_n x P_n with
the remaining modes ascending, earliest slowest; COO tensors hold lexsorted
int64 coordinates and float64 values.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse as sp

MERSENNE = (1 << 31) - 1


class RankDeficient(ValueError):
    """Restates src/linalg.py:16 (RankDeficientError subclasses ValueError)."""


# --------------------------------------------------------------------------
# random streams                                        src/rng.py:16-26
# --------------------------------------------------------------------------

def generator(seed):
    if isinstance(seed, np.random.Generator):
        return seed
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))


def streams(seed, n):
    return [np.random.Generator(np.random.Philox(child))
            for child in np.random.SeedSequence(seed).spawn(n)]


# --------------------------------------------------------------------------
# sparse tensor container                               src/tensors.py:26-98
# --------------------------------------------------------------------------

class Coo:
    """Lexsorted, duplicate-free COO tensor (src/tensors.py:35-60)."""

    def __init__(self, shape, coords, values, presorted=False):
        self.shape = tuple(int(s) for s in shape)
        c = np.asarray(coords, dtype=np.int64).reshape(-1, len(self.shape))
        v = np.asarray(values, dtype=np.float64).ravel()
        if c.shape[0] != v.shape[0]:
            raise ValueError("coords/values length mismatch")
        if c.size and ((c < 0).any() or (c >= np.asarray(self.shape)).any()):
            raise ValueError("coordinate out of range")
        if not presorted:
            perm = np.lexsort(c.T[::-1])
            c, v = c[perm], v[perm]
        if c.shape[0] > 1 and (np.diff(c, axis=0) == 0).all(axis=1).any():
            raise ValueError("duplicate coordinates")
        self.coords, self.values = c, v
        self._cache = {}

    @property
    def ndim(self):
        return len(self.shape)

    @property
    def nnz(self):
        return self.values.shape[0]

    def dense(self):
        out = np.zeros(self.shape)
        out[tuple(self.coords.T)] = self.values
        return out


def _rest(ndim, n):
    return [k for k in range(ndim) if k != n]


def unfold(t, n):
    """Mode-n unfolding (src/tensors.py:151-166, 179-194)."""
    if isinstance(t, Coo):
        return _coo_unfold(t, n, False)
    t = np.asarray(t)
    return np.moveaxis(t, n, 0).reshape(t.shape[n], -1)


def unfold_t(t, n):
    """Transposed unfolding T_(n)^T (src/tensors.py:169-176)."""
    if isinstance(t, Coo):
        return _coo_unfold(t, n, True)
    return unfold(t, n).T


def _coo_unfold(t, n, transpose):
    key = (n, transpose)
    if key not in t._cache:
        others = _rest(t.ndim, n)
        ext = [t.shape[k] for k in others]
        cols = (np.ravel_multi_index([t.coords[:, k] for k in others], ext)
                if t.nnz else np.zeros(0, dtype=np.int64))
        rows = t.coords[:, n]
        pn = int(np.prod(ext))
        if transpose:
            mat = sp.coo_matrix((t.values, (cols, rows)), shape=(pn, t.shape[n]))
        else:
            mat = sp.coo_matrix((t.values, (rows, cols)), shape=(t.shape[n], pn))
        t._cache[key] = mat.tocsr()
    return t._cache[key]


def fold(mat, n, shape):
    """Inverse unfolding (src/tensors.py:197-201)."""
    shape = tuple(shape)
    rest = [shape[k] for k in _rest(len(shape), n)]
    return np.moveaxis(np.asarray(mat).reshape([shape[n]] + rest), 0, n)


def mode_product(t, mat, n):
    """T x_n mat (src/tensors.py:204-214)."""
    t = np.asarray(t)
    shp = list(t.shape)
    shp[n] = mat.shape[0]
    return fold(mat @ unfold(t, n), n, shp)


def project_all(t, factors):
    """ttmc with skip=None (src/tensors.py:217-258)."""
    if isinstance(t, Coo):
        w = (unfold_t(t, 0) @ factors[0]).T
        out = w.reshape([factors[0].shape[1]] + list(t.shape[1:]))
        for k in range(1, t.ndim):
            out = mode_product(out, factors[k].T, k)
        return out
    out = np.asarray(t)
    for k in range(out.ndim):
        out = mode_product(out, factors[k].T, k)
    return out


def ttmc(t, factors, skip=None, chunk=1 << 16):
    """Tensor times matrix-chain (src/tensors.py:217-247): contract every mode
    m != skip with factors[m]^T.  Sparse skip-mode: per chunk of the nonzeros
    (mode-`skip` stable order), each nonzero's Kronecker row product
    (first other mode slowest), segment sums, added into the unfolded output
    (src/tensors.py:261-277)."""
    if skip is None:
        return project_all(t, factors)
    if not isinstance(t, Coo):
        out = np.asarray(t)
        for k in range(out.ndim):
            if k != skip:
                out = mode_product(out, factors[k].T, k)
        return out
    others = _rest(t.ndim, skip)
    cols = int(np.prod([factors[k].shape[1] for k in others]))
    out = np.zeros((t.shape[skip], cols))
    shp = [t.shape[k] if k == skip else factors[k].shape[1] for k in range(t.ndim)]
    if t.nnz == 0:
        return fold(out, skip, shp)
    order = np.argsort(t.coords[:, skip], kind="stable")
    rows = t.coords[order, skip]
    for lo in range(0, t.nnz, chunk):
        hi = min(lo + chunk, t.nnz)
        idx = order[lo:hi]
        contrib = t.values[idx][:, None]
        for k in others:
            fk = factors[k][t.coords[idx, k]]
            contrib = (contrib[:, :, None] * fk[:, None, :]).reshape(hi - lo, -1)
        seg = rows[lo:hi]
        starts = np.flatnonzero(np.r_[True, seg[1:] != seg[:-1]])
        out[seg[starts]] += np.add.reduceat(contrib, starts, axis=0)
    return fold(out, skip, shp)


def hosvd_init(t, ranks):
    """Leading eigenvectors of the mode Grams (src/tucker.py:112-126)."""
    out = []
    for n, r in enumerate(ranks):
        tn = unfold(t, n)
        gram = (tn @ tn.T).toarray() if sp.issparse(tn) else tn @ tn.T
        _, vecs = np.linalg.eigh(gram)
        out.append(vecs[:, ::-1][:, :r])
    return out


def hooi(t, ranks, max_sweeps=5, init="hosvd", seed=0, tol=0.0):
    """Exact Tucker-ALS (src/tucker.py:155-193): per mode the leading left
    singular vectors of the skip-mode TTMc unfolding; residual from the
    captured energy; core from the last mode's contraction."""
    import time

    shape = tuple(t.shape)
    nd = len(shape)
    rng = generator(seed)
    if init == "hosvd":
        A = hosvd_init(t, ranks)
    elif init == "random":
        A = [np.linalg.qr(rng.standard_normal((shape[n], ranks[n])))[0][:, :ranks[n]]
             for n in range(nd)]
    else:
        raise ValueError("unknown init")
    nt2 = norm_of(t) ** 2
    tr = Trace()
    core = None
    for _ in range(max_sweeps):
        t0 = time.perf_counter()
        y = None
        for n in range(nd):
            y = ttmc(t, A, skip=n)
            u, sv, _ = np.linalg.svd(unfold(y, n), full_matrices=False)
            A[n] = u[:, :ranks[n]]
            tr.residuals.append(np.sqrt(max(nt2 - float(np.sum(sv[:ranks[n]] ** 2)), 0.0)))
        core = mode_product(y, A[nd - 1].T, nd - 1)
        fit = 1.0 - np.sqrt(max(nt2 - float(np.vdot(core, core)), 0.0)) / np.sqrt(nt2)
        tr.wall_s.append(time.perf_counter() - t0)
        tr.fitness.append(float(fit))
        if len(tr.fitness) > 1 and abs(tr.fitness[-1] - tr.fitness[-2]) < tol:
            break
    return core, A, tr


def khatri_rao(mats):
    """src/tensors.py:288-301 (first matrix slowest)."""
    out = np.asarray(mats[0])
    for m in mats[1:]:
        out = (out[:, None, :] * np.asarray(m)[None, :, :]).reshape(-1, out.shape[1])
    return out


def mttkrp(t, factors, n):
    """src/tensors.py:307-336."""
    ndim = t.ndim if isinstance(t, Coo) else np.asarray(t).ndim
    others = _rest(ndim, n)
    if isinstance(t, Coo) or n == 0:
        return unfold(t, n) @ khatri_rao([factors[k] for k in others])
    letters = "abcdefghijkl"[:ndim]
    expr = letters + "," + ",".join(letters[k] + "z" for k in others) + "->" + letters[n] + "z"
    return np.einsum(expr, np.asarray(t), *[factors[k] for k in others], optimize=True)


def norm_of(t):
    if isinstance(t, Coo):
        return float(np.linalg.norm(t.values))
    return float(np.linalg.norm(np.asarray(t)))


def fitness_tucker(t, core, factors):
    """src/tensors.py:339-353 + 364-368."""
    nt = norm_of(t)
    if nt == 0.0:
        raise ValueError("zero-norm tensor")
    cross = float(np.vdot(project_all(t, factors), core))
    mod = float(np.vdot(core, core))
    return _fit_from(nt, cross, mod)


def fitness_cp(t, factors, weights):
    """src/tensors.py:354-361 + 364-368."""
    nt = norm_of(t)
    if nt == 0.0:
        raise ValueError("zero-norm tensor")
    scaled = factors[0] * weights
    m0 = mttkrp(t, factors, 0)
    cross = float(np.sum(scaled * m0))
    g = np.ones((factors[0].shape[1],) * 2)
    for a in factors[1:]:
        g *= a.T @ a
    mod = float(np.sum((scaled.T @ scaled) * g))
    return _fit_from(nt, cross, mod)


def _fit_from(nt, cross, mod):
    r2 = nt ** 2 - 2.0 * cross + mod
    if r2 < 0.0:
        r2 = 0.0
    return 1.0 - np.sqrt(r2) / nt


# --------------------------------------------------------------------------
# dense linear algebra                                  src/linalg.py:38-113
# --------------------------------------------------------------------------

def qr_checked(a):
    a = np.asarray(a, dtype=np.float64)
    q, r = np.linalg.qr(a)
    tol = 1e-12 * np.linalg.norm(a)
    d = np.abs(np.diag(r))
    if (d < tol).any():
        raise RankDeficient(f"rank-deficient: min |R_ii| {d.min():.3e} < {tol:.3e}")
    return q, r


def leverage(a):
    a = np.asarray(a)
    if a.shape[0] <= a.shape[1]:
        raise ValueError("leverage scores need a strictly tall matrix")
    q, _ = qr_checked(a)
    return np.einsum("ij,ij->i", q, q)


def rsvd_lrls(z, y, rank, rng, oversample=10):
    z = np.asarray(z, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    m, r = z.shape
    if m < r:
        raise ValueError("z must have at least as many rows as columns")
    if rank > min(r, y.shape[1]):
        raise ValueError("rank too large")
    qz, rz = qr_checked(z)
    xls = scipy.linalg.solve_triangular(rz, qz.T @ y, lower=False)
    w = min(rank + oversample, y.shape[1])
    g = rng.standard_normal((y.shape[1], w))
    q, _ = np.linalg.qr(xls @ g)
    d = q.T @ xls
    u, s, vt = np.linalg.svd(d, full_matrices=False)
    return q @ (u[:, :rank] * s[:rank]), vt.T[:, :rank]


# --------------------------------------------------------------------------
# sketch operators                                      src/sketching.py
# --------------------------------------------------------------------------

def _horner(coeffs, n):
    xs = np.arange(n, dtype=np.uint64)
    acc = np.full(n, coeffs[0], dtype=np.uint64)
    for c in coeffs[1:]:
        acc = (acc * xs + np.uint64(c)) % np.uint64(MERSENNE)
    return acc


def ts_tables(extents, m, rng):
    """Per-mode (bucket, sign) tables: degree-3 hash then degree-4 sign family,
    mode by mode (src/sketching.py:25-43, 80-86)."""
    hs, ss = [], []
    for s in extents:
        ch = rng.integers(0, MERSENNE, size=4, dtype=np.int64)
        hs.append((_horner(ch, s) % np.uint64(m)).astype(np.int64))
        cs = rng.integers(0, MERSENNE, size=5, dtype=np.int64)
        ss.append((1 - 2 * (_horner(cs, s) % np.uint64(2))).astype(np.int64))
    return hs, ss


def ts_bucket_sign(hs, ss, m, multi):
    h = np.zeros(len(multi[0]), dtype=np.int64)
    g = np.ones(len(multi[0]), dtype=np.int64)
    for k, ix in enumerate(multi):
        h += hs[k][ix]
        g *= ss[k][ix]
    return h % m, g


def countsketch(h, s, m, mat):
    """src/sketching.py:58-63."""
    mat = np.asarray(mat)
    out = np.zeros((m, mat.shape[1]))
    np.add.at(out, h, s[:, None] * mat)
    return out


def ts_rhs(hs, ss, extents, m, b, chunk=1 << 20):
    """src/sketching.py:150-175."""
    rows = int(np.prod(extents))
    if b.shape[0] != rows:
        raise ValueError("rhs row count mismatch")
    out = np.zeros((m, b.shape[1]))
    if sp.issparse(b):
        c = b.tocoo()
        h, g = ts_bucket_sign(hs, ss, m, np.unravel_index(c.row, extents))
        np.add.at(out, (h, c.col), g * c.data)
        return out
    b = np.asarray(b)
    for lo in range(0, rows, chunk):
        hi = min(rows, lo + chunk)
        h, g = ts_bucket_sign(hs, ss, m, np.unravel_index(np.arange(lo, hi), extents))
        np.add.at(out, h, g[:, None] * b[lo:hi])
    return out


def ts_kron(hs, ss, extents, m, factors, method="auto"):
    """src/sketching.py:113-147."""
    if len(factors) != len(extents):
        raise ValueError("factor count mismatch")
    for k, f in enumerate(factors):
        if f.shape[0] != extents[k]:
            raise ValueError("factor extent mismatch")
    cs = [countsketch(hs[k], ss[k], m, f) for k, f in enumerate(factors)]
    if len(cs) == 1:
        return cs[0]
    if method == "auto":
        method = "direct" if m < 64 else "fft"
    if method == "fft":
        acc = np.fft.fft(cs[0], axis=0)
        for nxt in cs[1:]:
            acc = (acc[:, :, None] * np.fft.fft(nxt, axis=0)[:, None, :]).reshape(m, -1)
        return np.fft.ifft(acc, axis=0).real
    if method == "direct":
        shift = (np.arange(m)[:, None] - np.arange(m)[None, :]) % m
        acc = cs[0]
        for nxt in cs[1:]:
            acc = np.einsum("jp,tjq->tpq", acc, nxt[shift]).reshape(m, -1)
        return acc
    raise ValueError(f"unknown method {method!r}")


def lev_sample(factors, m, rng):
    """Random leverage sampler (src/sketching.py:193-217): per-mode scores
    first (all QRs before any draw), then one choice() per mode."""
    if m < 1:
        raise ValueError("sample count must be positive")
    scores = [leverage(f) for f in factors]
    probs = []
    for sc in scores:
        q = np.maximum(sc, 0.0)
        probs.append(q / q.sum())
    idx = np.stack([rng.choice(len(p), size=m, p=p) for p in probs], axis=1)
    pp = np.ones(m)
    for k, p in enumerate(probs):
        pp *= p[idx[:, k]]
    return idx, 1.0 / np.sqrt(m * pp), scores


def top_m_products(score_lists, m):
    """Best-first frontier search over score-sorted lists (src/sketching.py:
    224-259): the m largest products, ties by lexicographic original
    multi-index, in pop order."""
    import heapq

    total = int(np.prod([len(x) for x in score_lists]))
    if m > total:
        raise ValueError(f"cannot select {m} rows from {total}")
    orders, srt = [], []
    for x in score_lists:
        o = np.lexsort((np.arange(len(x)), -np.asarray(x)))
        orders.append(o)
        srt.append(np.asarray(x)[o])
    start = tuple(0 for _ in score_lists)
    first = tuple(int(orders[k][0]) for k in range(len(score_lists)))
    heap = [(-float(np.prod([x[0] for x in srt])), first, start)]
    seen = {start}
    out = []
    while len(out) < m:
        _, orig, pos = heapq.heappop(heap)
        out.append(orig)
        for k in range(len(pos)):
            if pos[k] + 1 >= len(srt[k]):
                continue
            nxt = pos[:k] + (pos[k] + 1,) + pos[k + 1:]
            if nxt in seen:
                continue
            seen.add(nxt)
            prod = float(np.prod([srt[j][nxt[j]] for j in range(len(nxt))]))
            norig = tuple(int(orders[j][nxt[j]]) for j in range(len(nxt)))
            heapq.heappush(heap, (-prod, norig, nxt))
    return np.array(out, dtype=np.int64)


def lev_det(factors, m):
    """Deterministic leverage sampler (src/sketching.py:218-220)."""
    if m < 1:
        raise ValueError("sample count must be positive")
    scores = [leverage(f) for f in factors]
    return top_m_products(scores, m), np.ones(m), scores


def lev_rows(idx, w, extents, factors, bt):
    """src/sketching.py:262-287: weighted Kronecker rows and RHS rows."""
    m = idx.shape[0]
    z = factors[0][idx[:, 0]]
    for k in range(1, len(factors)):
        rows = factors[k][idx[:, k]]
        z = (z[:, :, None] * rows[:, None, :]).reshape(m, -1)
    z = w[:, None] * z
    flat = np.ravel_multi_index(idx.T, extents)
    if sp.issparse(bt):
        y = np.asarray(bt.tocsr()[flat].todense())
    else:
        y = np.asarray(bt)[flat]
    return z, w[:, None] * y


def rrf_tables(ncols, k1, k2, rng):
    """src/sketching.py:54-56, 319-324."""
    if k2 < k1:
        raise ValueError("k2 < k1")
    h = rng.integers(0, k2, size=ncols)
    s = 1 - 2 * rng.integers(0, 2, size=ncols)
    g = rng.standard_normal((k2, k1)) / np.sqrt(k1)
    return h, s, g


def rrf_apply(mat, h, s, g, k2):
    """src/sketching.py:327-341."""
    tm = sp.csr_matrix((s, (np.arange(mat.shape[1]), h)), shape=(mat.shape[1], k2))
    if sp.issparse(mat):
        st1 = np.asarray((mat @ tm).todense())
    else:
        st1 = (tm.T @ np.asarray(mat).T).T
    return st1 @ g


def init_rrf(tn, rank, width, rng):
    """src/tucker.py:129-144."""
    if width < rank:
        raise ValueError("width below rank")
    k2 = rank * rank + width
    h, s, g = rrf_tables(tn.shape[1], width, k2, rng)
    b = rrf_apply(tn, h, s, g, k2)
    u, _, _ = np.linalg.svd(b, full_matrices=False)
    if u.shape[1] < rank:
        raise ValueError("sketch too narrow")
    return u[:, :rank]


# --------------------------------------------------------------------------
# drivers                                       src/tucker.py:57-89, 216-300
# --------------------------------------------------------------------------

def resolve_m(ranks, sketch_size=None, sketch_factor=None):
    if sketch_size is not None:
        return int(sketch_size)
    if sketch_factor is not None:
        return int(math.ceil(sketch_factor * max(ranks) ** 2))
    raise ValueError("need sketch_size or sketch_factor")


def resolve_k1(ranks, rank, rrf_width=None, sketch_size=None, sketch_factor=None):
    if rrf_width is not None:
        return max(int(rrf_width), rank)
    if sketch_factor is not None:
        kf = sketch_factor
    elif sketch_size is not None:
        kf = sketch_size / max(ranks) ** 2
    else:
        kf = 4.0
    return max(rank, int(math.ceil(math.sqrt(kf) * rank)))


@dataclass
class Trace:
    fitness: list = field(default_factory=list)
    residuals: list = field(default_factory=list)
    wall_s: list = field(default_factory=list)
    stage_split: int | None = None


def sketched_tucker(t, ranks, sketch, max_sweeps=5, sketch_size=None,
                    sketch_factor=None, init=None, rrf_width=None, seed=0, tol=0.0):
    """Alg. 4 of the paper as implemented at src/tucker.py:216-300."""
    import time

    if sketch not in ("tensorsketch", "leverage-random", "leverage-deterministic"):
        raise ValueError("oracle covers tensorsketch and leverage sampling")
    shape = tuple(t.shape)
    nd = len(shape)
    ranks = tuple(int(r) for r in ranks)
    for s, r in zip(shape, ranks):
        if not 1 <= r <= s:
            raise ValueError("invalid rank")
    m = resolve_m(ranks, sketch_size, sketch_factor)
    for j in range(nd):
        need = int(np.prod([ranks[k] for k in _rest(nd, j)]))
        if m < need:
            raise ValueError("sketch size below system width")
    r_init, r_sketch, r_solve = streams(seed, 3)
    init = init or "rrf"
    A = [None] * nd
    for n in range(1, nd):
        if init == "rrf":
            k1 = resolve_k1(ranks, ranks[n], rrf_width, sketch_size, sketch_factor)
            A[n] = init_rrf(unfold(t, n), ranks[n], k1, r_init)
        elif init == "random":
            A[n] = np.linalg.qr(r_init.standard_normal((shape[n], ranks[n])))[0][:, :ranks[n]]
        else:
            raise ValueError("unknown init")
    bts = [unfold_t(t, n) for n in range(nd)]
    use_ts = sketch == "tensorsketch"
    tabs = [None] * nd
    rhs = [None] * nd

    def prep(n):
        ext = tuple(shape[k] for k in _rest(nd, n))
        tabs[n] = ts_tables(ext, m, r_sketch)
        rhs[n] = ts_rhs(tabs[n][0], tabs[n][1], ext, m, bts[n])

    if use_ts:
        for n in range(nd):
            prep(n)

    def solve(n, redraw):
        others = [A[k] for k in _rest(nd, n)]
        ext = tuple(shape[k] for k in _rest(nd, n))
        if use_ts:
            if redraw:
                prep(n)
            z = ts_kron(tabs[n][0], tabs[n][1], ext, m, others)
            y = rhs[n]
        else:
            if sketch == "leverage-deterministic":
                idx, w, _ = lev_det(others, m)
            else:
                idx, w, _ = lev_sample(others, m, r_sketch)
            z, y = lev_rows(idx, w, ext, others, bts[n])
        ct, a = rsvd_lrls(z, y, ranks[n], r_solve)
        res = float(np.linalg.norm((z @ ct) @ a.T - y))
        return ct, a, res

    tr = Trace()
    ct = None
    for _ in range(max_sweeps):
        t0 = time.perf_counter()
        for n in range(nd):
            try:
                c, a, res = solve(n, False)
            except RankDeficient:
                c, a, res = solve(n, True)
            A[n] = a
            ct = c
            tr.residuals.append(res)
        core = fold(ct.T, nd - 1, ranks)
        tr.wall_s.append(time.perf_counter() - t0)
        tr.fitness.append(float(fitness_tucker(t, core, A)))
        if len(tr.fitness) > 1 and abs(tr.fitness[-1] - tr.fitness[-2]) < tol:
            break
    return core, A, tr


def _unit_columns(a):
    nrm = np.linalg.norm(a, axis=0)
    return a / np.where(nrm > 0, nrm, 1.0), nrm


def cp_on_core(core, rank, sweeps=25, seed=0):
    """Exact CP-ALS on a small dense core with hosvd-of-core init
    (src/cp.py:119-174 with on_core=True; src/tucker.py:112-126)."""
    import time

    core = np.asarray(core)
    nd = core.ndim
    nt = norm_of(core)
    if nt == 0.0:
        raise ValueError("zero-norm tensor")
    nt2 = nt ** 2
    A = []
    for n in range(nd):
        tn = unfold(core, n)
        _, vec = np.linalg.eigh(tn @ tn.T)
        A.append(np.asarray(vec[:, ::-1][:, :min(rank, core.shape[n])], dtype=np.float64))
    w = np.ones(rank)
    grams = [a.T @ a for a in A]
    tr = Trace()
    for _ in range(sweeps):
        t0 = time.perf_counter()
        for n in range(nd):
            go = np.ones((rank, rank))
            for k in range(nd):
                if k != n:
                    go *= grams[k]
            mm = mttkrp(core, A, n)
            sc = mm @ np.linalg.pinv(go, rcond=1e-12)
            cross = float(np.sum(sc * mm))
            mod = float(np.sum((sc.T @ sc) * go))
            tr.residuals.append(np.sqrt(max(nt2 - 2.0 * cross + mod, 0.0)))
            A[n], w = _unit_columns(sc)
            grams[n] = A[n].T @ A[n]
        fit = fitness_cp(core, [a.copy() for a in A], w.copy())
        tr.wall_s.append(time.perf_counter() - t0)
        tr.fitness.append(float(fit))
    return A, w, tr


def sketched_cp(t, rank, max_sweeps=30, sketch_size=None, sketch_factor=None, seed=0,
                init="rrf"):
    """Leverage-sampled CP-ALS on the full tensor (src/cp.py:110-116,
    119-174 sketched branch): RRF (or random) init of every mode from the
    first of two seed streams; per mode a random leverage sample of the
    Khatri-Rao rows (second stream), weighted Hadamard rows and fibres,
    least squares (numpy lstsq), column normalisation; fitness per sweep and
    residual (1 - fit) ||T||."""
    import time

    shape = tuple(t.shape)
    nd = len(shape)
    nt = norm_of(t)
    r_init, r_sketch = streams(seed, 2)
    width = None
    if sketch_factor is not None:
        width = max(rank, int(math.ceil(math.sqrt(sketch_factor) * rank)))
    elif sketch_size is not None:
        width = max(rank, int(math.ceil(math.sqrt(sketch_size / rank ** 2) * rank)))
    if init == "random":
        A = [r_init.uniform(size=(shape[n], rank)) for n in range(nd)]
    else:
        w0 = width or max(rank + 8, 2 * rank)
        A = [init_rrf(unfold(t, n), rank, min(w0, shape[n]), r_init) if shape[n] > rank
             else np.linalg.qr(r_init.standard_normal((shape[n], rank)))[0] for n in range(nd)]
    A = [np.asarray(a, dtype=np.float64) for a in A]
    w = np.ones(rank)
    m = int(sketch_size) if sketch_size is not None else int(math.ceil(sketch_factor * rank ** 2))
    bts = [unfold_t(t, n) for n in range(nd)]
    tr = Trace()
    for _ in range(max_sweeps):
        t0 = time.perf_counter()
        for n in range(nd):
            others = [A[k] for k in _rest(nd, n)]
            ext = tuple(shape[k] for k in _rest(nd, n))
            idx, wt, _ = lev_sample(others, m, r_sketch)
            z = others[0][idx[:, 0]].copy()
            for k in range(1, len(others)):
                z *= others[k][idx[:, k]]
            z = wt[:, None] * z
            flat = np.ravel_multi_index(idx.T, ext)
            bt = bts[n]
            y = np.asarray(bt.tocsr()[flat].todense()) if sp.issparse(bt) else np.asarray(bt)[flat]
            y = wt[:, None] * y
            sol, *_ = np.linalg.lstsq(z, y, rcond=None)
            A[n], w = _unit_columns(sol.T)
        fit = fitness_cp(t, [a.copy() for a in A], w.copy())
        tr.residuals.append((1.0 - fit) * nt)
        tr.wall_s.append(time.perf_counter() - t0)
        tr.fitness.append(float(fit))
    return A, w, tr


def cp_via_tucker(t, rank, tucker_sweeps=5, cp_sweeps=None, sketch_size=None,
                  sketch_factor=None, seed=0, tucker_rank=None, sketch="leverage-random"):
    """Alg. 6 as at src/cp.py:177-224 (sketch=None: the exact-HOOI compression
    stage with HOSVD init, src/cp.py:195-205).  tucker_rank=None ties the
    Tucker ranks to the CP rank exactly like the reference; config 5 of
    BASELINE.json sets tucker_rank=20 with rank=10."""
    shape = tuple(t.shape)
    nd = len(shape)
    if any(rank > s for s in shape):
        raise ValueError("rank exceeds a tensor extent")
    s_t, s_c = (c.generate_state(1)[0] for c in np.random.SeedSequence(seed).spawn(2))
    tr_rank = rank if tucker_rank is None else tucker_rank
    if sketch:
        core, B, ttr = sketched_tucker(t, (tr_rank,) * nd, "leverage-random",
                                       max_sweeps=tucker_sweeps, sketch_size=sketch_size,
                                       sketch_factor=sketch_factor, init="rrf", seed=int(s_t))
    else:
        core, B, ttr = hooi(t, (tr_rank,) * nd, max_sweeps=tucker_sweeps, init="hosvd",
                            seed=int(s_t))
    A, w, ctr = cp_on_core(core, rank, sweeps=25 if cp_sweeps is None else cp_sweeps,
                           seed=int(s_c))
    fac = [b @ a for b, a in zip(B, A)]
    weights = w.copy()
    out = []
    for a in fac:
        u, nrm = _unit_columns(a)
        out.append(u)
        weights *= nrm
    tr = Trace(fitness=list(ttr.fitness) + [fitness_cp(t, out, weights)],
               residuals=list(ctr.residuals),
               wall_s=list(ttr.wall_s) + [sum(ctr.wall_s)],
               stage_split=len(ttr.fitness))
    return out, weights, tr, (core, B)


def _vec_col(t):
    """vec(T) as a (prod shape, 1) column, sparse-aware (src/tucker.py:205-213)."""
    if isinstance(t, Coo):
        flat = np.ravel_multi_index(t.coords.T, t.shape)
        return sp.csr_matrix((t.values, (flat, np.zeros(len(flat), dtype=np.int64))),
                             shape=(int(np.prod(t.shape)), 1))
    return np.asarray(t).reshape(-1, 1)


def ref_tucker_ts(t, ranks, max_sweeps=5, sketch_size=None, sketch_factor=None, init=None,
                  rrf_width=None, seed=0, tol=0.0):
    """One-variable-at-a-time TensorSketch baseline (src/tucker.py:303-364):
    RRF init of every mode, per-mode operators + right-hand sides and one
    all-mode operator for the core, drawn once; per sweep N unconstrained
    factor solves (core fixed, QR re-orthonormalised) and one core solve."""
    import time

    shape = tuple(t.shape)
    nd = len(shape)
    ranks = tuple(int(r) for r in ranks)
    m = resolve_m(ranks, sketch_size, sketch_factor)
    r_init, r_sketch = streams(seed, 2)
    init = init or "rrf"
    A = []
    for n in range(nd):
        if init == "rrf":
            k1 = resolve_k1(ranks, ranks[n], rrf_width, sketch_size, sketch_factor)
            A.append(init_rrf(unfold(t, n), ranks[n], k1, r_init))
        else:
            A.append(np.linalg.qr(r_init.standard_normal((shape[n], ranks[n])))[0][:, :ranks[n]])
    tabs, rhs = [], []
    for n in range(nd):
        ext = tuple(shape[k] for k in _rest(nd, n))
        tb = ts_tables(ext, m, r_sketch)
        tabs.append((tb, ext))
        rhs.append(ts_rhs(tb[0], tb[1], ext, m, unfold_t(t, n)))
    ctab = ts_tables(shape, m, r_sketch)
    crhs = ts_rhs(ctab[0], ctab[1], shape, m, _vec_col(t))

    def core_solve():
        z = ts_kron(ctab[0], ctab[1], shape, m, A)
        sol = np.linalg.lstsq(z, crhs, rcond=None)[0]
        return sol.reshape(ranks), float(np.linalg.norm(z @ sol - crhs))

    core, _ = core_solve()
    tr = Trace()
    for _ in range(max_sweeps):
        t0 = time.perf_counter()
        for n in range(nd):
            (hs, ss), ext = tabs[n]
            z = ts_kron(hs, ss, ext, m, [A[k] for k in _rest(nd, n)]) @ unfold(core, n).T
            sol = np.linalg.lstsq(z, rhs[n], rcond=None)[0]
            tr.residuals.append(float(np.linalg.norm(z @ sol - rhs[n])))
            A[n] = np.linalg.qr(sol.T)[0][:, :ranks[n]]
        core, cres = core_solve()
        tr.residuals.append(cres)
        tr.wall_s.append(time.perf_counter() - t0)
        tr.fitness.append(float(fitness_tucker(t, core, A)))
        if len(tr.fitness) > 1 and abs(tr.fitness[-1] - tr.fitness[-2]) < tol:
            break
    return core, A, tr
