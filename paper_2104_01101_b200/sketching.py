"""Sketch operators (drop-in for src/sketching.py), executed by libskx.

Operators keep the reference's dataclass names and fields.  Table data lives
on the GPU; the numpy ``hash`` / ``signs`` arrays the reference exposes are
materialised lazily on attribute access.  Randomness follows the reference's
draw order exactly: TensorSketch coefficients are drawn on the host from the
numpy Generator (9 values per mode), while bulk draws (CountSketch tables,
leverage uniforms) are produced on the GPU from the Generator's Philox state
and the host Generator is advanced to where numpy would be.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import rng as rngmod
from .linalg import LeverageProfile, leverage_scores_dev, RankDeficientError

_MERSENNE = (1 << 31) - 1


def _torch():
    import torch
    return torch


def _dev(a):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).cuda()


def _unpack(tab):
    t = tab.cpu().numpy().astype(np.uint32)
    return (t & 0x7FFFFFFF).astype(np.int64), np.where(t >> 31, -1, 1).astype(np.int64)


def _pack(hash_, signs):
    torch = _torch()
    h = np.asarray(hash_, dtype=np.int64)
    s = np.asarray(signs)
    t = (h.astype(np.uint64) | np.where(s < 0, np.uint64(1 << 31), np.uint64(0))).astype(np.uint32)
    return torch.from_numpy(t.view(np.int32)).cuda()


# ============================================================ CountSketch
@dataclass
class CountSketchOp:
    """Bucket-and-sign projection: row i lands in bucket hash[i] (src/sketching.py:46-63)."""

    m: int
    hash: np.ndarray
    signs: np.ndarray

    @classmethod
    def build(cls, n, m, rng):
        rng = rngmod.make_rng(rng)
        h = rng.integers(0, m, size=n)
        s = 1 - 2 * rng.integers(0, 2, size=n)
        return cls(m, h, s)

    def apply(self, mat):
        """S @ mat for a dense (n, c) matrix -> (m, c), on the GPU."""
        torch = _torch()
        mat = _dev(mat)
        n, c = mat.shape
        tab = _pack(self.hash, self.signs)
        out = torch.empty((c, self.m), dtype=torch.float64, device="cuda")
        shp, sp_ = nat.host_i64([n, c])
        nat.call_ws("skx_rrf_stage1_dense", (nat.ptr(mat.contiguous()), 2, sp_, 1, nat.ptr(tab),
                                             self.m, nat.ptr(out)))
        return out.t().cpu().numpy()


# ============================================================ TensorSketch
class TensorSketchOp:
    """TensorSketch over a chain of modes (src/sketching.py:66-110): per-mode
    degree-3 polynomial bucket hash and degree-4 sign hash over GF(2^31-1),
    composed bucket = sum mod m, composed sign = product."""

    def __init__(self, m, extents, coeffs, tab=None):
        self.m = int(m)
        self.extents = tuple(int(s) for s in extents)
        self.coeffs = np.asarray(coeffs, dtype=np.int64).reshape(len(self.extents), 9)
        self.tab_off = np.concatenate([[0], np.cumsum(self.extents)[:-1]]).astype(np.int64)
        self._tab = tab
        self._modes = None

    @classmethod
    def build(cls, extents, m, rng):
        rng = rngmod.make_rng(rng)
        coeffs = []
        for _ in extents:
            ch = rng.integers(0, _MERSENNE, size=4, dtype=np.int64)
            cs = rng.integers(0, _MERSENNE, size=5, dtype=np.int64)
            coeffs.append(np.concatenate([ch, cs]))
        return cls(m, extents, np.array(coeffs).reshape(len(extents), 9))

    # device packed tables (sum(extents) uint32)
    @property
    def tab(self):
        torch = _torch()
        if self._tab is None:
            total = int(sum(self.extents))
            self._tab = torch.empty(max(total, 1), dtype=torch.int32, device="cuda")
            ext, ep = nat.host_i64(self.extents)
            cf, cp = nat.host_i64(self.coeffs.ravel())
            nat.call("skx_ts_tables", len(self.extents), ep, cp, self.m, nat.ptr(self._tab),
                     nat.stream())
        return self._tab

    @property
    def modes(self):
        if self._modes is None:
            mods = []
            t = self.tab
            for k, s in enumerate(self.extents):
                h, g = _unpack(t[self.tab_off[k]:self.tab_off[k] + s])
                mods.append(CountSketchOp(self.m, h, g))
            self._modes = mods
        return self._modes

    @property
    def n_rows(self):
        return int(np.prod(self.extents))

    def combined_hash(self, multi_idx):
        h = np.zeros(len(multi_idx[0]), dtype=np.int64)
        for k, idx in enumerate(multi_idx):
            h += self.modes[k].hash[idx]
        return h % self.m

    def combined_sign(self, multi_idx):
        s = np.ones(len(multi_idx[0]), dtype=np.int64)
        for k, idx in enumerate(multi_idx):
            s *= self.modes[k].signs[idx]
        return s

    def materialize(self):
        flat = np.arange(self.n_rows)
        multi = np.unravel_index(flat, self.extents)
        out = np.zeros((self.m, self.n_rows))
        out[self.combined_hash(multi), flat] = self.combined_sign(multi)
        return out

    def full_table(self):
        """Packed composed (bucket|sign) table over all prod(extents) rows."""
        torch = _torch()
        P = self.n_rows
        out = torch.empty(P, dtype=torch.int32, device="cuda")
        ext, ep = nat.host_i64(self.extents)
        off, op = nat.host_i64(self.tab_off)
        nat.call("skx_ts_combine", len(self.extents), ep, nat.ptr(self.tab), op, self.m, P,
                 nat.ptr(out), nat.stream())
        return out


def ts_kron_plan_dev(ts):
    """Per-operator Kronecker-sketch plan (bucket-sorted rows), cached on `ts`."""
    torch = _torch()
    plan = getattr(ts, "_kron_plan", None)
    if plan is None:
        lib = nat.load()
        ext, ep = nat.host_i64(ts.extents)
        off, op = nat.host_i64(ts.tab_off)
        pb = ctypes.c_size_t(0)
        wb = ctypes.c_size_t(0)
        st = nat.stream()
        nat.call("skx_ts_kron_plan", len(ts.extents), ep, nat.ptr(ts.tab), op, ts.m, None,
                 ctypes.byref(pb), None, ctypes.byref(wb), st)
        plan = torch.empty(max(pb.value, 256), dtype=torch.uint8, device="cuda")
        ws = nat.WS.get(wb.value, 0)
        pb2 = ctypes.c_size_t(plan.numel())
        wb2 = ctypes.c_size_t(ws.numel())
        nat.call("skx_ts_kron_plan", len(ts.extents), ep, nat.ptr(ts.tab), op, ts.m, nat.ptr(plan),
                 ctypes.byref(pb2), nat.ptr(ws), ctypes.byref(wb2), st)
        ts._kron_plan = plan
    return plan


def ts_kron_dev(ts, factors):
    """Z = S kron(factors) on device, returned as an (m, r) column-major view."""
    torch = _torch()
    plan = ts_kron_plan_dev(ts)
    fs = [f.contiguous() for f in factors]
    r = int(np.prod([f.shape[1] for f in fs]))
    zt = torch.empty((r, ts.m), dtype=torch.float64, device="cuda")
    ext, ep = nat.host_i64(ts.extents)
    rk, rp = nat.host_i64([f.shape[1] for f in fs])
    arr, fp = nat.host_ptrs(fs)
    nat.call_ws("skx_ts_kron_apply", (len(fs), ep, rp, fp, nat.ptr(plan), ts.m, nat.ptr(zt)))
    return zt.t()


def ts_apply_kron(ts, factors, method="auto"):
    """Apply a TensorSketch to the Kronecker chain of the factors
    (src/sketching.py:113-147).  `method` is accepted for interface parity: the
    device computes the circular convolutions exactly (no FFT), which agrees
    with both reference methods to rounding."""
    if len(factors) != len(ts.extents):
        raise ValueError("factor count does not match sketch mode count")
    for k, f in enumerate(factors):
        if np.shape(f)[0] != ts.extents[k]:
            raise ValueError(f"factor {k} has {np.shape(f)[0]} rows, sketch extent is {ts.extents[k]}")
    if method not in ("auto", "fft", "direct"):
        raise ValueError(f"unknown method {method!r}")
    z = ts_kron_dev(ts, [_dev(f) for f in factors])
    return z.cpu().numpy()


def ts_rhs_coo_dev(ts, colptr, rec, s_n, c1_mask=0xFFFFFFFF, packed_bb=-1):
    """Y^T (s_n x m) from a fibre-major COO layout (DeviceCoo.fibre); c1_mask /
    packed_bb describe a layout built with DeviceCoo.fibre(n, ts)."""
    torch = _torch()
    yt = torch.empty((s_n, ts.m), dtype=torch.float64, device="cuda")
    off, op = nat.host_i64(ts.tab_off)
    nat.call("skx_ts_rhs_coo", len(ts.extents), s_n, nat.ptr(colptr), nat.ptr(rec), nat.ptr(ts.tab),
             op, ts.m, ctypes.c_uint32(c1_mask), int(packed_bb), nat.ptr(yt), nat.stream())
    return yt


def ts_rhs_mode_dev(ts, d, n):
    """Y_n^T for mode n of a DeviceCoo, building (or reusing) its layout with
    ts's buckets folded in when possible."""
    colptr, rec = d.fibre(n, ts)
    return ts_rhs_coo_dev(ts, colptr, rec, d.shape[n], d.fibre_mask(n), d.fibre_packed_for(n, ts))


def _coo_from_pairs(rows, cols, data, shape):
    """DeviceCoo of a 2-D scipy-style (rows, cols, data) triple (lexsorted)."""
    from .tensors import DeviceCoo
    torch = _torch()
    order = np.lexsort((cols, rows))
    c = np.stack([np.asarray(rows)[order], np.asarray(cols)[order]]).astype(np.int32)
    return DeviceCoo(shape, torch.from_numpy(c).cuda(),
                     torch.from_numpy(np.ascontiguousarray(np.asarray(data)[order],
                                                           dtype=np.float64)).cuda())


# a mode-last copy of a dense tensor turns its sketches into the gather form
# (each other-mode index owns one contiguous s_n-vector): one permuting copy
# plus a bucket-sorted gather beat the shared-memory row form at large m
MODE_LAST_MAX_BYTES = 24 << 30


def mode_last_dev(t, mode):
    """(tensor, mode) with `mode` moved to the fastest-varying position when
    that is worth a copy (dense, not already last, small enough)."""
    torch = _torch()
    nd = t.dim()
    if mode == nd - 1 or t.numel() * 8 > MODE_LAST_MAX_BYTES:
        return t, mode
    a = int(np.prod(t.shape[:mode]))
    if a >= 65536:
        return t.movedim(mode, -1).contiguous(), nd - 1
    shape = tuple(t.shape)
    out = torch.empty(shape[:mode] + shape[mode + 1:] + (shape[mode],), dtype=torch.float64,
                      device="cuda")
    shp, sp_ = nat.host_i64(shape)
    nat.call("skx_mode_last", nat.ptr(t.contiguous()), nd, sp_, mode, nat.ptr(out), nat.stream())
    return out, nd - 1


def ts_rhs_dense_dev(ts, t, mode):
    """Y^T (s_n x m) for mode `mode` of a dense CUDA tensor (the other modes
    keep their order in the mode-last copy, so the tables apply unchanged)."""
    torch = _torch()
    t, mode = mode_last_dev(t, mode)
    shape = tuple(t.shape)
    yt = torch.empty((shape[mode], ts.m), dtype=torch.float64, device="cuda")
    shp, sp_ = nat.host_i64(shape)
    off, op = nat.host_i64(ts.tab_off)
    nat.call_ws("skx_ts_rhs_dense", (nat.ptr(t), len(shape), sp_, mode, nat.ptr(ts.tab), op, ts.m,
                                     nat.ptr(yt)))
    return yt


def ts_apply_rhs(ts, b, chunk=1 << 20):
    """Apply a TensorSketch to a tall right-hand side (src/sketching.py:150-175).
    b: (prod(extents), c) dense array or scipy sparse matrix."""
    import scipy.sparse as sp
    torch = _torch()
    n_rows = ts.n_rows
    if b.shape[0] != n_rows:
        raise ValueError(f"rhs has {b.shape[0]} rows, sketch expects {n_rows}")
    c = int(b.shape[1])
    if sp.issparse(b):
        coo = b.tocoo()
        if coo.nnz == 0:
            return np.zeros((ts.m, c))
        # as a (c, *extents) tensor: its mode-0 fibre layout is b's column-major order
        from .tensors import DeviceCoo
        multi = np.unravel_index(coo.row, ts.extents)
        cols = np.stack([coo.col] + list(multi)).astype(np.int64)
        order = np.lexsort(cols[::-1])
        d = DeviceCoo((c,) + tuple(ts.extents),
                      torch.from_numpy(np.ascontiguousarray(cols[:, order].astype(np.int32))).cuda(),
                      torch.from_numpy(np.ascontiguousarray(coo.data[order], dtype=np.float64)).cuda())
        return ts_rhs_mode_dev(ts, d, 0).t().cpu().numpy()
    bd = _dev(b).contiguous()
    full = ts.full_table()
    out = torch.empty((c, ts.m), dtype=torch.float64, device="cuda")
    shp, sp_ = nat.host_i64([n_rows, c])
    nat.call_ws("skx_rrf_stage1_dense", (nat.ptr(bd), 2, sp_, 1, nat.ptr(full), ts.m, nat.ptr(out)))
    return out.t().cpu().numpy()


# ============================================================ leverage sampling
@dataclass
class LevSamplerOp:
    """Row sampler over a Kronecker/Khatri-Rao chain (src/sketching.py:178-190)."""

    m: int
    extents: tuple
    profiles: list
    variant: str
    indices: np.ndarray
    weights: np.ndarray
    _dev: tuple = field(default=None, repr=False)

    def flat_indices(self):
        return np.ravel_multi_index(self.indices.T, self.extents)


def _lev_profile(f, check):
    """(scores, rank flag, p, cdf) of a factor, cached on the tensor: within a
    sweep each factor serves two sub-problems (mode n samples the factors of
    the other modes, and a factor is replaced -- not modified -- when its own
    mode is solved), so the second use needs no recomputation.  The cache is
    keyed by the check mode and the tensor's version counter."""
    torch = _torch()
    key = (bool(check), f._version)
    ent = getattr(f, "_skx_lev", None)
    if ent is not None and ent[0] == key:
        return ent[1]
    sc, bad = leverage_scores_dev(f, check=check)
    p = torch.empty_like(sc)
    cdf = torch.empty_like(sc)
    nat.call_ws("skx_lev_prepare", (nat.ptr(sc), int(sc.numel()), nat.ptr(p), nat.ptr(cdf)),
                slot=6)
    val = (sc, bad, p, cdf)
    f._skx_lev = (key, val)
    return val


def lev_sample_dev(factors, m, gen, check=True):
    """Random leverage sampler on device.  Computes every factor's scores
    first (QR rank check before any draw, as src/sketching.py:204-211), then
    m uniforms per factor from `gen`'s stream.  Returns (idx (m, k) int64,
    weights (m,), scores list, bad flag)."""
    torch = _torch()
    if m < 1:
        raise ValueError("sample count must be positive")
    scores, bads, ps, cdfs = [], [], [], []
    for f in factors:
        sc, bad, p, cdf = _lev_profile(f, check)
        scores.append(sc)
        bads.append(bad)
        ps.append(p)
        cdfs.append(cdf)
    k = len(factors)
    idx = torch.empty((m, k), dtype=torch.int64, device="cuda")
    w = torch.empty(m, dtype=torch.float64, device="cuda")
    c = rngmod.cursor(gen)
    ext, ep = nat.host_i64([f.shape[0] for f in factors])
    pa, pp = nat.host_ptrs(ps)
    ca, cp = nat.host_ptrs(cdfs)
    nat.call("skx_lev_sample", k, ep, pp, cp, m, ctypes.c_uint64(c.k0), ctypes.c_uint64(c.k1),
             ctypes.c_uint64(c.p), nat.ptr(idx), nat.ptr(w), nat.stream())
    rngmod.set_cursor(gen, c.p + k * m)
    bad = bads[0]
    for b in bads[1:]:
        bad = bad | b
    return idx, w, scores, bad


def top_m_products_dev(score_list, m):
    """Multi-indices (m, k) of the m largest products of one score per mode
    (src/sketching.py:224-259), in the reference's pop order: libskx sorts each
    list (descending, ties by index) and replays the best-first search on the
    device, so tied products (zero or repeated scores) come out exactly as the
    reference's heap pops them."""
    torch = _torch()
    lens = [int(x.numel()) for x in score_list]
    total = int(np.prod(lens))
    if m > total:
        raise ValueError(f"cannot select {m} rows from {total}")
    sc = [x.to(torch.float64).contiguous() for x in score_list]
    idx = torch.empty((m, len(sc)), dtype=torch.int64, device="cuda")
    ln, lp = nat.host_i64(lens)
    arr, sp_ = nat.host_ptrs(sc)
    nat.call_ws("skx_top_m_products", (len(sc), lp, sp_, m, nat.ptr(idx)), slot=6)
    return idx


def lev_det_dev(factors, m, check=True):
    """Deterministic leverage sampler (src/sketching.py:218-220): the m
    largest products of the factors' leverage scores, unit weights.  Returns
    (idx, weights, scores, bad) like lev_sample_dev."""
    torch = _torch()
    if m < 1:
        raise ValueError("sample count must be positive")
    scores, bads = [], []
    for f in factors:
        sc, bad = leverage_scores_dev(f, check=check)
        scores.append(sc)
        bads.append(bad)
    idx = top_m_products_dev(scores, m)
    bad = bads[0]
    for b in bads[1:]:
        bad = bad | b
    return idx, torch.ones(m, dtype=torch.float64, device="cuda"), scores, bad


def lev_build(factors, m, variant, rng):
    """Build a leverage-score row sampler (src/sketching.py:193-221)."""
    if m < 1:
        raise ValueError("sample count must be positive")
    if variant not in ("random", "deterministic"):
        raise ValueError(f"unknown variant {variant!r}")
    fs = [_dev(f) for f in factors]
    if variant == "deterministic":
        idx, w, scores, _ = lev_det_dev(fs, m)
    else:
        idx, w, scores, _ = lev_sample_dev(fs, m, rngmod.make_rng(rng))
    extents = tuple(f.shape[0] for f in fs)
    profiles = [LeverageProfile(s.cpu().numpy(), f.shape[1]) for s, f in zip(scores, fs)]
    return LevSamplerOp(m, extents, profiles, variant, idx.cpu().numpy(), w.cpu().numpy(),
                        _dev=(idx, w))


def kron_rows_dev(factors, idx, w):
    """Z (m, r) column-major view: weighted Kronecker rows."""
    torch = _torch()
    m = idx.shape[0]
    fs = [f.contiguous() for f in factors]
    r = int(np.prod([f.shape[1] for f in fs]))
    zt = torch.empty((r, m), dtype=torch.float64, device="cuda")
    rk, rp = nat.host_i64([f.shape[1] for f in fs])
    arr, fp = nat.host_ptrs(fs)
    nat.call("skx_kron_rows", len(fs), rp, fp, nat.ptr(idx), nat.ptr(w), m, nat.ptr(zt), nat.stream())
    return zt.t()


def gather_dense_dev(t, mode, idx, w):
    """Y (m, s_n) row-major: weighted mode-`mode` fibres of a dense tensor."""
    torch = _torch()
    shape = tuple(t.shape)
    m = idx.shape[0]
    y = torch.empty((m, shape[mode]), dtype=torch.float64, device="cuda")
    shp, sp_ = nat.host_i64(shape)
    nat.call("skx_gather_fibers_dense", nat.ptr(t), len(shape), sp_, mode, nat.ptr(idx), nat.ptr(w), m,
             nat.ptr(y), nat.stream())
    return y


def gather_coo_dev(keys, vals, ext_others, s_n, idx, w):
    """Sparse fibre gather -> (hit_off (m+1), hit_col, hit_val) on device."""
    torch = _torch()
    m = idx.shape[0]
    nnz = int(vals.numel())
    # count first to size the outputs exactly (one small D2H)
    hit_off = torch.empty(m + 1, dtype=torch.int64, device="cuda")
    cap = 0
    dummy_c = torch.empty(1, dtype=torch.int64, device="cuda")
    dummy_v = torch.empty(1, dtype=torch.float64, device="cuda")
    ext, ep = nat.host_i64(ext_others)
    nat.call_ws("skx_gather_fibers_coo", (len(ext_others), ep, s_n, nnz, nat.ptr(keys), nat.ptr(vals),
                                          nat.ptr(idx), nat.ptr(w), m, nat.ptr(hit_off),
                                          nat.ptr(dummy_c), nat.ptr(dummy_v), cap))
    total = int(hit_off[m].item())
    hit_col = torch.empty(max(total, 1), dtype=torch.int64, device="cuda")
    hit_val = torch.empty(max(total, 1), dtype=torch.float64, device="cuda")
    nat.call_ws("skx_gather_fibers_coo", (len(ext_others), ep, s_n, nnz, nat.ptr(keys), nat.ptr(vals),
                                          nat.ptr(idx), nat.ptr(w), m, nat.ptr(hit_off),
                                          nat.ptr(hit_col), nat.ptr(hit_val), total))
    return hit_off, hit_col[:total], hit_val[:total]


def gather_slices_dev(d, n, idx, w):
    """(hit_off, hit_col, hit_val) of the sampled mode-n fibres of an order-3
    DeviceCoo, n in (1, 2), from slices of its mode-0 layout (skx_slice_hits):
    same result as filter_fibers_dev + gather_coo_dev without a pass over
    every nonzero."""
    torch = _torch()
    colptr, rec = d.fibre(0)
    m = idx.shape[0]
    hit_off = torch.empty(m + 1, dtype=torch.int64, device="cuda")
    args = (n, d.shape[0], nat.ptr(colptr), nat.ptr(rec), ctypes.c_uint32(d.fibre_mask(0)),
            nat.ptr(idx.contiguous()), nat.ptr(w), m, nat.ptr(hit_off))
    nat.call_ws("skx_slice_hits", args + (None, None, 0), slot=9)
    total = int(hit_off[m].item())
    hit_col = torch.empty(max(total, 1), dtype=torch.int64, device="cuda")
    hit_val = torch.empty(max(total, 1), dtype=torch.float64, device="cuda")
    nat.call_ws("skx_slice_hits", args + (nat.ptr(hit_col), nat.ptr(hit_val), total), slot=9)
    return hit_off, hit_col[:total], hit_val[:total]


# Sync-free (speculative) forms of the sparse leverage gathers: fixed
# capacities, totals kept on the device, and an overflow flag the sweep checks
# with the rest of its deferred flags (a flagged sweep is replayed on the
# checked path, which sizes everything exactly).  Config 5: ~160 +- 13 hits
# per sub-problem against a capacity of 4096.
HITS_CAP = 1 << 12


def gather_slices_fixed_dev(d, n, idx, w, cap=None):
    """gather_slices_dev without the host read of the hit count: (hit_off
    (m + 1), hit_col (cap), hit_val (cap), overflow flag); entries past the
    device total are sentinel column s_n with value 0."""
    torch = _torch()
    cap = HITS_CAP if cap is None else cap
    colptr, rec = d.fibre(0)
    m = idx.shape[0]
    s_n = d.shape[n]
    hit_off = torch.empty(m + 1, dtype=torch.int64, device="cuda")
    args = (n, d.shape[0], nat.ptr(colptr), nat.ptr(rec), ctypes.c_uint32(d.fibre_mask(0)),
            nat.ptr(idx.contiguous()), nat.ptr(w), m, nat.ptr(hit_off))
    nat.call_ws("skx_slice_hits", args + (None, None, 0), slot=9)
    hit_col = torch.empty(cap, dtype=torch.int64, device="cuda")
    hit_val = torch.empty(cap, dtype=torch.float64, device="cuda")
    nat.call_ws("skx_slice_hits", args + (nat.ptr(hit_col), nat.ptr(hit_val), cap), slot=9)
    return _sanitize_hits(hit_off, hit_col, hit_val, m, s_n, cap)


def _sanitize_hits(hit_off, hit_col, hit_val, m, s_n, cap):
    torch = _torch()
    total = hit_off[m]
    valid = torch.arange(cap, device="cuda") < total
    hit_col = torch.where(valid, hit_col, torch.full_like(hit_col, s_n))
    hit_val = torch.where(valid, hit_val, torch.zeros_like(hit_val))
    return hit_off, hit_col, hit_val, total > cap


def filter_gather_fixed_dev(d, n, idx, w, cap=None):
    """filter_fibers_dev + gather_coo_dev without host syncs (any mode):
    fixed-capacity filter output sorted with sentinel padding, then the key
    gather into a fixed-capacity hit list.  Same (hit_off, hit_col, hit_val,
    overflow) contract as gather_slices_fixed_dev."""
    torch = _torch()
    cap = HITS_CAP if cap is None else cap
    others = [k for k in range(d.ndim) if k != n]
    flat = torch.zeros(idx.shape[0], dtype=torch.int64, device="cuda")
    for c, k in enumerate(others):
        flat = flat * d.shape[k] + idx[:, c]
    sflat, _ = torch.sort(flat)  # duplicates are harmless for the membership test
    shape_a, shape_p = nat.host_i64(d.shape)
    rows = [d.coords[k] for k in range(d.ndim)]
    ptr_a, ptr_p = nat.host_ptrs(rows)
    count = torch.zeros(1, dtype=torch.int64, device="cuda")
    keys = torch.full((cap,), np.iinfo(np.int64).max, dtype=torch.int64, device="cuda")
    vals = torch.zeros(cap, dtype=torch.float64, device="cuda")
    nat.call("skx_filter_fibers_coo", d.ndim, shape_p, n, d.nnz, ptr_p, nat.ptr(d.vals),
             nat.ptr(sflat), int(sflat.numel()), nat.ptr(keys), nat.ptr(vals), cap,
             nat.ptr(count), nat.stream())
    keys, order = torch.sort(keys, stable=True)
    vals = vals[order].contiguous()
    over_f = count[0] > cap
    m = idx.shape[0]
    s_n = d.shape[n]
    ext = [d.shape[k] for k in others]
    hit_off = torch.empty(m + 1, dtype=torch.int64, device="cuda")
    hit_col = torch.empty(cap, dtype=torch.int64, device="cuda")
    hit_val = torch.empty(cap, dtype=torch.float64, device="cuda")
    ep_a, ep = nat.host_i64(ext)
    nat.call_ws("skx_gather_fibers_coo", (len(ext), ep, s_n, cap, nat.ptr(keys), nat.ptr(vals),
                                          nat.ptr(idx), nat.ptr(w), m, nat.ptr(hit_off),
                                          nat.ptr(hit_col), nat.ptr(hit_val), cap))
    hit_off, hit_col, hit_val, over = _sanitize_hits(hit_off, hit_col, hit_val, m, s_n, cap)
    return hit_off, hit_col, hit_val, over | over_f


FILTER_CAP0 = 1 << 16


def filter_fibers_dev(d, n, idx):
    """(keys, vals) of the nonzeros of DeviceCoo d lying in the sampled mode-n
    fibres (other-mode multi-indices = rows of idx), sorted by key = flat_other *
    s_n + i_n: the slice of d.keys(n) that gather_coo_dev reads, found with one
    pass over the coordinates instead of a full sort (src/sketching.py:262-264)."""
    torch = _torch()
    others = [k for k in range(d.ndim) if k != n]
    flat = torch.zeros(idx.shape[0], dtype=torch.int64, device="cuda")
    for c, k in enumerate(others):
        flat = flat * d.shape[k] + idx[:, c]
    sflat = torch.unique(flat)
    shape_a, shape_p = nat.host_i64(d.shape)
    rows = [d.coords[k] for k in range(d.ndim)]
    ptr_a, ptr_p = nat.host_ptrs(rows)
    cap = FILTER_CAP0
    count = torch.zeros(1, dtype=torch.int64, device="cuda")
    while True:
        keys = torch.empty(cap, dtype=torch.int64, device="cuda")
        vals = torch.empty(cap, dtype=torch.float64, device="cuda")
        nat.call("skx_filter_fibers_coo", d.ndim, shape_p, n, d.nnz, ptr_p, nat.ptr(d.vals),
                 nat.ptr(sflat), int(sflat.numel()), nat.ptr(keys), nat.ptr(vals), cap,
                 nat.ptr(count), nat.stream())
        found = int(count.item())
        if found <= cap:
            break
        cap = found
    keys, order = torch.sort(keys[:found])
    return keys, vals[:found][order].contiguous()


def hits_to_dense(hit_off, hit_col, hit_val, m, s_n):
    torch = _torch()
    y = torch.zeros((m, s_n), dtype=torch.float64, device="cuda")
    counts = hit_off[1:] - hit_off[:-1]
    rows = torch.repeat_interleave(torch.arange(m, device="cuda"), counts)
    y[rows, hit_col] = hit_val
    return y


def lev_apply(sampler, factors, bt):
    """Sampled-and-rescaled (Z, Y) for a Kronecker chain (src/sketching.py:270-287)."""
    import scipy.sparse as sp
    torch = _torch()
    if tuple(np.shape(f)[0] for f in factors) != sampler.extents:
        raise ValueError("factors do not match the sampler's extents")
    if bt.shape[0] != int(np.prod(sampler.extents)):
        raise ValueError("rhs row count does not match the sampled chain")
    idx, w = sampler._dev if sampler._dev is not None else (
        torch.from_numpy(sampler.indices).cuda(), torch.from_numpy(sampler.weights).cuda())
    fs = [_dev(f) for f in factors]
    z = kron_rows_dev(fs, idx, w)
    flat = torch.zeros(idx.shape[0], dtype=torch.int64, device="cuda")
    for k, e in enumerate(sampler.extents):
        flat = flat * e + idx[:, k]
    P, s = bt.shape
    if sp.issparse(bt):
        c = bt.tocsr()
        c.sort_indices()
        rows = np.repeat(np.arange(P, dtype=np.int64), np.diff(c.indptr))
        keys = torch.from_numpy(rows * s + c.indices.astype(np.int64)).cuda()
        vals = torch.from_numpy(np.ascontiguousarray(c.data, dtype=np.float64)).cuda()
        off, col, val = gather_coo_dev(keys, vals, [P], s, flat.view(-1, 1).contiguous(), w)
        y = hits_to_dense(off, col, val, idx.shape[0], s)
    else:
        y = gather_dense_dev(_dev(bt).contiguous(), 1, flat.view(-1, 1).contiguous(), w)
    return z.cpu().numpy(), y.cpu().numpy()


def lev_apply_krp(sampler, factors, bt):
    """Khatri-Rao variant (src/sketching.py:290-301): Hadamard rows."""
    torch = _torch()
    if tuple(np.shape(f)[0] for f in factors) != sampler.extents:
        raise ValueError("factors do not match the sampler's extents")
    idx, w = sampler._dev if sampler._dev is not None else (
        torch.from_numpy(sampler.indices).cuda(), torch.from_numpy(sampler.weights).cuda())
    fs = [_dev(f) for f in factors]
    z = fs[0][idx[:, 0]].clone()
    for k in range(1, len(fs)):
        z *= fs[k][idx[:, k]]
    z = w[:, None] * z
    _, y = lev_apply(sampler, [np.zeros((e, 1)) for e in sampler.extents], bt)
    return z.cpu().numpy(), y


# ============================================================ composite (RRF)
class RrfTables:
    """Device description of CountSketch tables drawn as numpy's
    integers(0,k2,P) then integers(0,2,P) from a Philox stream: the start
    cursor, the sorted rejection offsets d_i and the sign run start."""

    def __init__(self, k0, k1, p0, has, pending, d, nd, sign_q0, k2, P):
        self.k0, self.k1, self.p0, self.has, self.pending = k0, k1, p0, has, pending
        self.d, self.nd, self.sign_q0, self.k2, self.P = d, nd, sign_q0, k2, P

    def args(self):
        return (ctypes.c_uint64(self.k0), ctypes.c_uint64(self.k1), ctypes.c_uint64(self.p0),
                ctypes.c_uint32(self.has), ctypes.c_uint32(self.pending),
                ctypes.c_uint64(self.sign_q0), nat.ptr(self.d), self.nd)


def _rej_cap(P, k2):
    thresh = (2 ** 32 - k2) % k2
    expect = P * thresh / 2 ** 32
    return int(max(1024, 4 * expect + 64 * np.sqrt(expect + 1) + 64))


class RrfScan:
    """A Lemire rejection scan over raw words [raw_lo, raw_hi) in flight.
    `pre` optionally holds a finish already enqueued behind it for a known
    start cursor (see plan_rrf_scans)."""

    def __init__(self, key, raw_lo, raw_hi, k2, cap, rej, count, stream, tag=0):
        self.key, self.raw_lo, self.raw_hi, self.k2, self.cap = key, raw_lo, raw_hi, k2, cap
        self.rej, self.count, self.stream, self.tag = rej, count, stream, tag
        self.pre = None
        self.comm = None


def launch_rrf_scan(key, raw_lo, raw_hi, k2, cap, stream=None, comm=None):
    """Enqueue the rejection scan of raw words [raw_lo, raw_hi) for bound k2.
    Compute-bound (one Philox block per 4 raw words); meant to run on a side
    stream, overlapping memory-bound work, before the exact start of the
    integers() call it serves is known.  With a multi-rank `comm`
    every rank scans its 1/world share; the finish gathers the lists."""
    torch = _torch()
    st = stream or torch.cuda.current_stream()
    lo, hi = comm.split(raw_lo, raw_hi) if comm is not None and comm.world > 1 else (raw_lo, raw_hi)
    with torch.cuda.stream(st):
        rej = torch.empty(cap, dtype=torch.int64, device="cuda")
        nat.call("skx_fill_u64max", nat.ptr(rej), cap, nat.stream())
        count = torch.zeros(1, dtype=torch.int64, device="cuda")
        if hi > lo:
            nat.call("skx_lemire_scan", ctypes.c_uint64(key[0]), ctypes.c_uint64(key[1]),
                     ctypes.c_uint64(lo), ctypes.c_uint64(hi), ctypes.c_uint32(k2), nat.ptr(rej),
                     cap, nat.ptr(count), nat.stream())
    sc = RrfScan(key, raw_lo, raw_hi, k2, cap, rej, count, st)
    sc.comm = comm if comm is not None and comm.world > 1 else None
    return sc


def _enqueue_finish(scan, c, P):
    """Enqueue skx_lemire_finish for a hash run starting at cursor `c` on the
    scan's stream, plus a pinned copy of (largest per-rank count, #rejections
    among the P hash draws) and an event marking both.  A rank-split scan
    first gathers every rank's list (the sort inside the finish merges them)."""
    torch = _torch()
    pend_raw = c.p - 1 if c.has else 0
    with torch.cuda.stream(scan.stream):
        rej, count, cap = scan.rej, scan.count, scan.cap
        if scan.comm is not None:
            counts = scan.comm.allgather(scan.count)
            rej = scan.comm.allgather(scan.rej)
            cap = int(rej.numel())
            count, cmax = counts.sum().view(1), counts.max().view(1)
        else:
            cmax = count
        d = torch.empty(cap, dtype=torch.int64, device="cuda")
        n_le = torch.zeros(1, dtype=torch.int64, device="cuda")
        nat.call_ws("skx_lemire_finish", (nat.ptr(rej), nat.ptr(count), cap,
                                          ctypes.c_uint64(c.p), ctypes.c_uint32(c.has),
                                          ctypes.c_uint64(pend_raw), ctypes.c_uint64(P),
                                          nat.ptr(d), nat.ptr(n_le)), slot=3 + 8 * scan.tag)
        host = torch.empty(2, dtype=torch.int64, pin_memory=True)
        host[0:1].copy_(cmax, non_blocking=True)
        host[1:2].copy_(n_le, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(scan.stream)
    return (c.p, c.has, P), d, host, ev


def finish_rrf_scan(scan, gen, P):
    """Resolve `scan` for the integers(0,k2,P); integers(0,2,P) call that `gen`
    makes next: build its d-array, read the rejection count (host waits on the
    scan's stream only, and only up to this scan's finish if it was enqueued
    with the scan), check the scanned range covered the call (else scan again
    exactly), and advance `gen` as numpy would."""
    torch = _torch()
    c = rngmod.cursor(gen)
    pend_raw = c.p - 1 if c.has else 0
    fin = scan.pre if scan.pre is not None and scan.pre[0] == (c.p, c.has, P) else None
    if fin is None:
        fin = _enqueue_finish(scan, c, P)
    _, d, host, ev = fin
    ev.synchronize()
    count, nrej = int(host[0]), int(host[1])  # count: largest per-rank list
    need_hi = c.p + (P + nrej - c.has + 1) // 2  # raw words the hash run reads
    covered = (count < scan.cap and c.p >= scan.raw_lo and need_hi <= scan.raw_hi
               and (not c.has or pend_raw >= scan.raw_lo))
    if not covered:  # prediction missed or too many rejections: exact rescan
        cap = max(scan.cap * 4, _rej_cap(P, scan.k2))
        lo = pend_raw if c.has else c.p
        exact = launch_rrf_scan(scan.key, lo, c.p + (P + cap) // 2 + 2, scan.k2, cap, scan.stream,
                                scan.comm)
        return finish_rrf_scan(exact, gen, P)
    cur = torch.cuda.current_stream()
    cur.wait_event(ev)
    d.record_stream(cur)
    tabs = RrfTables(c.k0, c.k1, c.p, c.has, c.pending, d, int(d.numel()), P + nrej, scan.k2, P)
    rngmod.advance_u32(gen, 2 * P + nrej)
    return tabs


def draw_rrf_tables(gen, P, k2, stream=None):
    """Reproduce rng.integers(0,k2,P); rng.integers(0,2,P) on device without
    materialising them; advances `gen` exactly as numpy would."""
    c = rngmod.cursor(gen)
    cap = _rej_cap(P, k2)
    lo = c.p - 1 if c.has else c.p
    scan = launch_rrf_scan((c.k0, c.k1), lo, c.p + (P + cap) // 2 + 2, k2, cap, stream)
    return finish_rrf_scan(scan, gen, P)


def plan_rrf_scans(gen, jobs, stream=None, comm=None):
    """Launch the scans of consecutive RRF table draws at once.  jobs =
    [(P, k2, n_gauss)] in draw order, where n_gauss normals follow each pair of
    integers() calls.  Later starts are bracketed (rejections < cap, ziggurat
    consumption in [n, 1.1 n + 256]); finish_rrf_scan verifies and rescans
    exactly if a bracket was missed."""
    c = rngmod.cursor(gen)
    key = (c.k0, c.k1)
    lo = c.p - 1 if c.has else c.p
    hi_start = c.p
    scans = []
    for i, (P, k2, n_gauss) in enumerate(jobs):
        cap = _rej_cap(P, k2)
        sc = launch_rrf_scan(key, lo, hi_start + (P + cap) // 2 + 2, k2, cap, stream, comm)
        sc.tag = i
        if i == 0 and sc.comm is None:
            # the first draw's cursor is known now: its finish goes right behind
            # its scan, so the host need not wait for the later scans.  (Not with
            # a multi-rank comm: its gather would sit in NCCL's queue ahead of the
            # right-hand-side all-reduces issued next and stall them behind the scan.)
            sc.pre = _enqueue_finish(sc, c, P)
        scans.append(sc)
        # the next call starts after the hash + sign draws and the normals; a
        # buffered high half left by the integers() pair sits *before* the
        # normals, so the next scan starts there (>= lo + P - 2)
        lo = lo + P - 2
        hi_start = hi_start + (2 * P + cap) // 2 + 2 + int(1.1 * n_gauss) + 256
    return scans


@dataclass
class CompositeSketchOp:
    """CountSketch stage followed by a Gaussian stage (src/sketching.py:304-324)."""

    k1: int
    k2: int
    stage: CountSketchOp
    gauss: np.ndarray

    @classmethod
    def build(cls, n_cols, k1, k2, rng):
        if k2 < k1:
            raise ValueError(f"intermediate width {k2} below target width {k1}")
        rng = rngmod.make_rng(rng)
        tabs = draw_rrf_tables(rng, n_cols, k2)
        tab = rrf_table_dev(tabs)
        h, s = _unpack(tab)
        gauss = rng.standard_normal((k2, k1)) / np.sqrt(k1)
        op = cls(k1, k2, CountSketchOp(k2, h, s), gauss)
        return op


def rrf_table_dev(tabs):
    torch = _torch()
    tab = torch.empty(max(tabs.P, 1), dtype=torch.int32, device="cuda")
    nat.call("skx_rrf_table", *tabs.args(), tabs.P, tabs.k2, nat.ptr(tab), nat.stream())
    return tab[:tabs.P]


def composite_apply(mat, op):
    """mat @ (countsketch stage) @ (gaussian stage) (src/sketching.py:327-341)."""
    import scipy.sparse as sp
    torch = _torch()
    if mat.shape[1] != len(op.stage.hash):
        raise ValueError(f"matrix has {mat.shape[1]} columns, sketch expects {len(op.stage.hash)}")
    s, P = mat.shape
    tab = _pack(op.stage.hash, op.stage.signs)
    st1 = torch.empty((s, op.k2), dtype=torch.float64, device="cuda")
    if sp.issparse(mat):
        c = mat.tocoo()
        colptr, rec = _coo_from_pairs(c.row, c.col, c.data, (s, P)).fibre(0)
        off = np.zeros(1, dtype=np.int64)
        nat.call("skx_ts_rhs_coo", 1, s, nat.ptr(colptr), nat.ptr(rec), nat.ptr(tab),
                 off.ctypes.data_as(ctypes.c_void_p), op.k2, ctypes.c_uint32(0xFFFFFFFF), -1,
                 nat.ptr(st1), nat.stream())
    else:
        md = _dev(mat).contiguous()
        shp, sp_ = nat.host_i64([s, P])
        nat.call_ws("skx_rrf_stage1_dense", (nat.ptr(md), 2, sp_, 0, nat.ptr(tab), op.k2, nat.ptr(st1)))
    return (st1 @ _dev(op.gauss)).cpu().numpy()
