"""Dense factorisations, leverage scores and the randomized rank-constrained
least-squares solver (drop-in for src/linalg.py), computed on the GPU.

QR/SVD/TRSM/GEMM run on-device through cuSOLVER/cuBLAS (torch.linalg with the
cuSOLVER backend); the Gaussian test matrix of rsvd_lrls is drawn on-device by
libskx's bit-exact numpy ziggurat; the sub-problem residual is a fused libskx
pass over Y.  numpy in / numpy out at the API boundary, torch CUDA tensors in
the drivers (the *_dev functions).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from . import rng as rngmod


class RankDeficientError(ValueError):
    """A matrix that must have full column rank numerically does not."""


@dataclass
class SvdResult:
    u: np.ndarray
    singular_values: np.ndarray
    v: np.ndarray

    def reconstruct(self):
        return (self.u * self.singular_values) @ self.v.T


@dataclass
class LeverageProfile:
    """Squared row norms of an orthonormal column basis; they sum to the rank."""

    scores: np.ndarray
    rank: int


_BACKEND_SET = False


def _torch():
    global _BACKEND_SET
    import torch
    if not _BACKEND_SET:
        # cuSOLVER for every factorisation (MAGMA's hybrid paths would run on the host)
        torch.backends.cuda.preferred_linalg_library("cusolver")
        _BACKEND_SET = True
    return torch


def _dev(a):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).cuda()


def _np(t):
    return t.detach().contiguous().cpu().numpy()


# ------------------------------------------------------------------ QR
def qr_flag_dev(mat):
    """Reduced QR on device plus the reference's rank test as a device bool:
    any |R_ii| < 1e-12 * ||mat||_F (src/linalg.py:38-52)."""
    torch = _torch()
    q, r = torch.linalg.qr(mat, mode="reduced")
    tol = 1e-12 * torch.linalg.vector_norm(mat)
    bad = (torch.diagonal(r).abs() < tol).any()
    return q, r, bad


def reduced_qr_dev(mat):
    q, r, bad = qr_flag_dev(mat)
    if bool(bad.item()):
        d = _torch().diagonal(r).abs()
        raise RankDeficientError(
            f"rank-deficient input: min |R_ii| = {float(d.min()):.3e} < "
            f"{1e-12 * float(_torch().linalg.vector_norm(mat)):.3e}")
    return q, r


def reduced_qr(mat):
    q, r = reduced_qr_dev(_dev(mat))
    return _np(q), _np(r)


# ------------------------------------------------------------------ SVD
def thin_svd_dev(mat):
    """Thin SVD (k = min(m, n)), singular values non-increasing.  Wide or tall
    inputs are first reduced by a QR so cuSOLVER only sees a k x k problem."""
    torch = _torch()
    m, n = mat.shape
    if m >= n:
        q, r = torch.linalg.qr(mat, mode="reduced")
        u, s, vh = torch.linalg.svd(r, full_matrices=False)
        return q @ u, s, vh.transpose(0, 1)
    q, r = torch.linalg.qr(mat.transpose(0, 1), mode="reduced")  # mat^T = q r
    u, s, vh = torch.linalg.svd(r.transpose(0, 1), full_matrices=False)  # r^T = u s vh
    return u, s, q @ vh.transpose(0, 1)


def tsqr_r_dev(a):
    """R factor (w x w) of a tall-skinny CUDA matrix view (w <= 96) by libskx TSQR."""
    torch = _torch()
    n, w = a.shape
    r = torch.empty((w, w), dtype=torch.float64, device="cuda")
    nat.call_ws("skx_tsqr_r", (nat.ptr(a), n, w, int(a.stride(0)), int(a.stride(1)), nat.ptr(r)),
                slot=2)
    return r


def chol_upper_dev(g):
    """Upper Cholesky factor R (R^T R = g) of a small SPD matrix (n <= 128), one
    CTA; returns (R, info) with info a device int (0 = success)."""
    torch = _torch()
    n = g.shape[0]
    r = torch.empty((n, n), dtype=torch.float64, device="cuda")
    info = torch.empty(1, dtype=torch.int32, device="cuda")
    nat.call("skx_chol_upper", nat.ptr(g.contiguous()), n, nat.ptr(r), nat.ptr(info), nat.stream())
    return r, info


def chol_inv_upper_dev(g):
    """Upper Cholesky factor R of an SPD n x n Gram (n <= 512) and R^-1, one
    libskx CTA (blocked, FP64 tensor cores); returns (R, R^-1, info) with info
    a device int (0 = success)."""
    torch = _torch()
    n = g.shape[0]
    r = torch.empty((n, n), dtype=torch.float64, device="cuda")
    rinv = torch.empty((n, n), dtype=torch.float64, device="cuda")
    info = torch.empty(1, dtype=torch.int32, device="cuda")
    nat.call("skx_chol_inv_upper", nat.ptr(g.contiguous()), n, nat.ptr(r), nat.ptr(rinv),
             nat.ptr(info), nat.stream())
    return r, rinv, info


def house_q_dev(c):
    """Thin Householder Q (LAPACK sign convention) of a tall r x w matrix with
    w <= 32, one libskx CTA."""
    torch = _torch()
    r, w = c.shape
    q = torch.empty((r, w), dtype=torch.float64, device="cuda")
    nat.call("skx_house_q", nat.ptr(c.contiguous()), r, w, nat.ptr(q), nat.stream())
    return q


CHOL_INV_MAX = 512
HOUSE_Q_SMEM = 227 * 1024


def jacobi_svd_dev(a):
    """SVD of a small square matrix (n <= 112) by one-sided Jacobi in one CTA:
    a = U diag(s) V^T, s descending."""
    torch = _torch()
    n = a.shape[0]
    u = torch.empty((n, n), dtype=torch.float64, device="cuda")
    v = torch.empty((n, n), dtype=torch.float64, device="cuda")
    s = torch.empty(n, dtype=torch.float64, device="cuda")
    nat.call("skx_jacobi_svd", nat.ptr(a), n, int(a.stride(0)), int(a.stride(1)), nat.ptr(u),
             nat.ptr(s), nat.ptr(v), nat.stream())
    return u, s, v


def _small_svd(r):
    """(u, s, vh) of a small square R: libskx Jacobi when n <= 112."""
    torch = _torch()
    if r.shape[0] <= 112:
        u, s, v = jacobi_svd_dev(r)
        return u, s, v.transpose(0, 1)
    return torch.linalg.svd(r, full_matrices=False)


def top_svd_dev(mat, k, wide=False):
    """Leading k singular triplets of a matrix with one small dimension.

    Skinny side <= 96 (config 5's RRF sketch has k1 = 80): R from TSQR, SVD
    of the small R by one-CTA Jacobi, and the long singular vectors recovered
    as mat V / sigma (or mat^T U / sigma).  Otherwise the cuSOLVER thin SVD.  wide=True forces the m < n formulation for a square
    input (as the caller's larger matrix would take)."""
    torch = _torch()
    m, n = mat.shape
    if min(m, n) > 96:
        u, s, v = thin_svd_dev(mat)
        return u[:, :k], s[:k], v[:, :k]
    if m >= n and not (wide and m == n):
        r = _tall_r_dev(mat)
        _, s, vh = _small_svd(r)
        v = vh[:k].transpose(0, 1)
        sk = s[:k]
        u = (mat @ v) / torch.where(sk > 0, sk, torch.ones_like(sk))
        return u, sk, v.contiguous()
    r = tsqr_r_dev(mat.transpose(0, 1))  # mat^T = Q r  ->  mat = r^T Q^T
    u, s, _ = _small_svd(r.transpose(0, 1))
    u = u[:, :k]
    sk = s[:k]
    v = (mat.transpose(0, 1) @ u) / torch.where(sk > 0, sk, torch.ones_like(sk))
    return u.contiguous(), sk, v


# widths above this take the R of a tall matrix from CholeskyQR2 (two Gram
# passes, one-CTA Choleskys) when that is provably accurate, instead of a TSQR
# whose Householder tiles serialise over many columns (k1 = 80: ~7 ms vs ~0.5)
CHOLQR_MIN_W = 65


def _tall_r_dev(mat):
    """R factor of a tall matrix (m >= n <= 96) with R^T R = mat^T mat.
    n >= CHOLQR_MIN_W: CholeskyQR2 -- R = R2 R1, R1 = chol(A^T A), R2 =
    chol(Q1^T Q1), Q1 = A R1^-1 -- which is orthogonal to working accuracy
    when cond(A) < ~1e7; the same safety test as the sketched system's
    (first Cholesky succeeds and diag(R1) spans < 1e6, else TSQR) decides on
    the host (the range-finder init syncs per mode anyway).  Else TSQR."""
    torch = _torch()
    n = mat.shape[1]
    if n < CHOLQR_MIN_W:
        return tsqr_r_dev(mat)
    g1 = mat.transpose(0, 1) @ mat
    r1, i1 = chol_upper_dev(g1)
    d = torch.diagonal(r1).abs()
    ok = (i1[0] == 0) & (d.min() > 0) & (d.max() < 1e6 * d.min())
    if not bool(ok.item()):
        return tsqr_r_dev(mat)
    eye = torch.eye(n, dtype=mat.dtype, device=mat.device)
    q1 = mat @ torch.linalg.solve_triangular(r1, eye, upper=True)
    r2, i2 = chol_upper_dev(q1.transpose(0, 1) @ q1)
    if int(i2[0].item()) != 0:
        return tsqr_r_dev(mat)
    return r2 @ r1


def thin_svd(mat):
    u, s, v = thin_svd_dev(_dev(mat))
    return SvdResult(_np(u), _np(s), _np(v))


def truncated_svd(mat, rank):
    res = thin_svd(mat)
    return SvdResult(res.u[:, :rank], res.singular_values[:rank], res.v[:, :rank])


# ------------------------------------------------------------------ leverage
def leverage_scores_dev(a, check=True):
    """Leverage scores of a tall factor on the device (src/linalg.py:73-84)
    and the reference's rank flag.  R <= 32: libskx's Gram-Cholesky route
    (skx_lev_scores, two passes over A); if it flags (possible rank
    deficiency or cond(A) > ~100), the checked call decides on a Householder
    R from TSQR instead, the unchecked (speculative) call returns the flag so
    the sweep is replayed on the checked path."""
    torch = _torch()
    if a.shape[0] <= a.shape[1]:
        raise ValueError("leverage scores need a strictly tall matrix")
    a = a.contiguous()
    if a.shape[1] <= 32:
        sc = torch.empty(a.shape[0], dtype=torch.float64, device="cuda")
        flag = torch.empty(1, dtype=torch.int32, device="cuda")
        nat.call_ws("skx_lev_scores", (nat.ptr(a), a.shape[0], a.shape[1], nat.ptr(sc),
                                       nat.ptr(flag)), slot=7)
        if not check:
            return sc, (flag[0] != 0)
        if int(flag.item()) == 0:
            return sc, torch.zeros((), dtype=torch.bool, device="cuda")
    if a.shape[1] <= 64:
        # Householder R by TSQR; Q = A R^-1 (same rank test on diag(R))
        r = tsqr_r_dev(a)
        tol = 1e-12 * torch.linalg.vector_norm(a)
        bad = (torch.diagonal(r).abs() < tol).any()
        if check and bool(bad.item()):
            raise RankDeficientError("rank-deficient factor in leverage_scores")
        # Q = A R^-1 through the small inverse and one GEMM (a TRSM with the
        # tall operand is latency-bound: 0.5 ms at 2e5 x 20)
        eye = torch.eye(r.shape[0], dtype=r.dtype, device=r.device)
        q = a @ torch.linalg.solve_triangular(r, eye, upper=True)
    else:
        q, r, bad = qr_flag_dev(a)
        if check and bool(bad.item()):
            raise RankDeficientError("rank-deficient factor in leverage_scores")
    return (q * q).sum(dim=1), bad


def leverage_scores(a):
    a = _dev(a)
    sc, _ = leverage_scores_dev(a)
    return LeverageProfile(_np(sc), a.shape[1])


# ------------------------------------------------------------------ normals
class NormalSource:
    """Device-resident cursor over a Generator's raw stream for
    standard_normal draws (the position lives in HBM, so consecutive draws
    need no host round trip).

    numpy's standard_normal keeps no state between calls, so k consecutive
    draws of sizes n_1..n_k are the first n_1 + ... + n_k normals of the
    stream.  With batch > 0 the source generates at least `batch` normals at
    a time and serves later draws from those segments (one ziggurat pass per
    sweep instead of one per subproblem).  Generated segments are kept until
    commit(), so snapshot()/restore() can rewind the consumption point (a
    replayed speculative sweep re-reads the same normals)."""

    def __init__(self, gen, batch=0):
        torch = _torch()
        self.gen = gen
        c = rngmod.cursor(gen)
        self.k0, self.k1 = c.k0, c.k1
        self.pos = torch.tensor([c.p], dtype=torch.int64, device="cuda")
        self.batch = int(batch)
        self._segs = []  # [(tensor, event or None)] in stream order
        self._base = 0  # absolute index of _segs[0] (segments before it were committed)
        self._i, self._off = 0, 0  # consumption point: segment, offset

    def _generate(self, n):
        torch = _torch()
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        nat.call_ws("skx_philox_normal",
                    (ctypes.c_uint64(self.k0), ctypes.c_uint64(self.k1), nat.ptr(self.pos), n,
                     nat.ptr(out), nat.ptr(self.pos)), slot=1)
        return out

    def _left(self):
        return sum(t.numel() for t, _ in self._segs[self._i:]) - self._off

    def prefetch(self):
        """Generate the next batch now (e.g. while the GPU is otherwise busy
        with compute-bound work) so the next draws are served from memory."""
        if self.batch and self._left() == 0:
            cur = _torch().cuda.current_stream()
            for _, ev in self._segs:
                if ev is not None:
                    cur.wait_event(ev)
            self._segs.append((self._generate(self.batch), None))

    def prefetch_async(self, stream):
        """Enqueue one more batch on `stream` (the draws are data-independent)
        unless a full batch beyond the buffered normals is already on its way;
        the caller's stream waits for it only when it is first used."""
        torch = _torch()
        if not self.batch or self._left() >= 2 * self.batch:
            return
        stream.wait_stream(torch.cuda.current_stream())  # device cursor order
        with torch.cuda.stream(stream):
            nxt = self._generate(self.batch)
            ev = torch.cuda.Event()
            ev.record(stream)
        self._segs.append((nxt, ev))

    def normal(self, shape):
        torch = _torch()
        n = int(np.prod(shape))
        left = self._left()
        cur = torch.cuda.current_stream()
        if left < n:
            # the device cursor (and workspace slot 1) may still be in use by a
            # segment generated on another stream: order after all of them
            for _, ev in self._segs:
                if ev is not None:
                    cur.wait_event(ev)
            self._segs.append((self._generate(max(n - left, self.batch)), None))
        parts, need = [], n
        while need > 0:
            t, ev = self._segs[self._i]
            if ev is not None:
                cur.wait_event(ev)
                t.record_stream(cur)
            take = min(need, t.numel() - self._off)
            parts.append(t[self._off:self._off + take])
            need -= take
            self._off += take
            if self._off == t.numel():
                self._i, self._off = self._i + 1, 0
        out = parts[0] if len(parts) == 1 else torch.cat(parts)
        return out.view(*shape)

    def snapshot(self):
        """Consumption point to return to if a speculative sweep is replayed
        (absolute segment index, offset)."""
        return (self._base + self._i, self._off)

    def restore(self, snap):
        i, off = snap
        if i < self._base:
            raise RuntimeError("NormalSource.restore: point already committed")
        self._i, self._off = i - self._base, off

    def commit(self, snap=None):
        """Release the segments fully consumed before `snap` (default: the
        current point); no rewind before it afterwards."""
        i = self._base + self._i if snap is None else snap[0]
        drop = max(0, i - self._base)
        del self._segs[:drop]
        self._base += drop
        self._i -= drop

    def sync_host(self):
        """Move the numpy Generator to where numpy would be (one D2H)."""
        if self._left() != 0:
            raise RuntimeError("NormalSource.sync_host: buffered normals not consumed")
        rngmod.set_cursor(self.gen, int(self.pos.item()))


# ------------------------------------------------------------------ rsvd_lrls
def _row_major(t):
    """(tensor, leading dim) of a 2-D view whose rows are contiguous."""
    if t.stride(1) == 1 and t.stride(0) >= t.shape[1]:
        return t, int(t.stride(0))
    t = t.contiguous()
    return t, int(t.shape[1])


def y_times_dev(y, g):
    """Y G (m x w) for the m x s right-hand side Y -- stored row-major or as
    the transpose of a row-major s x m Y^T -- and a narrow s x w G (w <= 32):
    libskx FP64 tensor-core streaming kernels (skx_gemm_ab / skx_gemm_atb)."""
    torch = _torch()
    m, s = y.shape
    w = int(g.shape[1])
    if w > 32:
        return y @ g
    gm, ldg = _row_major(g)
    out = torch.empty((m, w), dtype=torch.float64, device="cuda")
    if y.stride(0) == 1 and y.stride(1) >= m:  # Y^T storage: Y G = (Y^T)^T G
        nat.call_ws("skx_gemm_atb", (m, w, s, nat.ptr(y), int(y.stride(1)), nat.ptr(gm), ldg,
                                     nat.ptr(out), w), slot=10)
    else:
        ym, ldy = _row_major(y)
        nat.call_ws("skx_gemm_ab", (m, w, s, nat.ptr(ym), ldy, nat.ptr(gm), ldg, nat.ptr(out), w),
                    slot=10)
    return out


def ty_times_dev(wm, y):
    """W^T Y (w x s) for the m x s right-hand side Y (either storage) and a
    narrow m x w W, returned as the transpose of a contiguous s x w array."""
    torch = _torch()
    m, s = y.shape
    w = int(wm.shape[1])
    if w > 32:
        return wm.transpose(0, 1) @ y
    wmm, ldw = _row_major(wm)
    out = torch.empty((s, w), dtype=torch.float64, device="cuda")  # (W^T Y)^T = Y^T W
    if y.stride(0) == 1 and y.stride(1) >= m:  # Y^T row-major s x m: Y^T W streams its rows
        nat.call_ws("skx_gemm_ab", (s, w, m, nat.ptr(y), int(y.stride(1)), nat.ptr(wmm), ldw,
                                    nat.ptr(out), w), slot=10)
    else:
        ym, ldy = _row_major(y)
        nat.call_ws("skx_gemm_atb", (s, w, m, nat.ptr(ym), ldy, nat.ptr(wmm), ldw, nat.ptr(out), w),
                    slot=10)
    return out.transpose(0, 1)


def resid_dev(z, core_t, a, y):
    """|| Z core_t a^T - Y ||_F as a device scalar (src/tucker.py:274); one
    fused pass over Y in its storage order."""
    torch = _torch()
    p = z @ core_t  # (m, R)
    m, s = y.shape
    R = int(p.shape[1])
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    if y.stride(0) == 1:  # Y^T storage (s, m): outer i, inner j
        u, vt, n_out, n_in, ld = a.contiguous(), p.t().contiguous(), s, m, y.stride(1)
    elif y.stride(1) == 1:  # row-major Y: outer j, inner i
        u, vt, n_out, n_in, ld = p.contiguous(), a.t().contiguous(), m, s, y.stride(0)
    else:
        y = y.contiguous()
        u, vt, n_out, n_in, ld = p.contiguous(), a.t().contiguous(), m, s, s
    nat.call_ws("skx_resid_sq", (nat.ptr(u), nat.ptr(vt), n_out, n_in, R, nat.ptr(y), ld,
                                 nat.ptr(out)))
    return torch.sqrt(out[0])


def sketch_qr_dev(z, defer=None):
    """Reduced QR of the sketched system Z (m x r) with the reference's rank
    test.  Cholesky QR (small Gram, Cholesky -- one-CTA libskx kernel up to
    r = 128, cuSOLVER potrf beyond -- TRSM; no LAPACK Householder panel).  One pass already gives Q orthonormal to 1e-13 for the
    well-conditioned Z a TensorSketch of orthonormal factors produces (the
    orthogonality defect of Q is measured, not assumed); otherwise a second
    pass (CholeskyQR2), and when even that is unsafe (first Cholesky fails or
    diag(R) spans >= 1e6, i.e. cond(Z) near eps^-1/2) the Householder QR of
    cuSOLVER runs -- the same rank decision as src/linalg.py:44-52.  One host
    sync decides (a second only on the CholeskyQR2 path).

    defer (a list): speculative form without the host sync -- the one-pass
    factors are returned and a device flag "this sub-problem must be redone
    on the checked path" (unsafe, second pass needed, or rank-deficient) is
    appended; the caller verifies the flags later and replays on failure."""
    torch = _torch()
    m, r = z.shape
    if m < r:
        return qr_flag_dev(z)

    def chol(g):
        """(R, R^-1 or None, info): one-CTA libskx kernels -- register Cholesky
        up to 128, blocked Cholesky + inverse up to 512; cuSOLVER potrf beyond
        (no host sync either way)."""
        if r <= 128:
            u, info = chol_upper_dev(g)
            return u, None, info
        if r <= CHOL_INV_MAX and not os.environ.get("SKX_CHOL_CUSOLVER"):  # (env: A/B runs)
            return chol_inv_upper_dev(g)
        u, info = torch.linalg.cholesky_ex(g, upper=True)
        return u, None, info.view(1)

    def inverse(u, uinv):
        if uinv is None:
            uinv = torch.linalg.solve_triangular(u, torch.eye(r, dtype=z.dtype, device=z.device),
                                                 upper=True)
        return uinv

    g1 = z.transpose(0, 1) @ z
    r1, r1inv, i1 = chol(g1)
    if r <= 128:
        z1 = torch.linalg.solve_triangular(r1, z, upper=True, left=False)
    else:
        # large r: R^-1 (from the Cholesky kernel itself up to r = 512) and one
        # GEMM, instead of a latency-bound TRSM with the m x r operand
        r1inv = inverse(r1, r1inv)
        z1 = z @ r1inv
        r1._skx_inv = r1inv  # reused by assoc_mid_dev when the one-pass R is kept
    g2 = z1.transpose(0, 1) @ z1
    # unsafe / one pass suffices / rank-deficient (+ replay flag) in one libskx CTA
    fl = torch.empty(4, dtype=torch.int32, device="cuda")
    nat.call("skx_cholqr_flags", nat.ptr(g1.contiguous()), nat.ptr(r1.contiguous()),
             nat.ptr(i1.to(torch.int32)), nat.ptr(g2.contiguous()), r, nat.ptr(fl), nat.stream())
    if defer is not None:
        defer.append(fl[3])
        return z1, r1, None
    flags = fl[:3].cpu()
    if bool(flags[0]):
        return qr_flag_dev(z)
    if bool(flags[1]):
        return z1, r1, flags[2]
    r2, r2inv, i2 = chol(g2)
    if r <= 128:
        q = torch.linalg.solve_triangular(r2, z1, upper=True, left=False)
    else:
        r2inv = inverse(r2, r2inv)
        q = z1 @ r2inv
    rz = r2 @ r1
    if r > 128:
        rz._skx_inv = r1inv @ r2inv  # (R2 R1)^-1
    tol = 1e-12 * torch.sqrt(torch.trace(g1))  # ||Z||_F
    bad = (torch.diagonal(rz).abs() < tol).any()
    flags2 = torch.stack([i2[0] != 0, bad]).cpu()
    if bool(flags2[0]):
        return qr_flag_dev(z)
    return q, rz, flags2[1]


def assoc_mid_dev(qz, rz, yg):
    """(q, W) of the associated rsvd_lrls form: c = R_z^-1 Q_z^T (Y G) and its
    thin Q (src/linalg.py:105-109: x_ls G = R^-1 Q^T (Y G)), W = Q_z R_z^-T q.
    One libskx CTA does both triangular solves and the Householder QR when
    r <= 128 and the width <= 32 (cuBLAS TRSM + cuSOLVER QR beyond)."""
    torch = _torch()
    r, w = rz.shape[0], yg.shape[1]
    b = qz.transpose(0, 1) @ yg
    if r <= 128 and w <= 32 and w <= r:
        q = torch.empty((r, w), dtype=torch.float64, device="cuda")
        x = torch.empty((r, w), dtype=torch.float64, device="cuda")
        nat.call("skx_lrls_mid", nat.ptr(rz.contiguous()), nat.ptr(b.contiguous()), r, w,
                 nat.ptr(q), nat.ptr(x), nat.stream())
        return q, qz @ x
    # r > 128: R^-1 once (one TRSM with r right-hand sides, or the one-pass
    # Cholesky QR's own), then GEMMs
    rinv = getattr(rz, "_skx_inv", None)
    if rinv is None:
        rinv = torch.linalg.solve_triangular(rz, torch.eye(r, dtype=rz.dtype, device=rz.device),
                                             upper=True)
    c = rinv @ b
    q = house_q_dev(c) if w <= 32 and 2 * r * w * 8 <= HOUSE_Q_SMEM else \
        torch.linalg.qr(c, mode="reduced")[0]
    return q, qz @ (rinv.transpose(0, 1) @ q)


def rsvd_lrls_dev(z, y, rank, normals, oversample=10, check=True, defer=None, pre=None):
    """Algorithm 5 (src/linalg.py:87-113) on device.
    z: (m, r) CUDA tensor (any strides), y: (m, s) CUDA tensor view.
    Returns (core_t (r, rank), a (s, rank), rank_bad flag).  defer: see
    sketch_qr_dev (the rank check is then the caller's).  pre = (g, yg,
    event): the Gaussian test matrix already drawn and Y G computed on another
    stream (speculative sweeps only: drawing before the rank check would
    consume the stream on a rank-deficient system)."""
    torch = _torch()
    m, r = z.shape
    s = y.shape[1]
    if m < r:
        raise ValueError(f"need at least as many rows as columns in z ({m} < {r})")
    if rank > min(r, s):
        raise ValueError(f"rank {rank} exceeds min({r}, {s})")
    qz, rz, bad = sketch_qr_dev(z, defer)
    if check and defer is None and bool(bad.item()):
        raise RankDeficientError("rank-deficient sketched system")
    width = min(rank + oversample, s)
    if pre is not None:
        g, yg, ev = pre
        cur = torch.cuda.current_stream()
        cur.wait_event(ev)
        yg.record_stream(cur)
    else:
        g = normals.normal((s, width))
        yg = None
    if width < r:
        # Same algebra, associated so that Y (m x s, the big operand) only meets
        # width-column matrices: X_ls G = R^-1 Q_z^T (Y G) and
        # Q^T X_ls = (Q_z R^-T Q)^T Y.  2.5x fewer flops at configs 2/4/5.
        q, wm = assoc_mid_dev(qz, rz, y_times_dev(y, g) if yg is None else yg)
        d = ty_times_dev(wm, y)
    else:
        x = torch.linalg.solve_triangular(rz, qz.transpose(0, 1) @ y, upper=True)
        q, _ = torch.linalg.qr(x @ g, mode="reduced")
        d = q.transpose(0, 1) @ x
    u, sv, v = top_svd_dev(d, rank)
    core_t = q @ (u * sv)
    return core_t, v.contiguous(), bad


def rsvd_lrls_rows_dev(z, yt_loc, row_lo, s, rank, normals, comm, oversample=10, check=True,
                       defer=None):
    """rsvd_lrls_dev + residual with the right-hand side split by columns over
    ranks: this rank holds Y^T rows [row_lo, row_lo + rows) as
    yt_loc.  Column-separable steps run on the local block -- Y G (all-reduced,
    m x w), D^T = Y^T W (local rows), the residual (all-reduced scalar) -- and
    the SVD of D goes through a TSQR whose leaves are the ranks' R factors
    (all-gathered, w x w each).  Returns (core_t, a_loc (rows x rank), bad,
    resid); the caller all-gathers a_loc."""
    torch = _torch()
    m, r = z.shape
    if m < r:
        raise ValueError(f"need at least as many rows as columns in z ({m} < {r})")
    if rank > min(r, s):
        raise ValueError(f"rank {rank} exceeds min({r}, {s})")
    qz, rz, bad = sketch_qr_dev(z, defer)
    if check and defer is None and bool(bad.item()):
        raise RankDeficientError("rank-deficient sketched system")
    width = min(rank + oversample, s)
    g = normals.normal((s, width))  # the whole stream is drawn on every rank
    rows = yt_loc.shape[0]
    g_loc = g[row_lo:row_lo + rows]
    y_loc = yt_loc.t()  # m x rows
    if width < r:
        yg = comm.allreduce((y_loc @ g_loc).contiguous())
        q, wm = assoc_mid_dev(qz, rz, yg)
        dt_loc = yt_loc @ wm  # rows x w  (= (W^T Y)^T on this block)
    else:
        xt_loc = torch.linalg.solve_triangular(rz, qz.transpose(0, 1) @ y_loc, upper=True).t()
        xg = comm.allreduce((xt_loc.t() @ g_loc).contiguous())
        q, _ = torch.linalg.qr(xg, mode="reduced")
        dt_loc = xt_loc @ q
    # SVD of D (wd x s, wd = q's width): TSQR over the ranks' row blocks of D^T
    wd = int(dt_loc.shape[1])
    if rows >= wd:
        r_loc = tsqr_r_dev(dt_loc.contiguous())
    else:
        pad = torch.zeros((wd, wd), dtype=torch.float64, device="cuda")
        pad[:rows] = dt_loc
        r_loc = tsqr_r_dev(pad)
    r_all = comm.allgather(r_loc.contiguous().reshape(-1)).reshape(-1, wd)
    rr = tsqr_r_dev(r_all)
    u, sv, _ = _small_svd(rr.transpose(0, 1))
    u = u[:, :rank]
    sk = sv[:rank]
    a_loc = (dt_loc @ u) / torch.where(sk > 0, sk, torch.ones_like(sk))
    core_t = q @ (u * sk)
    res2 = resid_dev(z, core_t, a_loc.contiguous(), y_loc) ** 2
    res = torch.sqrt(comm.allreduce(res2.reshape(1))[0])
    return core_t, a_loc, bad, res


def rsvd_lrls_hits_dev(z, hit_off, hit_col, hit_val, s, rank, normals, oversample=10,
                       check=True, hit_row=None, defer=None):
    """rsvd_lrls_dev for a sparse right-hand side given as leverage-gather hits
    (row j's entries at hit_col/hit_val[hit_off[j]:hit_off[j+1]], distinct
    columns per row; or explicit rows in hit_row), plus its residual.  Same algebra as the dense call on
    the m x s matrix of the hits, restricted to the set H of columns that hold
    a hit: every product with Y only sees Y's nonzero columns, D = W^T Y is
    zero outside H, so the SVD is taken of D_H and the factor rows outside H
    are exactly zero.  The Gaussian test matrix is still drawn s x w, so the
    rng_solve stream advances exactly as in the reference.  Returns
    (core_t, a (s x rank), bad, resid)."""
    torch = _torch()
    m, r = z.shape
    if m < r:
        raise ValueError(f"need at least as many rows as columns in z ({m} < {r})")
    if rank > min(r, s):
        raise ValueError(f"rank {rank} exceeds min({r}, {s})")
    qz, rz, bad = sketch_qr_dev(z, defer)
    if check and defer is None and bool(bad.item()):
        raise RankDeficientError("rank-deficient sketched system")
    width = min(rank + oversample, s)
    g = normals.normal((s, width))
    if hit_row is None:
        counts = hit_off[1:] - hit_off[:-1]
        rows = torch.repeat_interleave(torch.arange(m, device="cuda"), counts)
    else:  # explicit (row, col, val) triples (e.g. gathered from several ranks)
        rows = hit_row
    cols, inv = torch.unique(hit_col, return_inverse=True)
    nh = int(cols.numel())
    yh = torch.zeros((m, max(nh, 1)), dtype=torch.float64, device="cuda")
    if nh:
        yh[rows, inv] = hit_val
    gh = g[cols] if nh else torch.zeros((1, width), dtype=torch.float64, device="cuda")
    if width < r:
        q, wm = assoc_mid_dev(qz, rz, yh @ gh)
        dh = wm.transpose(0, 1) @ yh
    else:
        xh = torch.linalg.solve_triangular(rz, qz.transpose(0, 1) @ yh, upper=True)
        q, _ = torch.linalg.qr(xh @ gh, mode="reduced")
        dh = q.transpose(0, 1) @ xh
    # the dense call factors D (w x s, s >= w) through its wide branch; keep
    # that branch (zero columns appended when |H| < w leave R unchanged)
    if dh.shape[1] < dh.shape[0]:
        dh = torch.cat([dh, torch.zeros((dh.shape[0], dh.shape[0] - dh.shape[1]),
                                        dtype=torch.float64, device="cuda")], dim=1)
    u, sv, vh = top_svd_dev(dh, rank, wide=True)
    core_t = q @ (u * sv)
    a = torch.zeros((s, rank), dtype=torch.float64, device="cuda")
    if nh:
        a[cols] = vh[:nh]
    # residual: Z core_t a^T is zero outside H, so is Y
    p = z @ core_t
    resid = torch.linalg.vector_norm(p @ a[cols].transpose(0, 1) - yh[:, :nh]) if nh else \
        torch.zeros((), dtype=torch.float64, device="cuda")
    return core_t, a, bad, resid


def rsvd_lrls_hits_fixed_dev(z, hit_off, hit_col, hit_val, s, rank, normals, oversample=10,
                             defer=None):
    """rsvd_lrls_hits_dev with no host synchronisation: the hit list has a
    fixed capacity (entries past the device total carry column s and value
    0, see sketching.gather_slices_fixed_dev), the distinct hit columns are
    found by a stable sort with a device-side segment count, and every product
    with Y_H is a deterministic segment sum over the hits -- nothing is sized
    on the host.  Same algebra: Y G and W^T Y restricted to the hit columns,
    D padded with zero columns (the SVD of D and the factor rows are unchanged:
    rows outside the hit columns are exactly zero).  The residual
    ||Z core_t a^T - Y||_F^2 is split into the hit entries, sum (e_k - v_k)^2,
    and the model mass elsewhere, ||P a^T||_F^2 - sum e_k^2 with P = Z core_t.
    Returns (core_t, a (s x rank), bad, resid)."""
    torch = _torch()
    m, r = z.shape
    if m < r:
        raise ValueError(f"need at least as many rows as columns in z ({m} < {r})")
    if rank > min(r, s):
        raise ValueError(f"rank {rank} exceeds min({r}, {s})")
    qz, rz, bad = sketch_qr_dev(z, defer)
    width = min(rank + oversample, s)
    g = normals.normal((s, width))
    cap = int(hit_col.numel())
    offs = hit_off.clamp(max=cap)
    k = torch.arange(cap, device="cuda")
    row = (torch.searchsorted(hit_off, k, right=True) - 1).clamp(0, m - 1)
    gpad = torch.cat([g, torch.zeros((1, width), dtype=g.dtype, device="cuda")])
    # Y G (m x width): per row, its hits' v g[col] in hit order
    yg = torch.segment_reduce(hit_val[:, None] * gpad[hit_col], "sum", offsets=offs, axis=0,
                              unsafe=True)
    q, wm = assoc_mid_dev(qz, rz, yg)
    # distinct hit columns (ascending; the sentinel s sorts last)
    scol, perm = torch.sort(hit_col, stable=True)
    newseg = torch.ones(cap, dtype=torch.bool, device="cuda")
    newseg[1:] = scol[1:] != scol[:-1]
    uid = torch.cumsum(newseg, 0) - 1
    first = torch.full((cap + 1,), cap, dtype=torch.int64, device="cuda")
    first.scatter_reduce_(0, uid, k, reduce="amin")
    ucol = torch.full((cap,), s, dtype=torch.int64, device="cuda")
    ucol.scatter_(0, uid, scol)
    # D^T (cap x width): per distinct column, its hits' v W[row] in sorted order
    contrib = (hit_val[:, None] * wm[row])[perm]
    dt = torch.segment_reduce(contrib, "sum", offsets=first, axis=0, unsafe=True)
    u, sv, vh = top_svd_dev(dt.t(), rank, wide=True)
    core_t = q @ (u * sv)
    a = torch.zeros((s + 1, rank), dtype=torch.float64, device="cuda")
    a.index_copy_(0, ucol, vh)  # padded slots (column s) carry zero rows
    a = a[:s].contiguous()
    p = z @ core_t
    e = (p[row] * a.index_select(0, hit_col.clamp(max=s - 1))).sum(dim=1)
    e = torch.where(hit_col < s, e, torch.zeros_like(e))
    hit_part = ((e - hit_val) ** 2).sum()
    model = ((p.transpose(0, 1) @ p) * (a.transpose(0, 1) @ a)).sum()
    resid = torch.sqrt(torch.clamp(hit_part + model - (e * e).sum(), min=0.0))
    return core_t, a, bad, resid


def rsvd_lrls(z, y, rank, rng, oversample=10):
    """Rank-constrained least squares min ||z x - y|| via randomized SVD."""
    z = _dev(z)
    y = _dev(y)
    src = NormalSource(rngmod.make_rng(rng))
    core_t, v, _ = rsvd_lrls_dev(z, y, rank, src, oversample)
    src.sync_host()
    return _np(core_t), _np(v)


def qr_lapack_dev(a):
    """Thin Householder QR with LAPACK's reflector convention (dgeqrf/dlarfg:
    beta = -sign(alpha) ||x||, v(1) = 1, tau = (beta - alpha) / beta; Q from
    the reflectors as dorgqr), so Q's column signs are numpy.linalg.qr's.
    Needed where a factor's signs are not washed out downstream (ref_tucker_ts
    re-orthonormalises a factor while the core stays fixed, src/tucker.py:
    353-356).  Column loop of small device ops, no host sync; for narrow
    matrices (k = rank columns)."""
    torch = _torch()
    A = a.to(torch.float64).clone()
    m, k = A.shape
    vs, taus = [], []
    for j in range(min(m, k)):
        x = A[j:, j]
        alpha = x[0]
        xnorm = torch.linalg.vector_norm(x[1:]) if m - j > 1 else torch.zeros((), dtype=A.dtype,
                                                                              device=A.device)
        beta = -torch.copysign(torch.hypot(alpha, xnorm), alpha)
        trivial = xnorm == 0
        tau = torch.where(trivial, torch.zeros_like(beta), (beta - alpha) / beta)
        denom = torch.where(trivial, torch.ones_like(alpha), alpha - beta)
        v = x / denom
        v[0] = 1.0
        w = v @ A[j:, j:]
        A[j:, j:] -= tau * torch.outer(v, w)
        A[j, j] = torch.where(trivial, alpha, beta)
        vs.append(v)
        taus.append(tau)
    Q = torch.eye(m, k, dtype=A.dtype, device=A.device)
    for j in reversed(range(len(vs))):
        v = vs[j]
        Q[j:, :] -= taus[j] * torch.outer(v, v @ Q[j:, :])
    return Q, torch.triu(A[:k, :])
