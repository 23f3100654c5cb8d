"""GPU: the small dense factorisations behind K5/K6 at the widths the
BASELINE configs reach (config 5: RRF sketch k1 = 80), against LAPACK
(numpy): TSQR R factor (same dlarfg sign convention, so R itself matches),
one-CTA Jacobi SVD, top-k SVD, Gram-Cholesky leverage scores, and the
numpy-sign Householder QR."""
import numpy as np
import pytest

from tests.conftest import relerr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,w", [(20000, 8), (5000, 40), (200000, 80), (3000, 96)])
def test_tsqr_r_matches_lapack(n, w):
    import torch
    from paper_2104_01101_b200.linalg import tsqr_r_dev
    a = np.random.default_rng(w).standard_normal((n, w))
    r = tsqr_r_dev(torch.from_numpy(a).cuda()).cpu().numpy()
    rn = np.linalg.qr(a, mode="r")
    # same Householder sign convention: R itself, not only |R|
    assert relerr(np.abs(r), np.abs(rn)) <= 1e-12
    assert relerr(r.T @ r, a.T @ a) <= 1e-12


@pytest.mark.parametrize("n", [10, 64, 80, 112])
def test_jacobi_svd(n):
    import torch
    from paper_2104_01101_b200.linalg import jacobi_svd_dev
    g = np.random.default_rng(n)
    a = g.standard_normal((n, n)) @ np.diag(np.logspace(0, -6, n))
    u, s, v = (x.cpu().numpy() for x in jacobi_svd_dev(torch.from_numpy(a).cuda()))
    assert relerr(s, np.linalg.svd(a, compute_uv=False)) <= 1e-12
    assert relerr((u * s) @ v.T, a) <= 1e-12
    assert relerr(u.T @ u, np.eye(n)) <= 1e-12


def test_top_svd_k1_80():
    """The RRF sketch of config 5: B is s_n x k1 = 2e5 x 80."""
    import torch
    from paper_2104_01101_b200.linalg import top_svd_dev
    g = np.random.default_rng(5)
    b = g.standard_normal((20000, 80)) @ np.diag(np.logspace(0, -3, 80))
    u, s, v = (x.cpu().numpy() for x in top_svd_dev(torch.from_numpy(b).cuda(), 20))
    un, sn, vn = np.linalg.svd(b, full_matrices=False)
    assert relerr(s, sn[:20]) <= 1e-12
    assert relerr(np.abs(u), np.abs(un[:, :20])) <= 1e-10


@pytest.mark.parametrize("s,r", [(200000, 20), (400, 10), (50, 3)])
def test_leverage_scores_gram_route(s, r):
    import torch
    from paper_2104_01101_b200.linalg import leverage_scores_dev
    g = np.random.default_rng(s + r)
    a = np.linalg.qr(g.standard_normal((s, r)))[0]
    q = np.linalg.qr(a)[0]
    want = (q * q).sum(axis=1)
    got, bad = leverage_scores_dev(torch.from_numpy(a).cuda(), check=False)
    assert not bool(bad)
    assert relerr(got.cpu().numpy(), want) <= 1e-13


def test_leverage_scores_rank_deficient_falls_back():
    """A duplicated column: the Gram route flags it, the checked call decides
    on the Householder R and raises like the reference."""
    import torch
    from paper_2104_01101_b200.linalg import RankDeficientError, leverage_scores_dev
    g = np.random.default_rng(1)
    a = g.standard_normal((500, 4))
    a[:, 3] = a[:, 1]
    _, bad = leverage_scores_dev(torch.from_numpy(a).cuda(), check=False)
    assert bool(bad)
    with pytest.raises(RankDeficientError):
        leverage_scores_dev(torch.from_numpy(a).cuda(), check=True)
    # ill-conditioned but full rank: flagged, then served exactly by TSQR
    b = g.standard_normal((500, 4)) @ np.diag([1, 1, 1, 1e-4])
    sc, _ = leverage_scores_dev(torch.from_numpy(b).cuda(), check=True)
    q = np.linalg.qr(b)[0]
    assert relerr(sc.cpu().numpy(), (q * q).sum(axis=1)) <= 1e-12


@pytest.mark.parametrize("shape", [(20, 3), (5, 5), (300, 10), (1000, 20)])
def test_qr_lapack_signs(shape):
    import torch
    from paper_2104_01101_b200.linalg import qr_lapack_dev
    a = np.random.default_rng(shape[0]).standard_normal(shape)
    q, r = qr_lapack_dev(torch.from_numpy(a).cuda())
    qn, rn = np.linalg.qr(a)
    assert np.abs(q.cpu().numpy() - qn).max() <= 1e-12
    assert np.abs(r.cpu().numpy() - rn).max() <= 1e-11


@pytest.mark.parametrize("m,s,w,storage", [(1600, 100000, 20, "t"), (3200, 400, 20, "r"),
                                           (400, 120, 18, "t"), (37, 1001, 5, "r"),
                                           (100, 33, 32, "t"), (77, 9, 1, "r"),
                                           (12000, 2000, 24, "r"), (1024, 30000, 20, "t")])
def test_y_passes_vs_torch(m, s, w, storage):
    """Y G and W^T Y of rsvd_lrls on libskx's FP64 tensor-core kernels, for
    Y stored row-major (dense / leverage) or as Y^T (TensorSketch); the
    streamed-rows kernel with and without its K split (e.g. 1e5 rows: 3
    chunks; 12000 rows: 4)."""
    import torch
    from paper_2104_01101_b200.linalg import ty_times_dev, y_times_dev
    g = np.random.default_rng(m + s)
    yh = g.standard_normal((m, s))
    y = (torch.from_numpy(np.ascontiguousarray(yh.T)).cuda().t() if storage == "t"
         else torch.from_numpy(yh).cuda())
    G = torch.from_numpy(g.standard_normal((s, w))).cuda()
    W = torch.from_numpy(g.standard_normal((m, w))).cuda()
    assert relerr(y_times_dev(y, G).cpu().numpy(), yh @ G.cpu().numpy()) <= 1e-13
    assert relerr(ty_times_dev(W, y).cpu().numpy(), W.cpu().numpy().T @ yh) <= 1e-13


@pytest.mark.parametrize("n", [1, 31, 33, 129, 400, 401, 450, 512])
def test_chol_inv_upper(n):
    """One-CTA blocked Cholesky + inverse (r > 128: configs 3 and 5) vs LAPACK."""
    import torch
    from paper_2104_01101_b200.linalg import chol_inv_upper_dev
    g = np.random.default_rng(n)
    z = g.standard_normal((2 * n + 8, n)) @ np.diag(np.logspace(0, -2, n))
    gram = z.T @ z
    r, rinv, info = (x.cpu().numpy() for x in chol_inv_upper_dev(torch.from_numpy(gram).cuda()))
    assert int(info[0]) == 0
    rn = np.linalg.cholesky(gram).T
    assert np.all(np.tril(r, -1) == 0) and np.all(np.tril(rinv, -1) == 0)
    assert relerr(r, rn) <= 1e-12
    assert relerr(rinv, np.linalg.inv(rn)) <= 1e-11
    assert relerr(r @ rinv, np.eye(n)) <= 1e-12


@pytest.mark.parametrize("n", [300, 480])  # one CTA / cooperative grid
def test_chol_inv_upper_not_spd(n):
    import torch
    from paper_2104_01101_b200.linalg import chol_inv_upper_dev
    g = np.random.default_rng(1)
    a = g.standard_normal((n, n))
    gram = a @ a.T
    gram[100, 100] = -1.0  # pivot 100 (or earlier) fails
    r, rinv, info = (x.cpu().numpy() for x in chol_inv_upper_dev(torch.from_numpy(gram).cuda()))
    assert 1 <= int(info[0]) <= 101
    assert not r.any() and not rinv.any()


@pytest.mark.parametrize("r,w", [(400, 30), (512, 18), (130, 32), (40, 7)])
def test_house_q(r, w):
    """Thin Householder Q of the associated middle step (r > 128) vs LAPACK:
    same reflector convention, so Q itself matches numpy's."""
    import torch
    from paper_2104_01101_b200.linalg import house_q_dev
    g = np.random.default_rng(r + w)
    c = g.standard_normal((r, w)) @ np.diag(np.logspace(0, -8, w))
    q = house_q_dev(torch.from_numpy(c).cuda()).cpu().numpy()
    qn = np.linalg.qr(c)[0]
    assert relerr(q, qn) <= 1e-10
    assert relerr(q.T @ q, np.eye(w)) <= 1e-13
