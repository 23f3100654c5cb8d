"""GPU parity of the operators against fixtures from the real reference
(tests/golden) and against the CPU oracle on the same seeded inputs.

Tolerances: integer tables / index sets bit-exact; sketches
<= 1e-12 Frobenius-relative; factors after sign canonicalisation <= 1e-10."""
import numpy as np
import pytest
import scipy.sparse as sp

from tests.conftest import canon, relerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def skx():
    import paper_2104_01101_b200 as m
    return m


def test_ts_tables_bit_exact(golden, skx):
    for seed in (0, 7):
        op = skx.TensorSketchOp.build((100, 120, 90), 400, skx.make_rng(seed))
        for k in range(3):
            assert np.array_equal(op.modes[k].hash, golden[f"ts_tab_s{seed}_h{k}"])
            assert np.array_equal(op.modes[k].signs, golden[f"ts_tab_s{seed}_s{k}"])


def test_ts_apply_rhs(golden, skx):
    op = skx.TensorSketchOp.build((6, 5), 16, skx.make_rng(1))
    assert relerr(skx.ts_apply_rhs(op, golden["rhs_b"]), golden["rhs_dense"]) <= 1e-14
    bs = sp.csr_matrix(golden["rhs_bs"])
    assert relerr(skx.ts_apply_rhs(op, bs), golden["rhs_sparse"]) <= 1e-14


def test_ts_apply_rhs_single_nonzero_exact(skx):
    # reference pkg/tests/test_sketching.py:109-121 (array_equal)
    op = skx.TensorSketchOp.build((3, 4), 6, skx.make_rng(23))
    b = sp.coo_matrix(([2.5], ([7], [0])), shape=(12, 1))
    out = skx.ts_apply_rhs(op, b)
    multi = np.unravel_index(np.array([7]), (3, 4))
    exp = np.zeros((6, 1))
    exp[op.combined_hash(multi)[0], 0] = op.combined_sign(multi)[0] * 2.5
    assert np.array_equal(out, exp)


def test_ts_apply_rhs_empty_sparse(skx):
    op = skx.TensorSketchOp.build((3, 4), 6, skx.make_rng(31))
    assert np.array_equal(skx.ts_apply_rhs(op, sp.coo_matrix((12, 3))), np.zeros((6, 3)))


@pytest.mark.parametrize("m,ext", [(3, (4, 4)), (8, (4, 4)), (16, (5, 3, 4)), (64, (5, 3, 4)),
                                   (400, (30, 20))])
def test_ts_apply_kron(golden, skx, m, ext):
    op = skx.TensorSketchOp.build(ext, m, skx.make_rng(200 + m))
    fs = [golden[f"kron_m{m}_f{k}"] for k in range(len(ext))]
    assert relerr(skx.ts_apply_kron(op, fs), golden[f"kron_m{m}"]) <= 1e-13


def test_ts_apply_kron_materialized(skx):
    rng = np.random.default_rng(3)
    for m in (3, 8, 16, 97, 256):
        op = skx.TensorSketchOp.build((4, 5, 3), m, skx.make_rng(m))
        fs = [rng.standard_normal((s, 2)) for s in (4, 5, 3)]
        exp = op.materialize() @ np.kron(np.kron(fs[0], fs[1]), fs[2])
        assert relerr(skx.ts_apply_kron(op, fs), exp) <= 1e-13


def test_composite(golden, skx):
    op = skx.CompositeSketchOp.build(1000, 20, 45, skx.make_rng(3))
    assert np.array_equal(op.stage.hash, golden["rrf_hash"])
    assert np.array_equal(op.stage.signs, golden["rrf_signs"])
    assert np.array_equal(op.gauss, golden["rrf_gauss"])
    c = skx.CompositeSketchOp.build(50, 4, 20, skx.make_rng(4))
    mat = golden["comp_mat"]
    assert relerr(skx.composite_apply(mat, c), golden["comp_dense"]) <= 1e-13
    ms = sp.csr_matrix(mat * (np.abs(mat) > 0.8))
    assert relerr(skx.composite_apply(ms, c), golden["comp_sparse"]) <= 1e-13


def test_lev_build_bit_exact(golden, skx):
    f = [golden["lev_f0"], golden["lev_f1"]]
    s = skx.lev_build(f, 200, "random", skx.make_rng(9))
    assert np.array_equal(s.indices, golden["lev_idx"])
    assert np.allclose(s.weights, golden["lev_w"], rtol=1e-12, atol=0)


def test_lev_apply(golden, skx):
    f = [golden["levapp_f0"], golden["levapp_f1"]]
    s = skx.lev_build(f, 30, "random", skx.make_rng(12))
    assert np.array_equal(s.indices, golden["levapp_idx"])
    z, y = skx.lev_apply(s, f, golden["levapp_bt"])
    assert relerr(z, golden["levapp_z"]) <= 1e-13
    assert relerr(y, golden["levapp_y"]) <= 1e-13
    bt = golden["levapp_bt"]
    _, ys = skx.lev_apply(s, f, sp.csr_matrix(bt * (np.abs(bt) > 1.0)))
    assert relerr(ys, golden["levapp_ys"]) <= 1e-13


def test_lev_errors(skx):
    with pytest.raises(ValueError):
        skx.lev_build([np.eye(4)[:, :2]] * 2, 0, "random", skx.make_rng(0))
    col = np.random.default_rng(1).standard_normal((8, 1))
    with pytest.raises(skx.RankDeficientError):
        skx.leverage_scores(np.hstack([col, col]))


def test_rsvd_lrls(golden, skx):
    ct, v = skx.rsvd_lrls(golden["rsvd_z"], golden["rsvd_y"], 2, skx.make_rng(2))
    assert relerr(ct @ v.T, golden["rsvd_core_t"] @ golden["rsvd_v"].T) <= 1e-12
    (a,), _ = canon([v])
    (b,), _ = canon([golden["rsvd_v"]])
    assert relerr(a, b) <= 1e-11


def test_rsvd_rank_deficient(skx):
    col = np.random.default_rng(15).standard_normal((10, 1))
    with pytest.raises(skx.RankDeficientError):
        skx.rsvd_lrls(np.hstack([col, col]), np.ones((10, 4)), 1, skx.make_rng(0))
    with pytest.raises(ValueError):
        skx.rsvd_lrls(np.random.default_rng(0).standard_normal((10, 3)), np.ones((10, 4)), 4,
                      skx.make_rng(0))


def test_init_rrf(golden, skx):
    u = skx.init_rrf(golden["rrf_tn"], 4, 8, skx.make_rng(6))
    (a,), _ = canon([u])
    (b,), _ = canon([golden["rrf_u"]])
    assert relerr(a, b) <= 1e-11


def test_fitness(golden, skx):
    t = golden["fit_t"]
    fs = [golden[f"fit_a{k}"] for k in range(3)]
    core = golden["fit_core"]
    assert skx.fitness(t, skx.TuckerModel(core, fs)) == pytest.approx(float(golden["fit_dense"]), abs=1e-13)
    st = skx.SparseTensor.from_dense(t * (np.abs(t) > 0.7))
    assert skx.fitness(st, skx.TuckerModel(core, fs)) == pytest.approx(float(golden["fit_sparse"]), abs=1e-13)
    cpf = [golden[f"fitcp_a{k}"] for k in range(3)]
    w = golden["fitcp_w"]
    assert skx.fitness(t, skx.CPModel(cpf, w)) == pytest.approx(float(golden["fitcp_dense"]), abs=1e-13)
    assert skx.fitness(st, skx.CPModel(cpf, w)) == pytest.approx(float(golden["fitcp_sparse"]), abs=1e-13)


@pytest.mark.parametrize("n,w", [(1, 1), (2, 2), (7, 5), (31, 31), (256, 20), (257, 20), (300, 8),
                                 (600, 13), (5000, 16), (9000, 24), (70_000, 32), (100_000, 20),
                                 (3000, 33), (50_000, 64), (1000, -10)])
def test_tsqr_r_matches_lapack(n, w):
    import torch
    from paper_2104_01101_b200.linalg import tsqr_r_dev
    deficient = w < 0
    w = abs(w)
    a = np.random.default_rng(n + w).standard_normal((n, w))
    if deficient:  # zero column and a repeated column: reflectors with tau = 0
        a[:, 3] = 0.0
        a[:, 5] = a[:, 2]
    if n < w:
        return
    r = tsqr_r_dev(torch.from_numpy(a).cuda()).cpu().numpy()
    ref = np.linalg.qr(a, mode="r")
    if deficient:
        # R is not unique past a dependent column (the reflector there is built
        # from rounding noise); check it is an R factor: R^T R = A^T A
        assert np.allclose(r.T @ r, a.T @ a, rtol=0, atol=1e-10 * np.abs(a.T @ a).max())
        assert r[3, 3] == 0.0 and np.allclose(np.triu(r), r)
        return
    assert relerr(np.abs(r), np.abs(ref)) <= 1e-12
    # strided (transposed) input
    rt = tsqr_r_dev(torch.from_numpy(a.T.copy()).cuda().t()).cpu().numpy()
    assert np.array_equal(rt, r)


@pytest.mark.parametrize("n", [1, 2, 7, 20, 64, 100, 128])
def test_small_cholesky(n):
    import torch
    from paper_2104_01101_b200.linalg import chol_upper_dev
    a = np.random.default_rng(n).standard_normal((3 * n, n))
    g = a.T @ a
    r, info = chol_upper_dev(torch.from_numpy(g).cuda())
    assert int(info.item()) == 0
    ref = np.linalg.cholesky(g).T
    assert relerr(r.cpu().numpy(), ref) <= 1e-13
    bad = g.copy()
    bad[n // 2, n // 2] = -1.0
    _, info = chol_upper_dev(torch.from_numpy(bad).cuda())
    assert int(info.item()) >= 1


@pytest.mark.parametrize("n", [1, 2, 3, 15, 20, 30, 31, 64])
def test_small_jacobi_svd(n):
    import torch
    from paper_2104_01101_b200.linalg import jacobi_svd_dev
    a = np.random.default_rng(n).standard_normal((n, n)) @ np.diag(np.logspace(0, 3, n))
    u, s, v = (t.cpu().numpy() for t in jacobi_svd_dev(torch.from_numpy(a).cuda()))
    ss = np.linalg.svd(a, compute_uv=False)
    assert np.allclose(s, ss, rtol=1e-12)
    assert relerr((u * s) @ v.T, a) <= 1e-13
    assert np.allclose(u.T @ u, np.eye(n), atol=1e-12) and np.allclose(v.T @ v, np.eye(n), atol=1e-12)
    # transposed (strided) input
    ut, st, vt = (t.cpu().numpy() for t in jacobi_svd_dev(torch.from_numpy(a.T.copy()).cuda().t()))
    assert np.allclose(st, s, rtol=1e-13)


@pytest.mark.parametrize("shape,k", [((50_000, 20), 10), ((30, 100_000), 20), ((400, 300), 5)])
def test_top_svd(shape, k):
    import torch
    from paper_2104_01101_b200.linalg import top_svd_dev
    rng = np.random.default_rng(1)
    a = rng.standard_normal(shape) * np.linspace(1, 3, shape[1])
    u, s, v = (t.cpu().numpy() for t in top_svd_dev(torch.from_numpy(a).cuda(), k))
    uu, ss, vvt = np.linalg.svd(a, full_matrices=False)
    assert np.allclose(s, ss[:k], rtol=1e-12)
    (cu, cv), _ = canon([u, v])
    (ru, rv), _ = canon([uu[:, :k], vvt[:k].T])
    assert relerr(cu, ru) <= 1e-10 and relerr(cv, rv) <= 1e-10


# ---------------------------------------------------------- device kernels vs oracle
def _coo_rand(shape, nnz, seed):
    from paper_2104_01101_b200.synth import planted_cp_coo_host
    return planted_cp_coo_host(shape, nnz, rank=3, seed=seed)


@pytest.mark.parametrize("shape,nnz,m", [((30, 40, 50), 5000, 64), ((200, 150, 100), 60000, 1600),
                                         ((20, 10, 30, 8), 9000, 100)])
def test_sparse_ts_rhs_all_modes_vs_oracle(skx, oracle, shape, nnz, m):
    from paper_2104_01101_b200.sketching import ts_rhs_coo_dev
    from paper_2104_01101_b200.tensors import device_of
    c, v = _coo_rand(shape, nnz, 1)
    st = skx.SparseTensor(shape, c, v)
    oc = oracle.Coo(shape, c, v)
    d = device_of(st)
    gen = skx.make_rng(5)
    ogen = oracle.generator(5)
    for n in range(len(shape)):
        ext = tuple(shape[k] for k in range(len(shape)) if k != n)
        op = skx.TensorSketchOp.build(ext, m, gen)
        hs, ss = oracle.ts_tables(ext, m, ogen)
        colptr, rec = d.fibre(n)
        yt = ts_rhs_coo_dev(op, colptr, rec, shape[n]).cpu().numpy()
        ref = oracle.ts_rhs(hs, ss, ext, m, oracle.unfold_t(oc, n))
        # same per-cell summation order as numpy's add.at -> bit-exact
        assert np.array_equal(yt.T, ref)


@pytest.mark.parametrize("case", ["skewed", "tiny_columns", "single_nnz"])
def test_sparse_ts_rhs_column_edge_cases(skx, oracle, case):
    """Warp column ranges, columns straddling chunk boundaries, long runs of
    empty columns and a single giant column: still bit-identical to add.at."""
    from paper_2104_01101_b200.sketching import ts_rhs_coo_dev
    from paper_2104_01101_b200.tensors import device_of
    rng = np.random.default_rng(3)
    shape = (4000, 60, 50)
    if case == "skewed":  # 90% of nonzeros in 3 mode-0 slices, most slices empty
        i0 = np.where(rng.uniform(size=30000) < 0.9, rng.choice([5, 1999, 3998], 30000),
                      rng.integers(0, 4000, 30000))
    elif case == "tiny_columns":
        i0 = rng.integers(0, 4000, 3000)
    else:
        i0 = np.array([1234])
    n = i0.size
    c = np.stack([i0, rng.integers(0, 60, n), rng.integers(0, 50, n)], axis=1)
    c = np.unique(c, axis=0)
    v = rng.standard_normal(c.shape[0])
    st = skx.SparseTensor(shape, c, v)
    oc = oracle.Coo(shape, c, v)
    d = device_of(st)
    for n_mode in range(3):
        ext = tuple(shape[k] for k in range(3) if k != n_mode)
        op = skx.TensorSketchOp.build(ext, 300, skx.make_rng(n_mode))
        hs, ss = oracle.ts_tables(ext, 300, oracle.generator(n_mode))
        colptr, rec = d.fibre(n_mode)
        yt = ts_rhs_coo_dev(op, colptr, rec, shape[n_mode]).cpu().numpy()
        assert np.array_equal(yt.T, oracle.ts_rhs(hs, ss, ext, 300, oracle.unfold_t(oc, n_mode)))


def test_fibre_layout_matches_stable_sort(skx):
    """The radix-sorted fibre-major records equal a stable numpy sort by i_n."""
    import torch
    from paper_2104_01101_b200.tensors import device_of
    shape = (50, 3000, 7)
    c, v = _coo_rand(shape, 20000, 9)
    d = device_of(skx.SparseTensor(shape, c, v))
    for n in range(3):
        colptr, rec = d.fibre(n)
        order = np.argsort(c[:, n], kind="stable")
        others = [k for k in range(3) if k != n]
        raw = rec.cpu().numpy().view(np.int32).reshape(-1, 4)
        assert np.array_equal(raw[:, 0], c[order, others[0]])
        assert np.array_equal(raw[:, 1], c[order, others[1]])
        assert np.array_equal(rec.cpu().numpy().reshape(-1, 2)[:, 1], v[order])
        assert np.array_equal(colptr.cpu().numpy(),
                              np.searchsorted(c[order, n], np.arange(shape[n] + 1)))


@pytest.mark.parametrize("shape,m", [((50, 3000, 7), 1600), ((200, 150, 100), 64), ((9, 1, 40), 3)])
def test_packed_ts_layout(skx, oracle, shape, m):
    """skx_coo_fibre_ts: records carry mode n's TS bucket/sign above the second
    coordinate; every consumer (RHS sketch without lookups, RHS sketch with
    lookups + mask, Tucker cross term, RRF stage 1) matches the plain layout
    bit for bit."""
    import torch
    from paper_2104_01101_b200.sketching import draw_rrf_tables, ts_rhs_coo_dev, ts_rhs_mode_dev
    from paper_2104_01101_b200.tensors import DeviceCoo, device_of, tucker_cross_dev
    from paper_2104_01101_b200.tucker import rrf_stage1_dev
    c, v = _coo_rand(shape, min(20000, int(np.prod(shape)) // 2), 5)
    st = skx.SparseTensor(shape, c, v)
    plain = device_of(st)
    oc = oracle.Coo(shape, c, v)
    for n in range(3):
        ext = tuple(shape[k] for k in range(3) if k != n)
        op = skx.TensorSketchOp.build(ext, m, skx.make_rng(n))
        packed = DeviceCoo(shape, plain.coords, plain.vals)
        yt_p = ts_rhs_mode_dev(op, packed, n)
        assert packed.fibre_packed_for(n, op) >= 0
        colptr, rec = plain.fibre(n)
        yt = ts_rhs_coo_dev(op, colptr, rec, shape[n])
        assert torch.equal(yt_p, yt)
        hs, ss = oracle.ts_tables(ext, m, oracle.generator(n))
        assert np.array_equal(yt_p.cpu().numpy().T, oracle.ts_rhs(hs, ss, ext, m, oracle.unfold_t(oc, n)))
        # lookup path on the packed records (a different operator)
        op2 = skx.TensorSketchOp.build(ext, m, skx.make_rng(n + 10))
        assert packed.fibre_packed_for(n, op2) == -1
        pc, pr = packed.fibre(n)
        assert torch.equal(ts_rhs_coo_dev(op2, pc, pr, shape[n], packed.fibre_mask(n), -1),
                           ts_rhs_coo_dev(op2, colptr, rec, shape[n]))
        # RRF stage 1 on the packed layout
        P = int(np.prod(ext))
        t1 = rrf_stage1_dev(packed, n, draw_rrf_tables(skx.make_rng(7), P, 45))
        t0 = rrf_stage1_dev(plain, n, draw_rrf_tables(skx.make_rng(7), P, 45))
        assert torch.equal(t1, t0)
        if n == 0:
            rng = np.random.default_rng(1)
            A = [torch.from_numpy(np.linalg.qr(rng.standard_normal((s, 6)))[0]).cuda() for s in shape]
            core = torch.from_numpy(rng.standard_normal((6, 6, 6))).cuda()
            assert float(tucker_cross_dev(packed, core, A)) == float(tucker_cross_dev(plain, core, A))


@pytest.mark.parametrize("shape,m", [((30, 40, 50), 64), ((12, 13, 14, 15), 256), ((100, 100, 100), 400),
                                     ((3, 200, 5), 4096)])
def test_dense_ts_rhs_all_modes_vs_oracle(skx, oracle, shape, m):
    from paper_2104_01101_b200.sketching import ts_rhs_dense_dev
    from paper_2104_01101_b200.tensors import device_of
    t = np.random.default_rng(2).standard_normal(shape)
    d = device_of(t)
    gen = skx.make_rng(9)
    ogen = oracle.generator(9)
    for n in range(len(shape)):
        ext = tuple(shape[k] for k in range(len(shape)) if k != n)
        op = skx.TensorSketchOp.build(ext, m, gen)
        hs, ss = oracle.ts_tables(ext, m, ogen)
        yt = ts_rhs_dense_dev(op, d, n).cpu().numpy()
        ref = oracle.ts_rhs(hs, ss, ext, m, oracle.unfold_t(t, n))
        assert relerr(yt.T, ref) <= 1e-13


def test_sparse_rrf_stage1_vs_oracle(skx, oracle):
    from paper_2104_01101_b200.sketching import draw_rrf_tables
    from paper_2104_01101_b200.tensors import device_of
    from paper_2104_01101_b200.tucker import rrf_stage1_dev
    shape = (300, 200, 100)
    c, v = _coo_rand(shape, 50000, 2)
    st = skx.SparseTensor(shape, c, v)
    oc = oracle.Coo(shape, c, v)
    d = device_of(st)
    for n, k2 in ((1, 157), (2, 480), (0, 45)):
        P = int(np.prod(shape)) // shape[n]
        g = skx.make_rng(n)
        og = oracle.generator(n)
        tabs = draw_rrf_tables(g, P, k2)
        st1 = rrf_stage1_dev(d, n, tabs).cpu().numpy()
        h, s, gauss = oracle.rrf_tables(P, 4, k2, og)
        tm = sp.csr_matrix((s, (np.arange(P), h)), shape=(P, k2))
        ref = np.asarray((oracle.unfold(oc, n) @ tm).todense())
        assert relerr(st1, ref) <= 1e-14
        assert np.array_equal(g.standard_normal((k2, 4)) / 2.0, gauss)


def test_dense_gather_and_kron_rows(skx, oracle):
    from paper_2104_01101_b200.sketching import gather_dense_dev, kron_rows_dev, lev_sample_dev
    from paper_2104_01101_b200.tensors import device_of
    import torch
    shape = (20, 30, 25)
    t = np.random.default_rng(4).standard_normal(shape)
    d = device_of(t)
    rng = np.random.default_rng(8)
    A = [np.linalg.qr(rng.standard_normal((s, 3)))[0] for s in shape]
    for n in range(3):
        others = [k for k in range(3) if k != n]
        fs = [torch.from_numpy(A[k]).cuda() for k in others]
        g = skx.make_rng(3 + n)
        idx, w, _, _ = lev_sample_dev(fs, 77, g)
        oidx, ow, _ = oracle.lev_sample([A[k] for k in others], 77, oracle.generator(3 + n))
        assert np.array_equal(idx.cpu().numpy(), oidx)
        z = kron_rows_dev(fs, idx, w).cpu().numpy()
        y = gather_dense_dev(d, n, idx, w).cpu().numpy()
        ext = tuple(shape[k] for k in others)
        oz, oy = oracle.lev_rows(oidx, ow, ext, [A[k] for k in others], oracle.unfold_t(t, n))
        assert relerr(z, oz) <= 1e-14
        assert relerr(y, oy) <= 1e-14


def test_sparse_fitness_order3_and_generic(skx, oracle):
    rng = np.random.default_rng(6)
    cases = (((50, 40, 30), (3, 4, 5)), ((10, 12, 9, 7), (2, 3, 2, 2)), ((60, 50, 40), (20, 20, 20)),
             ((40, 50, 60), (10, 10, 10)), ((40, 50, 60), (4, 4, 4)), ((40, 50, 60), (7, 9, 13)),
             ((40, 50, 60), (12, 32, 17)))
    for shape, R in cases:
        c, v = _coo_rand(shape, 4000, 3)
        st = skx.SparseTensor(shape, c, v)
        oc = oracle.Coo(shape, c, v)
        A = [np.linalg.qr(rng.standard_normal((s, r)))[0] for s, r in zip(shape, R)]
        core = rng.standard_normal(R)
        got = skx.fitness(st, skx.TuckerModel(core, A))
        exp = oracle.fitness_tucker(oc, core, A)
        assert got == pytest.approx(exp, rel=1e-11, abs=1e-12)


@pytest.mark.parametrize("R", [1, 4, 5, 8, 10, 13, 20, 32, 40])
@pytest.mark.parametrize("orient", ["yt", "rowmajor", "odd_ld"])
def test_resid_pass(R, orient):
    """|| Z C A^T - Y ||_F of the rank-constrained solve (src/tucker.py:274) on
    every kernel path: tensor-core tiles (5 <= R <= 32), SIMT (R <= 4), generic
    (R > 32); ragged row/column counts and both storage orders of Y."""
    import torch
    from paper_2104_01101_b200.linalg import resid_dev
    rng = np.random.default_rng(R)
    m, s, r2 = 203, 1037, 24
    z = rng.standard_normal((m, r2))
    c = rng.standard_normal((r2, R))
    a = rng.standard_normal((s, R))
    y = z @ c @ a.T + 0.1 * rng.standard_normal((m, s))
    if orient == "yt":        # Y^T stored (s, m) row-major, as the sketches produce it
        yd = torch.from_numpy(y.T.copy()).cuda().t()
    elif orient == "rowmajor":
        yd = torch.from_numpy(y).cuda()
    else:                     # odd leading dimension (unaligned rows)
        buf = torch.from_numpy(np.zeros((s, m + 1))).cuda()
        buf[:, :m] = torch.from_numpy(y.T.copy()).cuda()
        yd = buf[:, :m].t()
    got = float(resid_dev(torch.from_numpy(z).cuda(), torch.from_numpy(c).cuda(),
                          torch.from_numpy(a).cuda(), yd))
    exp = np.linalg.norm(z @ c @ a.T - y)
    assert got == pytest.approx(exp, rel=1e-12)


@pytest.mark.parametrize("m,r,s,rank,nh", [(300, 100, 5000, 10, 40), (300, 16, 4000, 8, 400),
                                           (200, 25, 3000, 5, 7), (64, 9, 800, 3, 4)])
def test_rsvd_hits_matches_dense(m, r, s, rank, nh):
    """The hit-column rsvd (sparse leverage right-hand sides) equals the dense
    rsvd_lrls_dev + residual on the same hits and the same Gaussian stream:
    both reassociation branches (width < r and width >= r) and |H| < width."""
    import torch
    from paper_2104_01101_b200 import rng as rngmod
    from paper_2104_01101_b200.linalg import NormalSource, resid_dev, rsvd_lrls_dev, rsvd_lrls_hits_dev
    from paper_2104_01101_b200.sketching import hits_to_dense
    rng = np.random.default_rng(m + nh)
    z = torch.from_numpy(rng.standard_normal((m, r))).cuda()
    hit_cols = rng.choice(s, nh, replace=False)
    per_row = [np.sort(rng.choice(hit_cols, rng.integers(0, min(nh, 6) + 1), replace=False)) for _ in range(m)]
    off = torch.from_numpy(np.concatenate([[0], np.cumsum([len(p) for p in per_row])]).astype(np.int64)).cuda()
    col = torch.from_numpy(np.concatenate(per_row).astype(np.int64)).cuda()
    val = torch.from_numpy(rng.standard_normal(int(off[-1]))).cuda()
    y = hits_to_dense(off, col, val, m, s)
    ct0, a0, _ = rsvd_lrls_dev(z, y, rank, NormalSource(rngmod.make_rng(5)))
    res0 = float(resid_dev(z, ct0, a0, y))
    ct1, a1, _, res1 = rsvd_lrls_hits_dev(z, off, col, val, s, rank, NormalSource(rngmod.make_rng(5)))
    # singular vectors are defined up to sign (the R factors of D and D_H differ
    # in row signs): compare after the SURVEY 8c canonicalisation
    (a1c,), c1 = canon([a1.cpu().numpy()], ct1.cpu().numpy().T)
    (a0c,), c0 = canon([a0.cpu().numpy()], ct0.cpu().numpy().T)
    assert relerr(a1c, a0c) <= 1e-11
    assert relerr(c1, c0) <= 1e-11
    assert float(res1) == pytest.approx(res0, rel=1e-11)


def test_integration_md_ctypes_binding(skx, oracle):
    """The raw ctypes binding shown in INTEGRATION.md (no package code on the
    call path: skx_ts_tables, skx_coo_fibre_ts, skx_ts_rhs_coo) reproduces the
    reference's ts_apply_rhs bit for bit."""
    import ctypes
    import torch
    from paper_2104_01101_b200 import _native as nat
    lib = ctypes.CDLL(nat.lib_path())
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    lib.skx_ts_tables.argtypes = [ctypes.c_int, vp, vp, i64, vp, vp]
    lib.skx_coo_fibre_ts.argtypes = [vp, ctypes.c_int, i64, vp, vp, vp, vp, i64, vp, vp,
                                     ctypes.POINTER(ctypes.c_uint32), vp,
                                     ctypes.POINTER(ctypes.c_size_t), vp]
    lib.skx_ts_rhs_coo.argtypes = [ctypes.c_int, i64, vp, vp, vp, vp, i64, ctypes.c_uint32,
                                   ctypes.c_int, vp, vp]
    shape, m, mode = (60, 70, 80), 300, 1
    c, v = _coo_rand(shape, 20000, 11)
    ext = np.array([s for k, s in enumerate(shape) if k != mode], dtype=np.int64)
    shp = np.array(shape, dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(ext)[:-1]]).astype(np.int64)
    g = skx.make_rng(4)
    coeffs = np.stack([np.concatenate([g.integers(0, 2 ** 31 - 1, 4, dtype=np.int64),
                                       g.integers(0, 2 ** 31 - 1, 5, dtype=np.int64)])
                       for _ in range(2)])
    dc = torch.from_numpy(np.ascontiguousarray(c.T.astype(np.int32))).cuda()
    dv = torch.from_numpy(v).cuda()
    tab = torch.empty(int(ext.sum()), dtype=torch.int32, device="cuda")
    assert lib.skx_ts_tables(2, ext.ctypes.data_as(vp), coeffs.ctypes.data_as(vp), m,
                             vp(tab.data_ptr()), None) == 0
    rec = torch.empty(2 * len(v), dtype=torch.float64, device="cuda")
    colptr = torch.empty(shape[mode] + 1, dtype=torch.int64, device="cuda")
    mask, ws_n = ctypes.c_uint32(0), ctypes.c_size_t(0)
    args = (shp.ctypes.data_as(vp), mode, len(v), vp(dc.data_ptr()), vp(dv.data_ptr()),
            vp(tab.data_ptr()), off.ctypes.data_as(vp), m, vp(rec.data_ptr()),
            vp(colptr.data_ptr()), ctypes.byref(mask))
    assert lib.skx_coo_fibre_ts(*args, None, ctypes.byref(ws_n), None) == 0
    ws = torch.empty(ws_n.value, dtype=torch.uint8, device="cuda")
    assert lib.skx_coo_fibre_ts(*args, vp(ws.data_ptr()), ctypes.byref(ws_n), None) == 0
    yt = torch.empty((shape[mode], m), dtype=torch.float64, device="cuda")
    assert lib.skx_ts_rhs_coo(2, shape[mode], vp(colptr.data_ptr()), vp(rec.data_ptr()),
                              vp(tab.data_ptr()), off.ctypes.data_as(vp), m, mask.value,
                              mask.value.bit_length(), vp(yt.data_ptr()), None) == 0
    torch.cuda.synchronize()
    # the same operator through the reference's own draw order and the oracle
    hs, ss = oracle.ts_tables(tuple(ext), m, oracle.generator(4))
    ref = oracle.ts_rhs(hs, ss, tuple(ext), m, oracle.unfold_t(oracle.Coo(shape, c, v), mode))
    assert np.array_equal(yt.cpu().numpy().T, ref)


def test_device_ingest_matches_host_lexsort(skx, monkeypatch):
    """SparseTensor(shape, coords, values) above DEVICE_INGEST_NNZ sorts and
    validates on the GPU: same arrays as the host
    np.lexsort path, same errors for duplicates and out-of-range coordinates."""
    from paper_2104_01101_b200 import tensors
    rng = np.random.default_rng(12)
    shape = (300, 200, 150)
    lin = rng.choice(int(np.prod(shape)), 50_000, replace=False)
    coords = np.stack(np.unravel_index(lin, shape), axis=1).astype(np.int64)
    vals = rng.standard_normal(len(lin))
    host = skx.SparseTensor(shape, coords, vals)          # below threshold: host lexsort
    monkeypatch.setattr(tensors, "DEVICE_INGEST_NNZ", 1000)
    dev = skx.SparseTensor(shape, coords, vals)
    assert dev._device is not None
    assert np.array_equal(dev.coords, host.coords) and np.array_equal(dev.values, host.values)
    bad = coords.copy()
    bad[7] = bad[3]
    with pytest.raises(ValueError, match="duplicate"):
        skx.SparseTensor(shape, bad, vals)
    bad = coords.copy()
    bad[5, 1] = shape[1]
    with pytest.raises(ValueError, match="out of range"):
        skx.SparseTensor(shape, bad, vals)


@pytest.mark.parametrize("m,r,w", [(1600, 100, 20), (400, 25, 15), (300, 128, 32), (40, 7, 7),
                                   (64, 33, 1)])
def test_assoc_mid_vs_lapack(skx, m, r, w):
    """libskx one-CTA middle step (two triangular solves + Householder QR) vs
    scipy/numpy on the same operands (src/linalg.py:105-110)."""
    import scipy.linalg
    import torch
    from paper_2104_01101_b200.linalg import assoc_mid_dev
    rng = np.random.default_rng(m + r + w)
    z = rng.standard_normal((m, r))
    qz, rz = np.linalg.qr(z)
    yg = rng.standard_normal((m, w))
    q, wm = assoc_mid_dev(torch.from_numpy(qz).cuda(), torch.from_numpy(rz).cuda(),
                          torch.from_numpy(yg).cuda())
    c = scipy.linalg.solve_triangular(rz, qz.T @ yg, lower=False)
    q_ref, _ = np.linalg.qr(c)
    wm_ref = qz @ scipy.linalg.solve_triangular(rz.T, q_ref, lower=True)
    q, wm = q.cpu().numpy(), wm.cpu().numpy()
    sgn = np.sign(np.sum(q * q_ref, axis=0))
    assert np.all(sgn != 0)
    assert relerr(q * sgn, q_ref) <= 1e-12
    assert relerr(wm * sgn, wm_ref) <= 1e-12
    assert np.abs(q.T @ q - np.eye(w)).max() <= 1e-13


@pytest.mark.parametrize("shape,nnz,mode", [((50, 40, 30), 20000, 0), ((50, 40, 30), 20000, 1),
                                            ((50, 40, 30), 20000, 2), ((12, 9, 7, 5), 3000, 2)])
def test_filter_fibers_matches_sorted_keys(skx, shape, nnz, mode):
    """One-pass fibre filter + gather == gather over the fully sorted key array
    (bit-exact), with repeated sampled fibres and empty ones."""
    import torch
    from paper_2104_01101_b200.sketching import filter_fibers_dev, gather_coo_dev
    from paper_2104_01101_b200.tensors import device_of
    rng = np.random.default_rng(nnz + mode)
    lin = rng.choice(int(np.prod(shape)), size=nnz, replace=False)
    coords = np.stack(np.unravel_index(np.sort(lin), shape), axis=1)
    st = skx.SparseTensor(shape, coords, rng.standard_normal(nnz))
    d = device_of(st)
    others = [k for k in range(len(shape)) if k != mode]
    m = 300
    idx = np.stack([rng.integers(0, shape[k], m) for k in others], axis=1)
    idx[m // 2:m // 2 + 20] = idx[:20]  # repeated fibres
    idx_d = torch.from_numpy(idx).cuda()
    w = torch.from_numpy(rng.random(m) + 0.5).cuda()
    ext = [shape[k] for k in others]
    keys, vals = d.keys(mode)
    ref = gather_coo_dev(keys, vals, ext, shape[mode], idx_d, w)
    fk, fv = filter_fibers_dev(d, mode, idx_d)
    got = gather_coo_dev(fk, fv, ext, shape[mode], idx_d, w)
    for a, b in zip(got, ref):
        assert torch.equal(a, b)
    assert got[2].numel() > 0


@pytest.mark.parametrize("nnz", [50_000, 3_000_000])
def test_rrf_stage1_fixed_point_paths_agree(skx, nnz):
    """RRF stage 1 three ways on one tensor: the ordered warp accumulation over
    a fibre layout, and the exact fixed-point accumulation straight from the
    COO (row-block bucketed above 2^20 nonzeros, direct below).  The two
    fixed-point results are exact sums rounded once, so they must agree bit
    for bit with each other across runs; the ordered float sums agree to
    rounding."""
    from paper_2104_01101_b200.sketching import draw_rrf_tables
    from paper_2104_01101_b200.tensors import device_of
    from paper_2104_01101_b200.tucker import rrf_stage1_dev
    shape = (3000, 2000, 1000)
    c, v = _coo_rand(shape, nnz, 7)
    st = skx.SparseTensor(shape, c, v)
    d = device_of(st)
    for n, k2 in ((1, 157), (2, 480)):
        P = int(np.prod(shape)) // shape[n]
        fx1 = rrf_stage1_dev(d, n, draw_rrf_tables(skx.make_rng(n), P, k2)).cpu().numpy()
        fx2 = rrf_stage1_dev(d, n, draw_rrf_tables(skx.make_rng(n), P, k2)).cpu().numpy()
        assert np.array_equal(fx1, fx2)
        d.fibre(n)  # with a layout the ordered float path runs
        fl = rrf_stage1_dev(d, n, draw_rrf_tables(skx.make_rng(n), P, k2)).cpu().numpy()
        d.drop_fibre(n)
        assert relerr(fx1, fl) <= 1e-14


@pytest.mark.parametrize("packed", [False, True])
def test_slice_hits_match_filter_gather(skx, packed):
    """Leverage gather of modes 1 / 2 from slices of the mode-0 layout equals
    the full-scan filter + key gather (repeated samples, empty fibres, a
    mode-0 layout carrying TensorSketch bits)."""
    import torch
    from paper_2104_01101_b200.sketching import (filter_fibers_dev, gather_coo_dev,
                                                 gather_slices_dev)
    from paper_2104_01101_b200.tensors import device_of
    shape = (60, 50, 40)
    c, v = _coo_rand(shape, 30000, 11)
    d = device_of(skx.SparseTensor(shape, c, v))
    if packed:
        op = skx.TensorSketchOp.build((50, 40), 64, skx.make_rng(3))
        d.fibre(0, op)
    g = np.random.default_rng(5)
    for n in (1, 2):
        ext = [shape[k] for k in range(3) if k != n]
        idx = np.stack([g.integers(0, ext[0], 500), g.integers(0, ext[1], 500)], axis=1)
        idx[7] = idx[3]  # a repeated sample
        idx_t = torch.from_numpy(idx).cuda()
        w = torch.from_numpy(g.uniform(size=500)).cuda()
        keys, vals = filter_fibers_dev(d, n, idx_t)
        o1, c1, v1 = gather_coo_dev(keys, vals, ext, shape[n], idx_t, w)
        o2, c2, v2 = gather_slices_dev(d, n, idx_t, w)
        assert torch.equal(o1, o2)
        assert torch.equal(c1, c2)
        assert torch.equal(v1, v2)


@pytest.mark.parametrize("shape,nnz,R", [((2000, 4000, 3000), 2_000_000, 20),
                                         ((50, 20000, 20000), 2_000_000, 20),
                                         ((3000, 2000, 20), 1_000_000, 20),
                                         ((200000, 200000, 200000), 20_000_000, 20),
                                         ((100000, 100000, 100000), 10_000_000, 10),
                                         ((3000, 500, 700), 300_000, 7)])
@pytest.mark.parametrize("k7_async", [False, True])
def test_tucker_cross_kernels_vs_einsum(skx, shape, nnz, R, k7_async, monkeypatch):
    """The sparse fitness cross term (K7 at R = 20: mode-1 rows by cp.async and
    mode-2 rows by TMA gather4 with zero-filled padding columns, or both by
    cp.async; register pipeline at R = 10; generic otherwise) against a
    chunked einsum, including a 20-row mode-2 factor (the whole TMA tensor),
    many short slices (config-5-like: ~100 nonzeros per slice, several
    pipelined batches each) and long ones."""
    import torch
    from paper_2104_01101_b200.synth import planted_cp_coo_device
    from paper_2104_01101_b200.tensors import device_of, tucker_cross_dev
    if k7_async:
        if R != 20:
            pytest.skip("the cp.async / TMA choice exists at R = 20 only")
        monkeypatch.setenv("SKX_K7_ASYNC", "1")  # mode-2 rows by cp.async instead of TMA
    coords, vals = planted_cp_coo_device(shape, nnz, rank=10, noise_sd=0.1, seed=1)
    d = device_of(skx.SparseTensor.from_device(shape, coords, vals, validate=False))
    g = torch.Generator(device="cuda").manual_seed(1)
    fac = [torch.linalg.qr(torch.randn(s, R, dtype=torch.float64, device="cuda", generator=g))[0]
           for s in shape]
    core = torch.randn(R, R, R, dtype=torch.float64, device="cuda", generator=g)
    got = float(tucker_cross_dev(d, core, fac))
    c, v = d.coords.long(), d.vals
    ref, mag = 0.0, 0.0
    for lo in range(0, d.nnz, 1 << 20):
        hi = min(d.nnz, lo + (1 << 20))
        t = torch.einsum("ea,abc->ebc", fac[0][c[0, lo:hi]], core)
        t = torch.einsum("ebc,eb->ec", t, fac[1][c[1, lo:hi]])
        per = v[lo:hi] * (t * fac[2][c[2, lo:hi]]).sum(1)
        ref += float(per.sum())
        mag += float(per.abs().sum())
    assert abs(got - ref) <= 1e-12 * mag, (got, ref, mag)


@pytest.mark.gpu
def test_fitness_kernels_concurrent_streams_bitwise(skx):
    """The per-sweep Tucker fitness (side stream) and Algorithm 6's final CP
    fitness (another stream) run concurrently in a config-5 call and share
    the entry points' scratch slot: each stream must get its own scratch, so
    the concurrent results equal the serial ones bit for bit."""
    import torch
    from paper_2104_01101_b200.synth import planted_cp_coo_device
    from paper_2104_01101_b200.tensors import cp_cross_dev, device_of, tucker_cross_dev
    shape = (100_000,) * 3
    coords, vals = planted_cp_coo_device(shape, 20_000_000, rank=10, noise_sd=0.1, seed=3)
    d = device_of(skx.SparseTensor.from_device(shape, coords, vals, validate=False))
    g = torch.Generator(device="cuda").manual_seed(3)
    fac = [torch.linalg.qr(torch.randn(s, 20, dtype=torch.float64, device="cuda", generator=g))[0]
           for s in shape]
    core = torch.randn(20, 20, 20, dtype=torch.float64, device="cuda", generator=g)
    cfac = [torch.randn(s, 10, dtype=torch.float64, device="cuda", generator=g) for s in shape]
    w = torch.rand(10, dtype=torch.float64, device="cuda", generator=g)
    t_ser = tucker_cross_dev(d, core, fac).clone()
    c_ser = cp_cross_dev(d, cfac, w).clone()
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(3):
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s1):
            t_con = tucker_cross_dev(d, core, fac)
        with torch.cuda.stream(s2):
            c_con = cp_cross_dev(d, cfac, w)
        torch.cuda.synchronize()
        outs.append((t_con.clone(), c_con.clone()))
    for t_con, c_con in outs:
        assert torch.equal(t_con, t_ser)
        assert torch.equal(c_con, c_ser)


@pytest.mark.parametrize("nnz", [50_000, 3_000_000])
def test_rrf_stage1_partitioned_bitwise(skx, nnz):
    """RRF stage 1 from row-block-partitioned records (skx_rrf_partition +
    skx_rrf_stage1_rec, the L2-resident form the leverage driver uses) is
    bitwise the direct fixed-point accumulation from the COO: the same
    integer sums, rounded once."""
    from paper_2104_01101_b200.sketching import draw_rrf_tables
    from paper_2104_01101_b200.tensors import device_of
    from paper_2104_01101_b200.tucker import rrf_partition_dev, rrf_stage1_dev
    shape = (3000, 2000, 1000)
    c, v = _coo_rand(shape, nnz, 11)
    d = device_of(skx.SparseTensor(shape, c, v))
    part = rrf_partition_dev(d, [1, 2])
    assert part is not None and sorted(part) == [1, 2]
    for n, k2 in ((1, 157), (2, 480)):
        P = int(np.prod(shape)) // shape[n]
        keys, vals = part[n]
        # every nonzero exactly once, grouped by row block
        rows = (keys >> 40).cpu().numpy()
        assert len(rows) == nnz and np.array_equal(np.bincount(rows, minlength=shape[n]),
                                                   np.bincount(c[:, n], minlength=shape[n]))
        direct = rrf_stage1_dev(d, n, draw_rrf_tables(skx.make_rng(n), P, k2)).cpu().numpy()
        viapart = rrf_stage1_dev(d, n, draw_rrf_tables(skx.make_rng(n), P, k2),
                                 part[n]).cpu().numpy()
        assert np.array_equal(direct, viapart)


@pytest.mark.parametrize("shape,nnz", [((100, 1 << 22, 1 << 24), 1_500_000), ((3000, 2000, 1000), 2_000_000)])
def test_compact_staging_roundtrip(skx, shape, nnz):
    """SparseTensor.from_sorted stages an order-3 COO as slice pointers plus
    one packed word per nonzero (i1 increment << b2 | i2, escapes for large
    increments: shape 1 has b2 = 24, so every increment >= 255 escapes); the
    device unpack restores the coordinates exactly, whole and in the
    slice-aligned chunks the leverage driver uploads."""
    import torch
    from paper_2104_01101_b200.tensors import DeviceCoo, compact3_aux_to_device, unpack_compact3
    c, v = _coo_rand(shape, nnz, 5)
    st = skx.SparseTensor.from_sorted(shape, c.astype(np.int64), v)
    assert st._c3 is not None
    if shape[2] == 1 << 24:
        assert st._c3["exc_idx"].numel() > 1000
    d = DeviceCoo.from_host(st)
    assert np.array_equal(d.coords.cpu().numpy().T.astype(np.int64), c)
    # slice-aligned pieces into one buffer
    c3 = st._c3
    aux = compact3_aux_to_device(c3)
    packed = c3["packed"].cuda()
    out = torch.full((3, nnz), -1, dtype=torch.int32, device="cuda")
    s0 = shape[0]
    cuts = [0, s0 // 3, s0 // 3 + 1, (2 * s0) // 3, s0]
    for a, b in zip(cuts[:-1], cuts[1:]):
        unpack_compact3(c3, nnz, out, a, b, packed, aux)
    assert np.array_equal(out.cpu().numpy().T.astype(np.int64), c)


@pytest.mark.parametrize("shape,nnz,R0", [((3000, 4000, 3000), 2_000_000, 20),
                                          ((2000, 1000, 1500), 1_000_000, 7),
                                          ((200000, 200000, 200000), 5_000_000, 20),
                                          ((50, 20000, 20000), 500_000, 20)])
def test_ttmc3_full_vs_cross_kernels(skx, shape, nnz, R0):
    """The full TTMc P (skx_tucker_ttmc3_r20) against a chunked einsum, and
    the cross terms taken from it -- Tucker <P, G>, CP <P, [[w; B_0, B_1,
    B_2]]> -- against the per-nonzero fitness kernels (K7, CP K7c)."""
    import torch
    from paper_2104_01101_b200.synth import planted_cp_coo_device
    from paper_2104_01101_b200.tensors import (cp_cross_dev, device_of, ttmc3_full_dev,
                                               tucker_cross_dev)
    coords, vals = planted_cp_coo_device(shape, nnz, rank=10, noise_sd=0.1, seed=2)
    d = device_of(skx.SparseTensor.from_device(shape, coords, vals, validate=False))
    g = torch.Generator(device="cuda").manual_seed(2)
    ranks = (R0, 20, 20)
    fac = [torch.linalg.qr(torch.randn(s, r, dtype=torch.float64, device="cuda", generator=g))[0]
           for s, r in zip(shape, ranks)]
    core = torch.randn(*ranks, dtype=torch.float64, device="cuda", generator=g)
    P = ttmc3_full_dev(d, fac)
    c, v = d.coords.long(), d.vals
    ref = torch.zeros(ranks, dtype=torch.float64, device="cuda")
    for lo in range(0, d.nnz, 1 << 20):
        hi = min(d.nnz, lo + (1 << 20))
        ref += torch.einsum("e,ea,eb,ec->abc", v[lo:hi], fac[0][c[0, lo:hi]],
                            fac[1][c[1, lo:hi]], fac[2][c[2, lo:hi]])
    assert float((P - ref).abs().max()) <= 1e-12 * float(ref.abs().max())
    cross = float((P * core).sum())
    kref = float(tucker_cross_dev(d, core, fac))
    assert abs(cross - kref) <= 1e-12 * float(ref.abs().sum() * core.abs().max()), (cross, kref)
    # CP model on the same factors: factors A_n B_n, weights w
    B = [torch.randn(r, 10, dtype=torch.float64, device="cuda", generator=g) for r in ranks]
    w = torch.rand(10, dtype=torch.float64, device="cuda", generator=g) + 0.5
    gp = torch.einsum("r,ar,br,cr->abc", w, B[0], B[1], B[2])
    cross_cp = float((P * gp).sum())
    cf = [(a @ b).contiguous() for a, b in zip(fac, B)]
    kcp = float(cp_cross_dev(d, cf, w))
    assert abs(cross_cp - kcp) <= 1e-11 * float(ref.abs().sum() * gp.abs().max()), (cross_cp, kcp)
