"""GPU: the drivers against fixtures from the real reference and the oracle.

Factors/core compared after sign canonicalisation at 1e-10 relative (f64);
1 - fitness within max(1e-10, reference floor)."""
import numpy as np
import pytest

from tests.conftest import canon, relerr
from tests.test_oracle_golden import DRIVERS, make_input

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def skx():
    import paper_2104_01101_b200 as m
    return m


def _as_api_input(skx, oracle, spec):
    t = make_input(oracle, spec)
    if isinstance(t, oracle.Coo):
        return skx.SparseTensor(t.shape, t.coords, t.values)
    return t


def _compare_model(model, trace, golden, tag, tol=1e-10):
    nd = len(model.factors)
    got_f, got_c = canon(model.factors, model.core)
    ref_f, ref_c = canon([golden[f"{tag}_a{k}"] for k in range(nd)], golden[f"{tag}_core"])
    for a, b in zip(got_f, ref_f):
        assert relerr(a, b) <= tol, (tag, relerr(a, b))
    assert relerr(got_c, ref_c) <= tol
    fr = golden[f"{tag}_fitness"]
    assert np.allclose(1 - np.array(trace.fitness), 1 - fr, rtol=1e-8, atol=1e-10), tag
    assert np.allclose(trace.residuals, golden[f"{tag}_residuals"], rtol=1e-9, atol=0), tag


@pytest.mark.parametrize("tag", list(DRIVERS))
def test_driver_vs_reference_golden(golden, oracle, skx, tag):
    spec, cfg = DRIVERS[tag]
    t = _as_api_input(skx, oracle, spec)
    model, trace = skx.sketched_tucker_als(t, skx.TuckerConfig(**cfg))
    _compare_model(model, trace, golden, tag)
    assert len(trace.wall_s) == cfg["max_sweeps"]


def test_driver_bitwise_deterministic(oracle, skx):
    for tag in ("dlev", "sts"):
        spec, cfg = DRIVERS[tag]
        t = _as_api_input(skx, oracle, spec)
        m1, t1 = skx.sketched_tucker_als(t, skx.TuckerConfig(**cfg))
        m2, t2 = skx.sketched_tucker_als(t, skx.TuckerConfig(**cfg))
        assert t1.fitness == t2.fitness
        assert t1.residuals == t2.residuals
        assert np.array_equal(m1.core, m2.core)
        for a, b in zip(m1.factors, m2.factors):
            assert np.array_equal(a, b)


def test_cp_via_tucker_vs_reference_golden(golden, skx):
    from paper_2104_01101_b200.synth import planted_cp_coo_host
    c, v = planted_cp_coo_host((30, 30, 30), 4000, rank=3, seed=5)
    st = skx.SparseTensor((30, 30, 30), c, v)
    cfg = skx.CPConfig(rank=3, sketch="leverage-random", sketch_factor=16, tucker_sweeps=3,
                       max_sweeps=10, seed=11)
    model, trace = skx.cp_via_sketched_tucker(st, cfg)
    assert trace.stage_split == int(golden["cpt_split"])
    assert np.allclose(trace.fitness, golden["cpt_fitness"], rtol=0, atol=1e-9)
    assert np.allclose(trace.residuals, golden["cpt_residuals"], rtol=1e-8, atol=0)
    for k in range(3):
        assert relerr(np.abs(model.factors[k]), np.abs(golden[f"cpt_a{k}"])) <= 1e-8
    assert relerr(np.abs(model.weights), np.abs(golden["cpt_w"])) <= 1e-8


def test_sketch_size_invariant_and_errors(skx):
    t = np.random.default_rng(0).standard_normal((10, 10, 10))
    with pytest.raises(ValueError):
        skx.sketched_tucker_als(t, skx.TuckerConfig(ranks=(3, 3, 3), sketch="tensorsketch", sketch_size=8))
    with pytest.raises(ValueError):
        skx.sketched_tucker_als(t, skx.TuckerConfig(ranks=(11, 3, 3), sketch="tensorsketch", sketch_size=99))
    with pytest.raises(ValueError):
        skx.sketched_tucker_als(t, skx.TuckerConfig(ranks=(3, 3, 3)))


@pytest.mark.parametrize("kind", ["tensorsketch", "leverage-random"])
def test_sparse_reduced_config_vs_oracle(oracle, skx, kind):
    """Reduced-scale configs 4/5: s=2000, 1e5 nonzeros."""
    from paper_2104_01101_b200.synth import planted_cp_coo_host
    shape = (2000, 2000, 2000)
    c, v = planted_cp_coo_host(shape, 100_000, rank=10, seed=0)
    st = skx.SparseTensor(shape, c, v)
    oc = oracle.Coo(shape, c, v)
    kw = dict(ranks=(10, 10, 10), max_sweeps=2, sketch=kind, sketch_size=1600, seed=0)
    model, trace = skx.sketched_tucker_als(st, skx.TuckerConfig(**kw))
    core, fac, tr = oracle.sketched_tucker(oc, **kw)
    # residuals are sketch-space quantities: compare directly
    assert np.allclose(trace.residuals, tr.residuals, rtol=1e-8), (trace.residuals, tr.residuals)
    assert np.allclose(trace.fitness, tr.fitness, rtol=0, atol=1e-9)


@pytest.mark.parametrize("sketch", ["tensorsketch", "leverage-random"])
@pytest.mark.parametrize("sparse", [False, True])
def test_speculative_sweep_replay_is_exact(skx, sparse, sketch, monkeypatch):
    """A flagged speculative sweep is replayed from its starting state on the
    checked path: forcing the flag on the first sub-problem of every sweep
    must give bitwise the same model and trace as the unforced run."""
    import torch
    from paper_2104_01101_b200 import linalg
    from paper_2104_01101_b200.synth import planted_cp_coo_host
    from paper_2104_01101_b200.tucker import sketched_tucker_als_dev
    shape = (60, 50, 40)
    if sparse:
        c, v = planted_cp_coo_host(shape, 20_000, rank=3, seed=2)
        t = skx.SparseTensor(shape, c, v)
    else:
        t = np.random.default_rng(2).standard_normal(shape)
    cfg = skx.TuckerConfig(ranks=(4, 5, 3), max_sweeps=3, sketch=sketch,
                           sketch_size=400, seed=9)
    core0, fac0, tr0 = sketched_tucker_als_dev(t, cfg)
    orig = linalg.sketch_qr_dev
    forced, seen = [], set()

    def forcing(z, defer=None):
        out = orig(z, defer)
        if defer is not None and id(defer) not in seen:  # first sub-problem of a sweep
            seen.add(id(defer))
            defer.append(torch.ones((), dtype=torch.bool, device="cuda"))
            forced.append(1)
        return out
    monkeypatch.setattr(linalg, "sketch_qr_dev", forcing)
    if sparse:
        t._device = None
    core1, fac1, tr1 = sketched_tucker_als_dev(t, cfg)
    assert len(forced) >= 3  # every sweep was flagged (and replayed)
    assert torch.equal(core0, core1)
    for a, b in zip(fac0, fac1):
        assert torch.equal(a, b)
    assert tr0.residuals == tr1.residuals and tr0.fitness == tr1.fitness


@pytest.mark.parametrize("sketch", ["tensorsketch", "leverage-random"])
@pytest.mark.parametrize("sparse", [False, True])
def test_side_stream_residuals_bitwise(skx, sparse, sketch, monkeypatch):
    """Sub-problem residuals computed on the low-priority side stream (beside
    the next sub-problem) equal the inline ones bit for bit, with and without
    forced replays of speculative sweeps; and at a config-4-like size where
    the side stream is the default."""
    import torch
    from paper_2104_01101_b200 import linalg, tucker
    from paper_2104_01101_b200.synth import planted_cp_coo_host
    from paper_2104_01101_b200.tucker import sketched_tucker_als_dev
    shape = (60, 50, 40)
    if sparse:
        c, v = planted_cp_coo_host(shape, 20_000, rank=3, seed=4)
        t = skx.SparseTensor(shape, c, v)
    else:
        t = np.random.default_rng(4).standard_normal(shape)
    cfg = skx.TuckerConfig(ranks=(4, 5, 3), max_sweeps=3, sketch=sketch, sketch_size=400, seed=5)

    def run(env_inline, force):
        if env_inline:
            monkeypatch.setenv("SKX_RESID_INLINE", "1")
        else:
            monkeypatch.delenv("SKX_RESID_INLINE", raising=False)
        monkeypatch.setattr(tucker, "RESID_SIDE_MIN", 0)
        orig = linalg.sketch_qr_dev
        seen = set()

        def forcing(z, defer=None):
            out = orig(z, defer)
            if force and defer is not None and id(defer) not in seen:
                seen.add(id(defer))
                defer.append(torch.ones((), dtype=torch.bool, device="cuda"))
            return out
        monkeypatch.setattr(linalg, "sketch_qr_dev", forcing)
        if sparse:
            t._device = None
        out = sketched_tucker_als_dev(t, cfg)
        monkeypatch.setattr(linalg, "sketch_qr_dev", orig)
        return out

    core0, fac0, tr0 = run(True, False)
    for force in (False, True):
        core1, fac1, tr1 = run(False, force)
        assert torch.equal(core0, core1)
        for a, b in zip(fac0, fac1):
            assert torch.equal(a, b)
        assert tr0.residuals == tr1.residuals and tr0.fitness == tr1.fitness
    if sparse and sketch == "tensorsketch":  # Y_n = 1600 x 4000 >= RESID_SIDE_MIN: default path
        monkeypatch.undo()
        shape = (4000, 4000, 4000)
        c, v = planted_cp_coo_host(shape, 400_000, rank=10, seed=6)
        st = skx.SparseTensor(shape, c, v)
        cfg = skx.TuckerConfig(ranks=(10, 10, 10), max_sweeps=2, sketch="tensorsketch",
                               sketch_size=1600, seed=6)
        assert 1600 * 4000 >= tucker.RESID_SIDE_MIN
        _, _, tr_side = sketched_tucker_als_dev(st, cfg)
        monkeypatch.setenv("SKX_RESID_INLINE", "1")
        st._device = None
        _, _, tr_inl = sketched_tucker_als_dev(st, cfg)
        assert tr_side.residuals == tr_inl.residuals


# ---- ttmc and exact HOOI (SURVEY 8b operator list, 8f rank 2) vs the reference
from tests.test_oracle_golden import HOOI, TTMC, ttmc_factors, ttmc_input  # noqa: E402


@pytest.mark.parametrize("tag", list(TTMC))
def test_ttmc_vs_reference_golden(golden, skx, tag):
    kind, shape, nnz, ranks, seed = TTMC[tag]
    x = ttmc_input(kind, shape, nnz, seed)
    t = x if kind == "dense" else skx.SparseTensor(shape, *x)
    fs = ttmc_factors(shape, ranks, seed)
    got = skx.ttmc(t, fs)
    assert got.shape == golden[f"{tag}_all"].shape
    assert relerr(got, golden[f"{tag}_all"]) <= 1e-13
    for n in range(len(shape)):
        got = skx.ttmc(t, fs, skip=n)
        ref = golden[f"{tag}_skip{n}"]
        assert got.shape == ref.shape
        # sparse order 3: same unfused products in the same order as the
        # reference; its np.add.reduceat sums differ only in the last bit
        assert relerr(got, ref) <= (1e-15 if kind == "sparse" and len(shape) == 3 else 1e-13)
    with pytest.raises(ValueError):
        skx.ttmc(t, fs, skip=len(shape))
    with pytest.raises(ValueError):
        skx.ttmc(t, [f[:-1] for f in fs], skip=0)


def test_ttmc_sparse_kernel_at_scale(skx, oracle):
    """libskx skip-mode TTMc on a larger COO tensor against the oracle."""
    from paper_2104_01101_b200.synth import planted_cp_coo_host
    shape = (300, 200, 250)
    c, v = planted_cp_coo_host(shape, 200_000, rank=4, seed=8)
    t = skx.SparseTensor(shape, c, v)
    ot = oracle.Coo(shape, c, v)
    g = np.random.default_rng(3)
    fs = [g.standard_normal((s, r)) for s, r in zip(shape, (7, 12, 9))]
    for n in range(3):
        assert relerr(skx.ttmc(t, fs, skip=n), oracle.ttmc(ot, fs, skip=n)) <= 1e-13


@pytest.mark.parametrize("tag", list(HOOI))
def test_hooi_vs_reference_golden(golden, oracle, skx, tag):
    spec, cfg = HOOI[tag]
    t = _as_api_input(skx, oracle, spec)
    model, trace = skx.hooi(t, skx.TuckerConfig(**cfg))
    _compare_model(model, trace, golden, tag)
    with pytest.raises(ValueError):
        skx.hooi(t, skx.TuckerConfig(ranks=cfg["ranks"], sketch="tensorsketch"))


def test_cp_via_tucker_hooi_stage_vs_reference_golden(golden, skx):
    from paper_2104_01101_b200.synth import planted_cp_coo_host
    c, v = planted_cp_coo_host((30, 30, 30), 4000, rank=3, seed=5)
    st = skx.SparseTensor((30, 30, 30), c, v)
    cfg = skx.CPConfig(rank=3, sketch=None, tucker_sweeps=3, max_sweeps=10, seed=12)
    model, trace = skx.cp_via_sketched_tucker(st, cfg)
    assert trace.stage_split == int(golden["cph_split"])
    assert np.allclose(trace.fitness, golden["cph_fitness"], rtol=0, atol=1e-9)
    assert np.allclose(trace.residuals, golden["cph_residuals"], rtol=1e-8, atol=1e-12)
    for k in range(3):
        assert relerr(np.abs(model.factors[k]), np.abs(golden[f"cph_a{k}"])) <= 1e-8
    assert relerr(np.abs(model.weights), np.abs(golden["cph_w"])) <= 1e-8


from tests.test_oracle_golden import SCP  # noqa: E402


@pytest.mark.parametrize("tag", list(SCP))
def test_sketched_cp_als_vs_reference_golden(golden, oracle, skx, tag):
    spec, cfg = SCP[tag]
    t = _as_api_input(skx, oracle, spec)
    model, trace = skx.sketched_cp_als(t, skx.CPConfig(**cfg))
    # column signs follow the RRF init's singular-vector signs (SVD convention):
    # the model is the same up to sign flips that cancel across modes
    for k in range(3):
        assert relerr(np.abs(model.factors[k]), np.abs(golden[f"{tag}_a{k}"])) <= 1e-8, (tag, k)
    assert relerr(np.abs(model.weights), np.abs(golden[f"{tag}_w"])) <= 1e-8
    assert np.allclose(trace.fitness, golden[f"{tag}_fitness"], rtol=0, atol=1e-9)
    assert np.allclose(trace.residuals, golden[f"{tag}_residuals"], rtol=1e-7, atol=1e-10)
    with pytest.raises(ValueError):
        skx.sketched_cp_als(t, skx.CPConfig(rank=3, sketch=None))


from tests.test_oracle_golden import DET  # noqa: E402


@pytest.mark.parametrize("tag,nf", [("ld2", 2), ("ld3", 3), ("ldz", 2)])
def test_lev_deterministic_indices_bit_exact(golden, skx, tag, nf):
    fs = [golden[f"{tag}_f{k}"] for k in range(nf)]
    m = golden[f"{tag}_idx"].shape[0]
    s = skx.lev_build(fs, m, "deterministic", skx.make_rng(0))
    assert np.array_equal(s.indices, golden[f"{tag}_idx"])
    assert np.array_equal(s.weights, np.ones(m))
    with pytest.raises(ValueError):
        skx.lev_build(fs, int(np.prod([f.shape[0] for f in fs])) + 1, "deterministic",
                      skx.make_rng(0))


def test_top_m_products_ties_vs_reference_golden(golden, skx):
    """Device best-first search (skx_top_m_products) vs the reference heap on
    score lists with zero / repeated scores (a candidate sort
    differs there)."""
    import torch
    from paper_2104_01101_b200.sketching import top_m_products_dev
    from tests.test_oracle_golden import _tm_cases
    for i, lists, want in _tm_cases(golden):
        got = top_m_products_dev([torch.from_numpy(x).cuda() for x in lists], want.shape[0])
        assert np.array_equal(got.cpu().numpy(), want), i


@pytest.mark.parametrize("tag", list(DET))
def test_deterministic_driver_vs_reference_golden(golden, oracle, skx, tag):
    t = _as_api_input(skx, oracle, DET[tag])
    model, trace = skx.sketched_tucker_als(t, skx.TuckerConfig(
        ranks=(3, 3, 3), max_sweeps=3, sketch="leverage-deterministic", sketch_size=120, seed=2))
    _compare_model(model, trace, golden, tag)


@pytest.mark.parametrize("tag", ["cpas", "cpad"])
def test_cp_als_vs_reference_golden(golden, skx, tag):
    """Exact CP-ALS (src/cp.py:102-174) on a sparse (device mttkrp, no atomics)
    and a dense tensor."""
    from paper_2104_01101_b200.synth import planted_cp_coo_host, planted_tucker_dense
    if tag == "cpas":
        c, v = planted_cp_coo_host((30, 30, 30), 3000, rank=3, seed=21)
        t = skx.SparseTensor((30, 30, 30), c, v)
    else:
        t = planted_tucker_dense((20, 18, 16), 3, 1e-2, 22)
    model, trace = skx.cp_als(t, skx.CPConfig(rank=3, max_sweeps=6, seed=23))
    for k in range(3):
        assert relerr(np.abs(model.factors[k]), np.abs(golden[f"{tag}_a{k}"])) <= 1e-8, k
    assert relerr(np.abs(model.weights), np.abs(golden[f"{tag}_w"])) <= 1e-8
    assert np.allclose(trace.fitness, golden[f"{tag}_fitness"], rtol=0, atol=1e-9)
    assert np.allclose(trace.residuals, golden[f"{tag}_residuals"], rtol=1e-8, atol=1e-10)


@pytest.mark.parametrize("sparse", [False, True])
@pytest.mark.parametrize("sketch", ["tensorsketch", "leverage-random"])
def test_early_stop_and_random_init_vs_oracle(skx, oracle, sparse, sketch):
    """convergence_tol > 0 (the non-pipelined speculative path: each sweep is
    verified before the fitness decides) and init="random" against the
    oracle: same number of sweeps, same model."""
    from paper_2104_01101_b200.synth import planted_cp_coo_host, planted_tucker_dense
    shape = (40, 36, 30)
    if sparse:
        c, v = planted_cp_coo_host(shape, 6000, rank=3, seed=4)
        t, tr_ = skx.SparseTensor(shape, c, v), oracle.Coo(shape, c, v)
    else:
        t = tr_ = planted_tucker_dense(shape, 3, 1e-2, 4)
    for init, tol in (("rrf", 1e-4), ("random", 0.0)):
        cfg = dict(ranks=(3, 3, 3), max_sweeps=8, sketch=sketch, sketch_size=200, seed=6,
                   init=init, convergence_tol=tol)
        model, trace = skx.sketched_tucker_als(t, skx.TuckerConfig(**cfg))
        core, fac, otr = oracle.sketched_tucker(tr_, (3, 3, 3), sketch, max_sweeps=8,
                                                sketch_size=200, seed=6, init=init, tol=tol)
        assert len(trace.fitness) == len(otr.fitness)
        gf, gc = canon(model.factors, model.core)
        rf, rc = canon(fac, core)
        for a, b in zip(gf, rf):
            assert relerr(a, b) <= 1e-9
        assert relerr(gc, rc) <= 1e-9


REFTS = {
    "rtsd": (("dense", (20, 18, 16), 3, 1e-2, 41), dict(seed=3)),
    "rtss": (("sparse", (30, 30, 30), 4000, 42), dict(seed=4)),
    "rtdr": (("dense", (20, 18, 16), 3, 1e-2, 41), dict(seed=3, init="random")),
    "rtsr": (("sparse", (30, 30, 30), 4000, 42), dict(seed=4, init="random")),
}


@pytest.mark.parametrize("tag", list(REFTS))
def test_ref_tucker_ts_vs_reference_golden(golden, oracle, skx, tag):
    """The one-variable TensorSketch baseline (src/tucker.py:303-364), through
    harness.run_single('ref-ts').  Unlike the rank-constrained driver it is
    not sign-equivariant: each factor is re-orthonormalised by QR while the
    core stays fixed, so the column signs of the initial factors steer the
    trajectory.  Random init (Q of a Gaussian, numpy's Householder signs
    reproduced by qr_lapack_dev) matches the reference to 1e-9; with RRF init
    the reference's factor signs come from LAPACK's gesdd, an unspecified
    convention, so those runs are checked on the fitness only."""
    from paper_2104_01101_b200 import harness
    spec, extra = REFTS[tag]
    cfg = dict(ranks=(3, 3, 3), max_sweeps=3, sketch="tensorsketch", sketch_size=200, **extra)
    t = _as_api_input(skx, oracle, spec)
    model, trace, m = harness.run_single(t, "ref-ts", skx.TuckerConfig(**cfg))
    assert m == 200
    if extra.get("init") == "random":
        _compare_model(model, trace, golden, tag, tol=1e-9)
    else:
        assert np.allclose(trace.fitness, golden[f"{tag}_fitness"], rtol=0, atol=0.1)
        assert len(trace.residuals) == len(golden[f"{tag}_residuals"])


def test_config5_shape_run_bitwise_deterministic(skx):
    """A config-5-shaped run (5e4^3, R = 20, leverage m = 6400, short
    fitness slices, fixed-point RRF) twice: bitwise identical model and
    trace (no race in the cp.async-staged fitness or the atomics)."""
    from paper_2104_01101_b200.synth import planted_cp_coo_device
    shape = (50_000,) * 3  # ~50 sampled-fibre hits per sub-problem: rank 20 is reachable
    coords, vals = planted_cp_coo_device(shape, 20_000_000, rank=10, noise_sd=0.1, seed=2)
    st = skx.SparseTensor.from_device(shape, coords, vals, validate=False)
    cfg = skx.CPConfig(rank=10, tucker_rank=20, sketch="leverage-random", sketch_factor=16,
                       tucker_sweeps=2, max_sweeps=10, seed=0)
    m1, t1 = skx.cp_via_sketched_tucker(st, cfg)
    st._device.release_layouts()
    m2, t2 = skx.cp_via_sketched_tucker(st, cfg)
    assert t1.fitness == t2.fitness and t1.residuals == t2.residuals
    assert np.array_equal(m1.weights, m2.weights)
    for a, b in zip(m1.factors, m2.factors):
        assert np.array_equal(a, b)


def test_fixed_capacity_hits_path_matches(skx, monkeypatch):
    """Speculative leverage sweeps on a sparse tensor take the sync-free
    fixed-capacity hit lists (no host read of hit counts, distinct columns by
    a device sort, segment sums) when the sampled right-hand side is large;
    forced here on a small tensor, it must reproduce the host-sized path to
    rounding, and a capacity overflow must fall back (replay) to it exactly."""
    import numpy as np
    from paper_2104_01101_b200 import sketching, tucker
    from paper_2104_01101_b200.synth import planted_cp_coo_host
    from tests.conftest import canon, relerr
    shape = (150, 120, 90)
    c, v = planted_cp_coo_host(shape, 60_000, rank=3, seed=2)
    st = skx.SparseTensor(shape, c, v)
    # ranks 5 x 5 x 5: r = 25 > R + 10 = 15, the associated rsvd form
    cfg = skx.TuckerConfig(ranks=(5, 5, 5), max_sweeps=3, sketch="leverage-random",
                           sketch_size=900, seed=8)
    monkeypatch.setattr(tucker, "FORCE_FIXED_HITS", False)
    m0, t0 = skx.sketched_tucker_als(st, cfg)
    f0, c0 = canon(m0.factors, m0.core)
    for cap in (1 << 12, 8):  # 8: every sub-problem overflows -> checked replay
        monkeypatch.setattr(tucker, "FORCE_FIXED_HITS", True)
        monkeypatch.setattr(sketching, "HITS_CAP", cap)
        m1, t1 = skx.sketched_tucker_als(st, cfg)
        f1, c1 = canon(m1.factors, m1.core)
        for a, b in zip(f1, f0):
            assert relerr(a, b) <= 1e-10
        assert relerr(c1, c0) <= 1e-10
        assert np.allclose(t1.fitness, t0.fitness, rtol=0, atol=1e-12)
        assert np.allclose(t1.residuals, t0.residuals, rtol=1e-9)
