"""GPU parity on every BASELINE.json configuration against fixtures made by
running the REAL reference (tests/golden/make_golden_configs.py ->
tests/golden/configs.npz).

* config 2 (dense 400^3, leverage-random, m = 3200, 10 sweeps) and config 3
  (dense 120^4, TensorSketch m = 4096, r = 512 -> the r > 128 sketched-QR
  branch) at their full size;
* configs 4 (TensorSketch) and 5 (Algorithm 6: leverage Tucker rank 20 ->
  CP rank 10 on the core, 50 core sweeps) at SURVEY 8(c)'s reduced scales
  2000^3 / 1e6 and 1e4^3 / 1e7 nonzeros.

Contracts: leverage index sets and sparse TensorSketch right-hand
sides bit-exact (sha256 of the bytes), dense right-hand sides <= 1e-12
Frobenius-relative (seeded projection), factors / core <= 1e-10 after sign
canonicalisation where the spectrum is low-rank (configs 2, 3), residuals and
1 - fitness to the stated tolerances.
"""
import hashlib
import os

import numpy as np
import pytest

from tests.conftest import ROOT, canon, relerr

pytestmark = pytest.mark.gpu

PROJ_SEED = 20260101
CFG_PATH = os.path.join(ROOT, "tests", "golden", "configs.npz")


@pytest.fixture(scope="module")
def cg():
    return dict(np.load(CFG_PATH))


@pytest.fixture(scope="module")
def skx():
    import paper_2104_01101_b200 as m
    return m


def proj_matrix(rows, k, salt):
    return np.random.default_rng([PROJ_SEED, rows, k, salt]).standard_normal((rows, k))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_input(skx, spec):
    from paper_2104_01101_b200.synth import planted_cp_coo_host, planted_tucker_dense
    if spec[0] == "dense":
        _, shape, r, noise, seed = spec
        return planted_tucker_dense(shape, r, noise, seed)
    _, shape, nnz, seed = spec
    c, v = planted_cp_coo_host(shape, nnz, rank=10, seed=seed)
    return skx.SparseTensor(shape, c, v)


CASES = {
    "c2": (("dense", (400,) * 3, 10, 1e-2, 0),
           dict(ranks=(10,) * 3, max_sweeps=10, sketch="leverage-random", sketch_size=3200, seed=0)),
    "c3": (("dense", (120,) * 4, 8, 1e-3, 0),
           dict(ranks=(8,) * 4, max_sweeps=10, sketch="tensorsketch", sketch_size=4096, seed=0)),
    "c4a": (("sparse", (2000,) * 3, 1_000_000, 0),
            dict(ranks=(10,) * 3, max_sweeps=5, sketch="tensorsketch", sketch_size=1600, seed=0)),
    "c4b": (("sparse", (10_000,) * 3, 10_000_000, 0),
            dict(ranks=(10,) * 3, max_sweeps=5, sketch="tensorsketch", sketch_size=1600, seed=0)),
    "c5a": (("sparse", (2000,) * 3, 1_000_000, 0),
            dict(rank=10, tucker_rank=20, sketch="leverage-random", sketch_factor=16,
                 tucker_sweeps=5, max_sweeps=50, seed=0)),
    "c5b": (("sparse", (10_000,) * 3, 10_000_000, 0),
            dict(rank=10, tucker_rank=20, sketch="leverage-random", sketch_factor=16,
                 tucker_sweeps=5, max_sweeps=50, seed=0)),
}


class Recorder:
    """Observes the driver's TensorSketch right-hand sides and leverage
    samples (the package functions are wrapped, not changed)."""

    def __init__(self, monkeypatch):
        from paper_2104_01101_b200 import tucker
        self.rhs, self.lev = [], []
        rec = self
        orig_rhs = tucker._Run._rhs
        orig_lev = tucker.lev_sample_dev

        def rhs(run, n, op):
            yt = orig_rhs(run, n, op)
            rec.rhs.append(yt.t().contiguous().cpu().numpy())  # reference layout m x s_n
            return yt

        def lev(factors, m, gen, check=True):
            out = orig_lev(factors, m, gen, check=check)
            rec.lev.append((out[0].cpu().numpy().astype(np.int64), out[1].cpu().numpy()))
            return out

        monkeypatch.setattr(tucker._Run, "_rhs", rhs)
        monkeypatch.setattr(tucker, "lev_sample_dev", lev)


def _factor_check(cg, key, got, tol):
    if key in cg:
        assert relerr(got, cg[key]) <= tol, (key, relerr(got, cg[key]))
    else:
        assert relerr(got[:256], cg[key + "_head"]) <= tol, (key, relerr(got[:256], cg[key + "_head"]))
        pj = got.T @ proj_matrix(got.shape[0], 8, 1)
        assert relerr(pj, cg[key + "_proj"]) <= tol, (key, relerr(pj, cg[key + "_proj"]))


def _check_rhs(cg, tag, rec, exact):
    n = int(cg[f"{tag}_n_rhs"])
    assert len(rec.rhs) == n
    for i, y in enumerate(rec.rhs):
        if exact:  # sparse: numpy add.at order, bit for bit
            assert sha(y) == str(cg[f"{tag}_rhs{i}_sha"]), (tag, i)
        pj = y @ proj_matrix(y.shape[1], 4, 2)
        assert relerr(pj, cg[f"{tag}_rhs{i}_proj"]) <= 1e-12, (tag, i)
        assert abs(np.linalg.norm(y) - float(cg[f"{tag}_rhs{i}_norm"])) <= 1e-13 * float(
            cg[f"{tag}_rhs{i}_norm"])


def _check_lev(cg, tag, rec):
    n = int(cg[f"{tag}_n_lev"])
    assert len(rec.lev) == n, (len(rec.lev), n)
    assert np.array_equal(rec.lev[0][0], cg[f"{tag}_lev0_idx"])
    for i, (idx, w) in enumerate(rec.lev):
        assert sha(idx) == str(cg[f"{tag}_lev{i}_sha"]), (tag, i)
        # weights 1/sqrt(m prod p) follow the factors' rounding (the index
        # sets above are the bit-exact contract)
        assert abs(w.sum() - float(cg[f"{tag}_lev{i}_wsum"])) <= 1e-8 * abs(
            float(cg[f"{tag}_lev{i}_wsum"]))


@pytest.mark.parametrize("tag", ["c2", "c3"])
def test_dense_config_full_size_vs_reference(cg, skx, monkeypatch, tag):
    spec, cfg = CASES[tag]
    t = make_input(skx, spec)
    rec = Recorder(monkeypatch)
    model, trace = skx.sketched_tucker_als(t, skx.TuckerConfig(**cfg))
    if cfg["sketch"] == "tensorsketch":
        _check_rhs(cg, tag, rec, exact=False)
    else:
        _check_lev(cg, tag, rec)
    nd = len(model.factors)
    gf, gc = canon(model.factors, model.core)
    for k in range(nd):
        _factor_check(cg, f"{tag}_a{k}", gf[k], 1e-10)
    assert relerr(gc, cg[f"{tag}_core"]) <= 1e-10
    # 1 - fitness: max(1e-10, 10x the reference's own 1-vs-N-BLAS-thread
    # spread), which is 3e-9 on config 3
    tol = 3e-8 if tag == "c3" else 1e-10
    assert np.allclose(1 - np.array(trace.fitness), 1 - cg[f"{tag}_fitness"], rtol=0, atol=tol)
    assert np.allclose(trace.residuals, cg[f"{tag}_residuals"], rtol=1e-9, atol=0)


@pytest.mark.parametrize("tag", ["c4a", "c4b"])
def test_config4_reduced_vs_reference(cg, skx, monkeypatch, tag):
    spec, cfg = CASES[tag]
    t = make_input(skx, spec)
    rec = Recorder(monkeypatch)
    model, trace = skx.sketched_tucker_als(t, skx.TuckerConfig(**cfg))
    _check_rhs(cg, tag, rec, exact=True)
    res, want = np.array(trace.residuals), cg[f"{tag}_residuals"]
    # first sub-problem: identical inputs up to the RRF factors' rounding
    assert abs(res[0] - want[0]) <= 1e-12 * want[0]
    assert np.allclose(res, want, rtol=1e-9, atol=0)
    assert np.allclose(trace.fitness, cg[f"{tag}_fitness"], rtol=0, atol=1e-10)
    # the factors of these non-low-rank tensors (fitness < 0: 1e6 samples of a
    # 2000^3 CP model) sit in a noise-dominated spectrum with tiny singular
    # gaps, which amplifies rounding differences by ~1e8 over 5 sweeps
    # (subspace comparisons only where the gap permits); the
    # sketch-space quantities above carry the tight contract
    gf, gc = canon(model.factors, model.core)
    for k in range(3):
        _factor_check(cg, f"{tag}_a{k}", gf[k], 1e-6)
    assert relerr(gc, cg[f"{tag}_core"]) <= 1e-6


@pytest.mark.parametrize("tag", ["c5a", "c5b"])
def test_config5_alg6_reduced_vs_reference(cg, skx, oracle, monkeypatch, tag):
    """Algorithm 6 at config 5's parameters.  Tucker stage vs the reference:
    every leverage index set bit-exact, Tucker fitness / residuals tight.
    The Tucker core of this noise-dominated reduced tensor (fitness ~ 0)
    carries ~1e-8 relative rounding drift (factors in a spectrum without
    gaps), which 50 CP-ALS sweeps on the core amplify further; so the core
    stage (K8) and the composition are checked against the oracle run on the
    device's own Tucker output at 1e-8, and against the reference's final
    numbers at the drift-limited tolerance."""
    from paper_2104_01101_b200 import cp as cpmod
    spec, cfg = CASES[tag]
    if f"{tag}_fitness" not in cg:
        pytest.skip(f"{tag} fixture not generated")
    t = make_input(skx, spec)
    rec = Recorder(monkeypatch)
    seen = {}
    orig = cpmod.sketched_tucker_run_dev

    def tucker(*a, **k):
        core, fac, finish = orig(*a, **k)
        seen["core"] = core.cpu().numpy()
        seen["fac"] = [f.cpu().numpy() for f in fac]

        def fin():
            seen["trace"] = finish()
            return seen["trace"]
        fin.last_ttmc = finish.last_ttmc  # the last pass's full TTMc (final CP fitness)
        return core, fac, fin

    monkeypatch.setattr(cpmod, "sketched_tucker_run_dev", tucker)
    model, trace = skx.cp_via_sketched_tucker(t, skx.CPConfig(**cfg))
    _check_lev(cg, tag, rec)
    assert trace.stage_split == int(cg[f"{tag}_split"])
    assert np.allclose(seen["trace"].fitness, cg[f"{tag}_tucker_fitness"], rtol=0, atol=1e-10)
    res = np.array(seen["trace"].residuals)
    want = cg[f"{tag}_tucker_residuals"]
    rel = np.abs(res - want) / want
    # first sub-problem: same inputs up to the RRF factors' rounding; later ones
    # inherit the factor drift of this gap-free spectrum (see the docstring)
    assert rel[0] <= 1e-10, rel
    assert rel.max() <= 1e-6, rel
    gf, gc = canon(seen["fac"], seen["core"])
    assert relerr(gc, cg[f"{tag}_core"]) <= 1e-6
    # core stage + composition vs the oracle on the same Tucker output
    A, w, ctr = oracle.cp_on_core(seen["core"], cfg["rank"], sweeps=cfg["max_sweeps"])
    assert np.allclose(trace.residuals, ctr.residuals, rtol=1e-8, atol=1e-10)
    want_w = w.copy()
    for k in range(3):
        u = seen["fac"][k] @ A[k]
        nrm = np.linalg.norm(u, axis=0)
        want_w = want_w * nrm
        assert relerr(np.abs(model.factors[k]), np.abs(u / np.where(nrm > 0, nrm, 1.0))) <= 1e-8
    assert relerr(model.weights, want_w) <= 1e-8
    # against the reference's final numbers
    assert np.allclose(trace.fitness, cg[f"{tag}_fitness"], rtol=0, atol=1e-9)
    assert np.allclose(trace.residuals, cg[f"{tag}_residuals"], rtol=1e-5, atol=0)
    assert relerr(model.weights, cg[f"{tag}_cp_w"]) <= 1e-4


def test_config5_chunked_host_upload_is_exact(cg, skx, monkeypatch):
    """Algorithm 6 from a HOST COO (the public-API path the e2e bench times):
    the tensor is uploaded in chunks and the range-finder sketches accumulate
    each chunk as it lands.  Exact fixed-point sums make the result bitwise
    identical to the device-resident run, and the leverage index sets match
    the reference."""
    from paper_2104_01101_b200 import tucker
    from paper_2104_01101_b200.synth import planted_cp_coo_host
    spec, cfg = CASES["c5b"]
    _, shape, nnz, seed = spec
    c, v = planted_cp_coo_host(shape, nnz, rank=10, seed=seed)
    monkeypatch.setattr(tucker, "UPLOAD_CHUNK", 1 << 21)  # 5 chunks
    rec = Recorder(monkeypatch)
    host = skx.SparseTensor.from_sorted(shape, c, v)
    m1, t1 = skx.cp_via_sketched_tucker(host, skx.CPConfig(**cfg))
    _check_lev(cg, "c5b", rec)
    dev = skx.SparseTensor(shape, c, v)  # device ingest: one-shot path
    m2, t2 = skx.cp_via_sketched_tucker(dev, skx.CPConfig(**cfg))
    assert t1.fitness == t2.fitness and t1.residuals == t2.residuals
    assert np.array_equal(m1.weights, m2.weights)
    for a, b in zip(m1.factors, m2.factors):
        assert np.array_equal(a, b)
