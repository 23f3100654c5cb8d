"""Pin the CPU oracle (oracle/sketchals_port.py) against golden fixtures made
by running the real reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest
import scipy.sparse as sp

from paper_2104_01101_b200.synth import planted_cp_coo_host, planted_tucker_dense
from tests.conftest import canon, relerr


def gen(seed):
    from oracle.sketchals_port import generator
    return generator(seed)


def test_ts_tables_bit_exact(golden, oracle):
    for seed in (0, 7):
        hs, ss = oracle.ts_tables((100, 120, 90), 400, gen(seed))
        for k in range(3):
            assert np.array_equal(hs[k], golden[f"ts_tab_s{seed}_h{k}"])
            assert np.array_equal(ss[k], golden[f"ts_tab_s{seed}_s{k}"])
    hs, ss = oracle.ts_tables((3, 4, 2), 5, gen(7))
    for k in range(3):
        assert np.array_equal(hs[k], golden[f"ts_small_h{k}"])
        assert np.array_equal(ss[k], golden[f"ts_small_s{k}"])


def test_rrf_tables_bit_exact(golden, oracle):
    h, s, g = oracle.rrf_tables(1000, 20, 45, gen(3))
    assert np.array_equal(h, golden["rrf_hash"])
    assert np.array_equal(s, golden["rrf_signs"])
    assert np.array_equal(g, golden["rrf_gauss"])


def test_leverage_sample_indices_bit_exact(golden, oracle):
    f = [golden["lev_f0"], golden["lev_f1"]]
    idx, w, _ = oracle.lev_sample(f, 200, gen(9))
    assert np.array_equal(idx, golden["lev_idx"])
    assert np.allclose(w, golden["lev_w"], rtol=1e-14, atol=0)


def test_ts_rhs(golden, oracle):
    hs, ss = oracle.ts_tables((6, 5), 16, gen(1))
    out = oracle.ts_rhs(hs, ss, (6, 5), 16, golden["rhs_b"])
    assert relerr(out, golden["rhs_dense"]) <= 1e-15
    outs = oracle.ts_rhs(hs, ss, (6, 5), 16, sp.csr_matrix(golden["rhs_bs"]))
    assert relerr(outs, golden["rhs_sparse"]) <= 1e-15


@pytest.mark.parametrize("m,ext", [(3, (4, 4)), (8, (4, 4)), (16, (5, 3, 4)),
                                   (64, (5, 3, 4)), (400, (30, 20))])
def test_ts_kron(golden, oracle, m, ext):
    hs, ss = oracle.ts_tables(ext, m, gen(200 + m))
    fs = [golden[f"kron_m{m}_f{k}"] for k in range(len(ext))]
    assert relerr(oracle.ts_kron(hs, ss, ext, m, fs), golden[f"kron_m{m}"]) <= 1e-14


def test_composite(golden, oracle):
    h, s, g = oracle.rrf_tables(50, 4, 20, gen(4))
    mat = golden["comp_mat"]
    assert relerr(oracle.rrf_apply(mat, h, s, g, 20), golden["comp_dense"]) <= 1e-14
    ms = sp.csr_matrix(mat * (np.abs(mat) > 0.8))
    assert relerr(oracle.rrf_apply(ms, h, s, g, 20), golden["comp_sparse"]) <= 1e-14


def test_lev_apply(golden, oracle):
    f = [golden["levapp_f0"], golden["levapp_f1"]]
    idx, w, _ = oracle.lev_sample(f, 30, gen(12))
    assert np.array_equal(idx, golden["levapp_idx"])
    bt = golden["levapp_bt"]
    z, y = oracle.lev_rows(idx, w, (8, 6), f, bt)
    assert relerr(z, golden["levapp_z"]) <= 1e-15
    assert relerr(y, golden["levapp_y"]) <= 1e-15
    _, ys = oracle.lev_rows(idx, w, (8, 6), f, sp.csr_matrix(bt * (np.abs(bt) > 1.0)))
    assert relerr(ys, golden["levapp_ys"]) <= 1e-15


def test_rsvd_lrls(golden, oracle):
    ct, v = oracle.rsvd_lrls(golden["rsvd_z"], golden["rsvd_y"], 2, gen(2))
    assert relerr(ct @ v.T, golden["rsvd_core_t"] @ golden["rsvd_v"].T) <= 1e-13
    assert relerr(np.abs(v), np.abs(golden["rsvd_v"])) <= 1e-12


def test_init_rrf(golden, oracle):
    u = oracle.init_rrf(golden["rrf_tn"], 4, 8, gen(6))
    a, _ = canon([u])
    b, _ = canon([golden["rrf_u"]])
    assert relerr(a[0], b[0]) <= 1e-12


def test_fitness(golden, oracle):
    t = golden["fit_t"]
    fs = [golden[f"fit_a{k}"] for k in range(3)]
    assert oracle.fitness_tucker(t, golden["fit_core"], fs) == pytest.approx(
        float(golden["fit_dense"]), abs=1e-14)
    tsp = t * (np.abs(t) > 0.7)
    c = np.argwhere(tsp != 0)
    st = oracle.Coo(t.shape, c, tsp[tuple(c.T)])
    assert oracle.fitness_tucker(st, golden["fit_core"], fs) == pytest.approx(
        float(golden["fit_sparse"]), abs=1e-14)
    cpf = [golden[f"fitcp_a{k}"] for k in range(3)]
    w = golden["fitcp_w"]
    assert oracle.fitness_cp(t, cpf, w) == pytest.approx(float(golden["fitcp_dense"]), abs=1e-14)
    assert oracle.fitness_cp(st, cpf, w) == pytest.approx(float(golden["fitcp_sparse"]), abs=1e-14)


DRIVERS = {
    "cfg1": (("dense", (100, 100, 100), 5, 1e-2, 0),
             dict(ranks=(5, 5, 5), max_sweeps=5, sketch="tensorsketch", sketch_factor=16, seed=0)),
    "dlev": (("dense", (30, 30, 30), 3, 1e-2, 1),
             dict(ranks=(3, 3, 3), max_sweeps=3, sketch="leverage-random", sketch_size=144, seed=0)),
    "d4ts": (("dense", (12, 12, 12, 12), 2, 1e-3, 2),
             dict(ranks=(2, 2, 2, 2), max_sweeps=3, sketch="tensorsketch", sketch_size=64, seed=0)),
    "sts": (("sparse", (40, 40, 40), 3000, 3),
            dict(ranks=(4, 4, 4), max_sweeps=3, sketch="tensorsketch", sketch_size=256, seed=0)),
    "slev": (("sparse", (40, 40, 40), 3000, 4),
             dict(ranks=(4, 4, 4), max_sweeps=3, sketch="leverage-random", sketch_size=256, seed=0)),
}


def make_input(oracle, spec):
    if spec[0] == "dense":
        _, shape, r, noise, seed = spec
        return planted_tucker_dense(shape, r, noise, seed)
    _, shape, nnz, seed = spec
    c, v = planted_cp_coo_host(shape, nnz, rank=3, seed=seed)
    return oracle.Coo(shape, c, v)


@pytest.mark.parametrize("tag", list(DRIVERS))
def test_sketched_tucker_driver(golden, oracle, tag):
    spec, cfg = DRIVERS[tag]
    t = make_input(oracle, spec)
    core, fac, tr = oracle.sketched_tucker(t, **cfg)
    nd = len(fac)
    got_f, got_c = canon(fac, core)
    ref_f, ref_c = canon([golden[f"{tag}_a{k}"] for k in range(nd)], golden[f"{tag}_core"])
    for a, b in zip(got_f, ref_f):
        assert relerr(a, b) <= 1e-10
    assert relerr(got_c, ref_c) <= 1e-10
    fr = golden[f"{tag}_fitness"]
    assert np.allclose(1 - np.array(tr.fitness), 1 - fr, rtol=1e-9, atol=1e-12)
    assert np.allclose(tr.residuals, golden[f"{tag}_residuals"], rtol=1e-10, atol=0)


def test_cp_via_tucker(golden, oracle):
    c, v = planted_cp_coo_host((30, 30, 30), 4000, rank=3, seed=5)
    st = oracle.Coo((30, 30, 30), c, v)
    fac, w, tr, _ = oracle.cp_via_tucker(st, 3, tucker_sweeps=3, cp_sweeps=10,
                                         sketch_factor=16, seed=11)
    assert tr.stage_split == int(golden["cpt_split"])
    assert np.allclose(tr.fitness, golden["cpt_fitness"], rtol=0, atol=1e-10)
    assert np.allclose(tr.residuals, golden["cpt_residuals"], rtol=1e-9, atol=0)
    for k in range(3):
        assert relerr(np.abs(fac[k]), np.abs(golden[f"cpt_a{k}"])) <= 1e-9
    assert relerr(np.abs(w), np.abs(golden["cpt_w"])) <= 1e-9


# ---- ttmc, HOOI, CP via exact-HOOI compression
TTMC = {
    "ttd3": ("dense", (6, 5, 4), None, (2, 3, 2), 21),
    "tts3": ("sparse", (15, 12, 10), 300, (3, 2, 4), 22),
    "ttd4": ("dense", (5, 4, 3, 4), None, (2, 2, 3, 2), 23),
    "tts4": ("sparse", (8, 7, 6, 5), 200, (2, 3, 2, 2), 24),
}
HOOI = {
    "hooid": (("dense", (30, 30, 30), 3, 1e-2, 1), dict(ranks=(3, 3, 3), max_sweeps=4, seed=0)),
    "hoois": (("sparse", (40, 40, 40), 3000, 3), dict(ranks=(4, 4, 4), max_sweeps=3, seed=0)),
    "hooir": (("dense", (20, 18, 16), 2, 1e-2, 6),
              dict(ranks=(2, 3, 2), max_sweeps=3, init="random", seed=5)),
}


def ttmc_input(kind, shape, nnz, seed):
    """(dense array | (coords, values)) as tests/golden/make_golden.py draws them."""
    g = np.random.default_rng(seed)
    if kind == "dense":
        return g.standard_normal(shape)
    lin = np.sort(g.choice(int(np.prod(shape)), size=nnz, replace=False))
    return np.stack(np.unravel_index(lin, shape), axis=1), g.standard_normal(nnz)


def ttmc_factors(shape, ranks, seed):
    g = np.random.default_rng(seed + 100)
    return [g.standard_normal((s, r)) for s, r in zip(shape, ranks)]


@pytest.mark.parametrize("tag", list(TTMC))
def test_ttmc(golden, oracle, tag):
    kind, shape, nnz, ranks, seed = TTMC[tag]
    x = ttmc_input(kind, shape, nnz, seed)
    t = x if kind == "dense" else oracle.Coo(shape, *x)
    fs = ttmc_factors(shape, ranks, seed)
    assert relerr(oracle.ttmc(t, fs), golden[f"{tag}_all"]) <= 1e-13
    for n in range(len(shape)):
        assert relerr(oracle.ttmc(t, fs, skip=n), golden[f"{tag}_skip{n}"]) <= 1e-13


@pytest.mark.parametrize("tag", list(HOOI))
def test_hooi_driver(golden, oracle, tag):
    spec, cfg = HOOI[tag]
    t = make_input(oracle, spec)
    core, fac, tr = oracle.hooi(t, cfg["ranks"], max_sweeps=cfg["max_sweeps"],
                                init=cfg.get("init", "hosvd"), seed=cfg["seed"])
    got_f, got_c = canon(fac, core)
    ref_f, ref_c = canon([golden[f"{tag}_a{k}"] for k in range(3)], golden[f"{tag}_core"])
    for a, b in zip(got_f, ref_f):
        assert relerr(a, b) <= 1e-10
    assert relerr(got_c, ref_c) <= 1e-10
    assert np.allclose(tr.fitness, golden[f"{tag}_fitness"], rtol=0, atol=1e-12)
    assert np.allclose(tr.residuals, golden[f"{tag}_residuals"], rtol=1e-9, atol=1e-12)


def test_cp_via_tucker_hooi_stage(golden, oracle):
    c, v = planted_cp_coo_host((30, 30, 30), 4000, rank=3, seed=5)
    st = oracle.Coo((30, 30, 30), c, v)
    fac, w, tr, _ = oracle.cp_via_tucker(st, 3, tucker_sweeps=3, cp_sweeps=10, seed=12,
                                         sketch=None)
    assert tr.stage_split == int(golden["cph_split"])
    assert np.allclose(tr.fitness, golden["cph_fitness"], rtol=0, atol=1e-10)
    assert np.allclose(tr.residuals, golden["cph_residuals"], rtol=1e-9, atol=1e-12)
    for k in range(3):
        assert relerr(np.abs(fac[k]), np.abs(golden[f"cph_a{k}"])) <= 1e-9
    assert relerr(np.abs(w), np.abs(golden["cph_w"])) <= 1e-9


SCP = {
    "scpd": (("dense", (20, 18, 16), 3, 1e-2, 7),
             dict(rank=3, sketch="leverage-random", sketch_factor=16, max_sweeps=5, seed=13)),
    "scps": (("sparse", (30, 30, 30), 4000, 5),
             dict(rank=3, sketch="leverage-random", sketch_size=200, max_sweeps=4, seed=14)),
}


@pytest.mark.parametrize("tag", list(SCP))
def test_sketched_cp(golden, oracle, tag):
    spec, cfg = SCP[tag]
    t = make_input(oracle, spec)
    fac, w, tr = oracle.sketched_cp(t, cfg["rank"], max_sweeps=cfg["max_sweeps"],
                                    sketch_size=cfg.get("sketch_size"),
                                    sketch_factor=cfg.get("sketch_factor"), seed=cfg["seed"])
    for k in range(3):
        assert relerr(fac[k], golden[f"{tag}_a{k}"]) <= 1e-9
    assert relerr(w, golden[f"{tag}_w"]) <= 1e-9
    assert np.allclose(tr.fitness, golden[f"{tag}_fitness"], rtol=0, atol=1e-10)
    assert np.allclose(tr.residuals, golden[f"{tag}_residuals"], rtol=1e-8, atol=1e-12)


@pytest.mark.parametrize("tag,nf", [("ld2", 2), ("ld3", 3), ("ldz", 2)])
def test_lev_deterministic_bit_exact(golden, oracle, tag, nf):
    fs = [golden[f"{tag}_f{k}"] for k in range(nf)]
    m = golden[f"{tag}_idx"].shape[0]
    idx, w, _ = oracle.lev_det(fs, m)
    assert np.array_equal(idx, golden[f"{tag}_idx"])
    assert np.array_equal(w, np.ones(m))


def _tm_cases(golden):
    for i in range(int(golden["tm_count"])):
        lists, k = [], 0
        while f"tm{i}_s{k}" in golden:
            lists.append(golden[f"tm{i}_s{k}"])
            k += 1
        yield i, lists, golden[f"tm{i}_idx"]


def test_top_m_products_ties_bit_exact(golden, oracle):
    """Best-first top-m with zero and repeated scores (pop order, not a sort)."""
    for i, lists, want in _tm_cases(golden):
        got = oracle.top_m_products(lists, want.shape[0])
        assert np.array_equal(got, want), i


DET = {
    "ddet": ("dense", (30, 30, 30), 3, 1e-2, 8),
    "sdet": ("sparse", (40, 40, 40), 3000, 9),
}


@pytest.mark.parametrize("tag", list(DET))
def test_sketched_tucker_deterministic(golden, oracle, tag):
    t = make_input(oracle, DET[tag])
    core, fac, tr = oracle.sketched_tucker(t, (3, 3, 3), "leverage-deterministic", max_sweeps=3,
                                           sketch_size=120, seed=2)
    got_f, got_c = canon(fac, core)
    ref_f, ref_c = canon([golden[f"{tag}_a{k}"] for k in range(3)], golden[f"{tag}_core"])
    for a, b in zip(got_f, ref_f):
        assert relerr(a, b) <= 1e-10
    assert relerr(got_c, ref_c) <= 1e-10
    assert np.allclose(tr.residuals, golden[f"{tag}_residuals"], rtol=1e-10, atol=0)


@pytest.mark.parametrize("tag", ["rtsd", "rtss", "rtdr", "rtsr"])
def test_ref_tucker_ts_vs_reference_golden(golden, oracle, tag):
    dense = tag in ("rtsd", "rtdr")
    spec = ("dense", (20, 18, 16), 3, 1e-2, 41) if dense else ("sparse", (30, 30, 30), 4000, 42)
    seed = 3 if dense else 4
    init = "random" if tag in ("rtdr", "rtsr") else None
    t = make_input(oracle, spec)
    core, fac, tr = oracle.ref_tucker_ts(t, (3, 3, 3), max_sweeps=3, sketch_size=200, seed=seed,
                                         init=init)
    got_f, got_c = canon(fac, core)
    ref_f, ref_c = canon([golden[f"{tag}_a{k}"] for k in range(3)], golden[f"{tag}_core"])
    for a, b in zip(got_f, ref_f):
        assert relerr(a, b) <= 1e-10
    assert relerr(got_c, ref_c) <= 1e-10
    assert np.allclose(tr.residuals, golden[f"{tag}_residuals"], rtol=1e-10, atol=0)
    assert np.allclose(tr.fitness, golden[f"{tag}_fitness"], rtol=0, atol=1e-12)
