"""GPU: device draws are bit-identical to numpy 2.3.5 Generator(Philox)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gen(seed, i=0, n=3):
    from paper_2104_01101_b200.rng import split_rng
    return split_rng(seed, n)[i]


def test_uniform_bit_exact():
    import torch
    from paper_2104_01101_b200 import _native as nat
    from paper_2104_01101_b200.rng import cursor
    for seed in range(4):
        g = _gen(seed, 1)
        g.random(7)  # start mid-block
        c = cursor(g)
        out = torch.empty(10_007, dtype=torch.float64, device="cuda")
        nat.call("skx_philox_uniform", ctypes.c_uint64(c.k0), ctypes.c_uint64(c.k1),
                 ctypes.c_uint64(c.p), out.numel(), nat.ptr(out), nat.stream())
        assert np.array_equal(out.cpu().numpy(), g.random(10_007))


@pytest.mark.parametrize("n", [1, 17, 1000, 250_000, 2_000_000])
def test_normal_bit_exact_and_position(n):
    from paper_2104_01101_b200.linalg import NormalSource
    from paper_2104_01101_b200.rng import cursor
    for seed in (0, 3):
        g = _gen(seed, 2)
        g.standard_normal(5)
        ref_g = _gen(seed, 2)
        ref_g.standard_normal(5)
        src = NormalSource(g)
        a = src.normal((n,)).cpu().numpy()
        b = src.normal((3, 7)).cpu().numpy()
        assert np.array_equal(a, ref_g.standard_normal(n))
        assert np.array_equal(b, ref_g.standard_normal((3, 7)))
        src.sync_host()
        assert cursor(g).p == cursor(ref_g).p
        assert np.array_equal(g.standard_normal(3), ref_g.standard_normal(3))


@pytest.mark.parametrize("P,k2", [(1000, 45), (160_000, 157), (1_000_003, 480), (2_000_000, 140),
                                  (50_000, 128), (7, 3)])
def test_rrf_tables_bit_exact(P, k2):
    from paper_2104_01101_b200.sketching import _unpack, draw_rrf_tables, rrf_table_dev
    for seed, pre in ((0, 0), (5, 3)):
        g = _gen(seed, 0)
        ref = _gen(seed, 0)
        if pre:  # leave a buffered high half pending
            g.integers(0, 2, size=pre)
            ref.integers(0, 2, size=pre)
        tabs = draw_rrf_tables(g, P, k2)
        h, s = _unpack(rrf_table_dev(tabs))
        rh = ref.integers(0, k2, size=P)
        rs = 1 - 2 * ref.integers(0, 2, size=P)
        assert np.array_equal(h, rh)
        assert np.array_equal(s, rs)
        # the host generator continues exactly where numpy's does
        assert np.array_equal(g.standard_normal(11), ref.standard_normal(11))
        assert np.array_equal(g.integers(0, 99, size=5), ref.integers(0, 99, size=5))


@pytest.mark.parametrize("pre", [0, 1])
def test_planned_chain_of_rrf_draws_bit_exact(pre):
    """Scans launched up front for three consecutive (hash, sign, Gaussian)
    draw groups -- the RRF init of an order-4 tensor -- resolve to numpy's
    exact tables, including the buffered-half carry across the normals."""
    import torch
    from paper_2104_01101_b200.sketching import _unpack, finish_rrf_scan, plan_rrf_scans, rrf_table_dev
    jobs = [(300_001, 157, 157 * 57), (1_000_003, 480, 480 * 80), (77_777, 45, 45 * 20)]
    g = _gen(21, 0)
    ref = _gen(21, 0)
    if pre:
        g.integers(0, 2, size=1)
        ref.integers(0, 2, size=1)
    side = torch.cuda.Stream()
    scans = plan_rrf_scans(g, [(P, k2, n) for P, k2, n in jobs], side)
    for scan, (P, k2, n) in zip(scans, jobs):
        tabs = finish_rrf_scan(scan, g, P)
        h, s = _unpack(rrf_table_dev(tabs))
        assert np.array_equal(h, ref.integers(0, k2, size=P))
        assert np.array_equal(s, 1 - 2 * ref.integers(0, 2, size=P))
        assert np.array_equal(g.standard_normal(n), ref.standard_normal(n))


def test_lemire_large_offset_spot_check():
    """Full-scale style check: a 2e8-column table, compared at random columns
    against numpy positioned with the cursor."""
    import torch
    from paper_2104_01101_b200.rng import set_cursor, cursor
    from paper_2104_01101_b200.sketching import draw_rrf_tables, rrf_table_dev, _unpack
    P, k2 = 200_000_000, 480
    g = _gen(11, 0)
    tabs = draw_rrf_tables(g, P, k2)
    tab = rrf_table_dev(tabs)
    # exact check of the first 2e6 columns against numpy
    ref = _gen(11, 0)
    head = ref.integers(0, k2, size=2_000_000)
    h, _ = _unpack(tab[:2_000_000])
    assert np.array_equal(h, head)
    # sign run starts after P + nrej u32 draws: position numpy there and compare
    d = tabs.d.cpu().numpy().view(np.uint64)
    nrej = int(np.sum(d <= P - 1))
    assert tabs.sign_q0 == P + nrej
    rng = np.random.default_rng(0)
    cols = np.sort(rng.integers(0, P, size=20))
    _, s = _unpack(tab[torch.from_numpy(cols).cuda()])
    base = _gen(11, 0)
    c0 = cursor(base)
    for col, sg in zip(cols, s):
        q = P + nrej + int(col)  # u32 index of the sign draw
        set_cursor(base, c0.p + q // 2, 0, 0)
        if q % 2:
            base.integers(0, 2, size=1)
        assert 1 - 2 * int(base.integers(0, 2, size=1)[0]) == sg
