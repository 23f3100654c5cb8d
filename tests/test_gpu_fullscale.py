"""GPU: full-scale spot checks on the bench tensors themselves.

The parity fixtures stop at sizes the reference finishes in minutes; these
tests take the BASELINE-size inputs the bench times and recompute a few sampled
rows of the sketches on the host, independently of the device kernels:

* config 5 (2e5^3, 1e9 nonzeros): the RRF CountSketch stage 1 of modes 1 and 2
  over P_n = 4e10 composite columns (src/sketching.py:54-56, 327-341).  The
  table entry of every contributing column is drawn by numpy's own Generator
  positioned at the column's raw Philox position (rejections before it counted
  from the device's d-array), and each cell is summed exactly (math.fsum): the
  fixed-point kernel rounds the exact sum once, so the match is bitwise.
* config 4 (1e5^3, 1e8 nonzeros): TensorSketch right-hand sides Y_n
  (src/sketching.py:150-175) at sampled columns i_n, recomputed by np.add.at
  over that column's nonzeros in the reference's unfolding order (ascending
  composite index) with the oracle's hash tables: bitwise.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def skx():
    import paper_2104_01101_b200 as m
    m._native.load()
    return m


def _bench_tensor(skx, cfgno):
    import bench
    from paper_2104_01101_b200.synth import planted_cp_coo_device
    from paper_2104_01101_b200.tensors import device_of
    cfgd = bench.CONFIGS[cfgno]
    coords, vals = planted_cp_coo_device(cfgd["shape"], cfgd["nnz"], rank=10, noise_sd=0.1, seed=0)
    st = skx.SparseTensor.from_device(cfgd["shape"], coords.t().contiguous(), vals, validate=False)
    del coords, vals
    return cfgd, device_of(st)


def _row_entries(d, n, row):
    """(composite other index j, value) of the nonzeros with i_n == row,
    ascending j (the reference's unfolding order)."""
    import torch
    idx = torch.nonzero(d.coords[n] == row).flatten()
    c = d.coords[:, idx].long().cpu().numpy()
    v = d.vals[idx].cpu().numpy()
    others = [k for k in range(d.ndim) if k != n]
    j = np.ravel_multi_index([c[k] for k in others], [d.shape[k] for k in others])
    o = np.argsort(j, kind="stable")
    return j[o], v[o], c[:, o]


def test_config5_rrf_stage1_rows_at_full_scale(skx):
    from paper_2104_01101_b200 import rng as rngmod
    from paper_2104_01101_b200.sketching import draw_rrf_tables
    from paper_2104_01101_b200.tucker import _rrf_dims, rrf_stage1_dev
    cfgd, d = _bench_tensor(skx, 5)
    assert d.nnz == 1_000_000_000 and d.fixed_point_ok()
    R = cfgd["ranks"][0]
    for n, seed in ((1, 21), (2, 22)):
        P, k2 = _rrf_dims(d.shape, n, R, 4 * R)
        assert P == 40_000_000_000
        gen = rngmod.split_rng(seed, 3)[0]
        c0 = rngmod.cursor(gen)
        assert not c0.has
        tabs = draw_rrf_tables(gen, P, k2)
        st1 = rrf_stage1_dev(d, n, tabs).cpu().numpy()
        dl = tabs.d.cpu().numpy().view(np.uint64)
        dl = np.sort(dl[dl < np.uint64(1 << 62)]).astype(np.int64)  # drop the list's fillers
        nrej = int(np.sum(dl <= P - 1))
        assert tabs.sign_q0 == P + nrej and nrej > 1000  # ~ P k2 / 2^32 rejections
        base = rngmod.split_rng(seed, 3)[0]
        rows = np.random.default_rng(seed).integers(0, d.shape[n], size=3)
        for row in rows:
            j, v, _ = _row_entries(d, n, int(row))
            assert len(j) > 3000
            cells = {}
            for jj, vv in zip(j, v):
                q = int(jj) + int(np.searchsorted(dl, jj, side="right"))  # raw u32 of the hash
                rngmod.set_cursor(base, c0.p + q // 2, 0, 0)
                if q % 2:
                    base.integers(0, 2, size=1)
                h = int(base.integers(0, k2, size=1)[0])
                qs = P + nrej + int(jj)  # raw u32 of the sign (integers(0,2) never rejects)
                rngmod.set_cursor(base, c0.p + qs // 2, 0, 0)
                if qs % 2:
                    base.integers(0, 2, size=1)
                s = 1 - 2 * int(base.integers(0, 2, size=1)[0])
                cells.setdefault(h, []).append(s * float(vv))
            want = np.zeros(k2)
            for h, terms in cells.items():
                want[h] = math.fsum(terms)
            assert np.array_equal(st1[row], want), (n, row, np.abs(st1[row] - want).max())


def test_config4_ts_rhs_columns_at_full_scale(skx, oracle):
    import torch
    from paper_2104_01101_b200.sketching import ts_rhs_coo_dev
    cfgd, d = _bench_tensor(skx, 4)
    assert d.nnz == 100_000_000
    m = cfgd["sketch_size"]
    for n in range(3):
        ext = tuple(d.shape[k] for k in range(3) if k != n)
        op = skx.TensorSketchOp.build(ext, m, skx.make_rng(40 + n))
        hs, ss = oracle.ts_tables(ext, m, oracle.generator(40 + n))
        colptr, rec = d.fibre(n)
        yt = ts_rhs_coo_dev(op, colptr, rec, d.shape[n], d.fibre_mask(n))
        rows = np.random.default_rng(n).integers(0, d.shape[n], size=4)
        got = yt[torch.from_numpy(rows).cuda()].cpu().numpy()
        d.drop_fibre(n)
        for r, row in enumerate(rows):
            _, v, c = _row_entries(d, n, int(row))
            others = [k for k in range(3) if k != n]
            h, g = oracle.ts_bucket_sign(hs, ss, m, [c[k] for k in others])
            want = np.zeros(m)
            np.add.at(want, h, g * v)
            assert np.array_equal(got[r], want), (n, row)
