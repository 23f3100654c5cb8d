"""The composite C-ABI entries of SURVEY 8(b)'s export list, called through
ctypes the way a C caller would: model fitness in one call (Tucker sparse /
dense, CP sparse) against the Python layer and the CPU oracle, and the NCCL
binding on a one-rank communicator."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2104_01101_b200 as skx
    from paper_2104_01101_b200 import _native as nat
    nat.load()
    return torch, skx, nat


def _orthonormal(rng, s, r):
    return np.linalg.qr(rng.standard_normal((s, r)))[0]


@pytest.mark.parametrize("shape,nnz,R", [((300, 400, 500), 200_000, 10),
                                         ((2000, 1500, 1000), 1_000_000, 20),
                                         ((40, 30, 20, 10), 20_000, 4)])
def test_fitness_tucker_coo_entry(env, oracle, shape, nnz, R):
    torch, skx, nat = env
    from paper_2104_01101_b200.synth import planted_cp_coo_host
    from paper_2104_01101_b200.tensors import device_of
    c, v = planted_cp_coo_host(shape, nnz, rank=3, seed=5)
    st = skx.SparseTensor(shape, c, v)
    d = device_of(st)
    rng = np.random.default_rng(5)
    ranks = [min(R, s) for s in shape]
    fac = [_orthonormal(rng, s, r) for s, r in zip(shape, ranks)]
    core = rng.standard_normal(ranks)
    fd = [torch.from_numpy(a).cuda() for a in fac]
    cd = torch.from_numpy(core).cuda()
    shp, sp_ = nat.host_i64(shape)
    rk, rp = nat.host_i64(ranks)
    arr, fp = nat.host_ptrs(fd)
    cpt, rec0 = d.fibre(0) if d.ndim == 3 else (None, None)
    fit = torch.empty(1, dtype=torch.float64, device="cuda")
    nat.call_ws("skx_fitness_tucker_coo",
                (d.ndim, sp_, rp, d.nnz, nat.ptr(d.coords), nat.ptr(d.vals), fp, nat.ptr(cd),
                 nat.ptr(cpt), nat.ptr(rec0), ctypes.c_uint32(d.fibre_mask(0) if d.ndim == 3 else 0),
                 None, nat.ptr(fit)))
    got = float(fit.cpu())
    ref_py = skx.fitness(st, skx.TuckerModel(core, fac))
    ref_orc = oracle.fitness_tucker(oracle.Coo(shape, c, v), core, fac)
    assert abs(got - ref_py) <= 1e-13, (got, ref_py)
    assert abs(got - ref_orc) <= 1e-12, (got, ref_orc)
    # caller-supplied ||T||^2
    n2 = torch.tensor([float(np.sum(v * v))], dtype=torch.float64, device="cuda")
    fit2 = torch.empty(1, dtype=torch.float64, device="cuda")
    nat.call_ws("skx_fitness_tucker_coo",
                (d.ndim, sp_, rp, d.nnz, nat.ptr(d.coords), nat.ptr(d.vals), fp, nat.ptr(cd),
                 nat.ptr(cpt), nat.ptr(rec0), ctypes.c_uint32(d.fibre_mask(0) if d.ndim == 3 else 0),
                 nat.ptr(n2), nat.ptr(fit2)))
    assert abs(float(fit2.cpu()) - got) <= 1e-14


@pytest.mark.parametrize("shape,R", [((60, 50, 40), 5), ((20, 18, 16, 14), 4)])
def test_fitness_tucker_dense_entry(env, oracle, shape, R):
    torch, skx, nat = env
    rng = np.random.default_rng(7)
    t = rng.standard_normal(shape)
    ranks = [R] * len(shape)
    fac = [_orthonormal(rng, s, R) for s in shape]
    core = rng.standard_normal(ranks)
    td = torch.from_numpy(t).cuda()
    fd = [torch.from_numpy(a).cuda() for a in fac]
    cd = torch.from_numpy(core).cuda()
    shp, sp_ = nat.host_i64(shape)
    rk, rp = nat.host_i64(ranks)
    arr, fp = nat.host_ptrs(fd)
    fit = torch.empty(1, dtype=torch.float64, device="cuda")
    nat.call_ws("skx_fitness_tucker_dense",
                (len(shape), sp_, nat.ptr(td), rp, fp, nat.ptr(cd), None, nat.ptr(fit)))
    got = float(fit.cpu())
    assert abs(got - skx.fitness(t, skx.TuckerModel(core, fac))) <= 1e-13
    assert abs(got - oracle.fitness_tucker(t, core, fac)) <= 1e-12


@pytest.mark.parametrize("shape,nnz,R,layout", [((300, 400, 500), 200_000, 10, True),
                                                ((300, 400, 500), 200_000, 7, False),
                                                ((40, 30, 20, 10), 20_000, 5, False)])
def test_fitness_cp_coo_entry(env, oracle, shape, nnz, R, layout):
    torch, skx, nat = env
    from paper_2104_01101_b200.synth import planted_cp_coo_host
    from paper_2104_01101_b200.tensors import device_of
    c, v = planted_cp_coo_host(shape, nnz, rank=3, seed=8)
    st = skx.SparseTensor(shape, c, v)
    d = device_of(st)
    rng = np.random.default_rng(8)
    fac = [rng.standard_normal((s, R)) for s in shape]
    w = rng.random(R) + 0.5
    fd = [torch.from_numpy(a).cuda() for a in fac]
    wd = torch.from_numpy(w).cuda()
    shp, sp_ = nat.host_i64(shape)
    arr, fp = nat.host_ptrs(fd)
    cpt, rec0 = d.fibre(0) if layout else (None, None)
    fit = torch.empty(1, dtype=torch.float64, device="cuda")
    nat.call_ws("skx_fitness_cp_coo",
                (d.ndim, sp_, R, d.nnz, nat.ptr(d.coords), nat.ptr(d.vals), fp, nat.ptr(wd),
                 nat.ptr(cpt), nat.ptr(rec0), ctypes.c_uint32(d.fibre_mask(0) if layout else 0),
                 None, nat.ptr(fit)))
    got = float(fit.cpu())
    ref_py = skx.fitness(st, skx.CPModel(fac, w))
    ref_orc = oracle.fitness_cp(oracle.Coo(shape, c, v), fac, w)
    assert abs(got - ref_py) <= 1e-12 * max(1.0, abs(ref_py)), (got, ref_py)
    assert abs(got - ref_orc) <= 1e-11 * max(1.0, abs(ref_orc)), (got, ref_orc)


def test_nccl_one_rank(env):
    """A one-rank communicator: all-reduce, reduce-scatter and all-gather are
    copies (a B200 box gives one GPU per call; several ranks of one device are
    not a valid NCCL communicator)."""
    torch, skx, nat = env
    lib = nat.load()
    uid = ctypes.create_string_buffer(128)
    assert lib.skx_nccl_unique_id(uid) == 0
    comm = ctypes.c_void_p()
    assert lib.skx_nccl_init(uid, 0, 1, ctypes.byref(comm)) == 0
    try:
        x = torch.randn(1000, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        st = nat.stream()
        assert lib.skx_allreduce_sum(comm, nat.ptr(x), nat.ptr(y), ctypes.c_int64(1000), st) == 0
        torch.cuda.synchronize()
        assert torch.equal(x, y)
        y.zero_()
        assert lib.skx_reduce_scatter_sum(comm, nat.ptr(x), nat.ptr(y), ctypes.c_int64(1000), st) == 0
        torch.cuda.synchronize()
        assert torch.equal(x, y)
        y.zero_()
        assert lib.skx_allgather(comm, nat.ptr(x), nat.ptr(y), ctypes.c_int64(1000), st) == 0
        torch.cuda.synchronize()
        assert torch.equal(x, y)
    finally:
        assert lib.skx_nccl_destroy(comm) == 0


@pytest.mark.parametrize("shape,nnz", [((300, 400, 500), 200_000), ((40, 30, 20, 10), 20_000)])
def test_pack0_range_matches_mode0_layout(env, shape, nnz):
    """The mode-0 layout packed chunk by chunk (skx_coo_pack0_range, the e2e
    upload path) equals the one-pass layout (skx_coo_fibre, mode 0) bit for
    bit, records and slice pointers."""
    torch, skx, nat = env
    from paper_2104_01101_b200.synth import planted_cp_coo_host
    from paper_2104_01101_b200.tensors import device_of
    c, v = planted_cp_coo_host(shape, nnz, rank=3, seed=9)
    d = device_of(skx.SparseTensor(shape, c, v))
    colptr, rec = d.fibre(0)
    rw = int(nat.load().skx_coo_rec_words(len(shape)))
    rec2 = torch.full((d.nnz * rw,), float("nan"), dtype=torch.float64, device="cuda")
    bounds = np.linspace(0, d.nnz, 8).astype(np.int64)
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        nat.call("skx_coo_pack0_range", len(shape), d.nnz, int(lo), int(hi), nat.ptr(d.coords),
                 nat.ptr(d.vals), nat.ptr(rec2), nat.stream())
    torch.cuda.synchronize()
    assert torch.equal(rec.view(torch.int64)[:d.nnz * rw], rec2.view(torch.int64))
    ptr0 = np.searchsorted(c[:, 0], np.arange(shape[0] + 1), side="left")
    assert np.array_equal(colptr.cpu().numpy(), ptr0)


def test_to_host_matches_cpu(env):
    """Model download through the pinned staging buffer and parallel host
    copies equals .cpu() (large, small, non-contiguous and non-float64
    inputs); the returned arrays are fresh (a second download does not
    overwrite the first)."""
    torch, skx, nat = env
    from paper_2104_01101_b200.tensors import to_host
    g = torch.Generator(device="cuda").manual_seed(0)
    big = [torch.randn(200_000, 10, dtype=torch.float64, device="cuda", generator=g) for _ in range(3)]
    odd = torch.randn(30, 7, dtype=torch.float64, device="cuda", generator=g).t()
    core = torch.randn(20, 20, 20, dtype=torch.float64, device="cuda", generator=g)
    ts = big + [odd, core]
    got = to_host(ts)
    for a, b in zip(got, ts):
        assert a.shape == tuple(b.shape) and np.array_equal(a, b.cpu().numpy())
    again = to_host([t * 2 for t in ts])
    for a, b in zip(got, ts):
        assert np.array_equal(a, b.cpu().numpy())  # not aliased to the staging buffer
    for a, b in zip(again, ts):
        assert np.array_equal(a, (b * 2).cpu().numpy())
    ints = to_host([torch.arange(300_000, device="cuda")])
    assert np.array_equal(ints[0], np.arange(300_000))


@pytest.mark.parametrize("s", [1, 7, 1023, 1025, 200_000, 333_333])
def test_lev_prepare_fused_equals_five_launch_form(env, s, monkeypatch):
    """The one-CTA leverage cdf (batched loads) and the five-launch form give
    the same p and cdf bit for bit, zero and negative scores included."""
    torch, skx, nat = env
    g = torch.Generator(device="cuda").manual_seed(s)
    sc = torch.rand(s, dtype=torch.float64, device="cuda", generator=g)
    if s > 10:
        sc[::7] = 0.0
        sc[3::11] = -1e-17
    outs = []
    for five in (False, True):
        if five:
            monkeypatch.setenv("SKX_LEV_5K", "1")
        p = torch.empty(s, dtype=torch.float64, device="cuda")
        cdf = torch.empty(s, dtype=torch.float64, device="cuda")
        nat.call_ws("skx_lev_prepare", (nat.ptr(sc), s, nat.ptr(p), nat.ptr(cdf)), slot=7)
        torch.cuda.synchronize()
        outs.append((p.clone(), cdf.clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    ref = np.maximum(sc.cpu().numpy(), 0)
    ref = ref / ref.sum()
    c = np.cumsum(ref)
    # (numpy's sequential cumsum carries ~s eps of its own rounding)
    assert np.allclose(outs[0][1].cpu().numpy(), c / c[-1], rtol=0, atol=max(1e-14, 4e-16 * s))
