"""GPU: K8 (skx_cp_core_als, CP-ALS on the Tucker core in one CTA) against
the oracle restatement of src/cp.py:119-174 (on_core=True), plus the
minimum-norm least squares of sketched CP-ALS against numpy's gelsd."""
import numpy as np
import pytest

from tests.conftest import relerr

pytestmark = pytest.mark.gpu


def _planted_core(shape, rank, noise, seed):
    g = np.random.default_rng(seed)
    fs = [g.standard_normal((s, rank)) for s in shape]
    t = np.einsum("ir,jr,kr->ijk", *fs)
    e = g.standard_normal(shape)
    return t + noise * np.linalg.norm(t) / np.linalg.norm(e) * e


@pytest.mark.parametrize("shape,rank,sweeps,seed", [
    ((20, 20, 20), 10, 50, 0),   # config 5's core stage
    ((3, 3, 3), 3, 10, 1),
    ((15, 20, 12), 8, 30, 2),
    ((24, 24, 24), 12, 8, 3),
])
def test_cp_core_kernel_vs_oracle(oracle, shape, rank, sweeps, seed):
    import torch
    from paper_2104_01101_b200.cp import CPConfig, _core_kernel_ok, cp_core_als_dev
    core = _planted_core(shape, rank, 1e-2, seed)
    dev = torch.from_numpy(core).cuda()
    cfg = CPConfig(rank=rank, max_sweeps=sweeps, init="hosvd-of-core")
    if not _core_kernel_ok(dev, rank, "hosvd-of-core"):
        pytest.skip("core does not fit one CTA")
    fac, w, tr = cp_core_als_dev(dev, cfg)
    A, wr, otr = oracle.cp_on_core(core, rank, sweeps=sweeps)
    assert len(tr.residuals) == 3 * sweeps and len(tr.fitness) == sweeps
    assert np.allclose(tr.residuals, otr.residuals, rtol=1e-8, atol=1e-10)
    assert np.allclose(tr.fitness, otr.fitness, rtol=0, atol=1e-9)
    for a, b in zip(fac, A):
        assert relerr(np.abs(a.cpu().numpy()), np.abs(b)) <= 1e-8
    assert relerr(w.cpu().numpy(), wr) <= 1e-8


def test_cp_core_kernel_zero_core():
    import torch
    from paper_2104_01101_b200.cp import CPConfig, cp_core_als_dev
    with pytest.raises(ValueError):
        cp_core_als_dev(torch.zeros((4, 4, 4), dtype=torch.float64, device="cuda"),
                        CPConfig(rank=2, max_sweeps=3))


def test_cp_core_kernel_is_one_launch():
    """cp_via_sketched_tucker's core stage is one libskx launch."""
    import torch
    from paper_2104_01101_b200 import _native as nat
    from paper_2104_01101_b200.cp import CPConfig, cp_als_dev
    core = torch.from_numpy(_planted_core((20, 20, 20), 10, 1e-2, 5)).cuda()
    n0 = nat.launch_count()
    cp_als_dev(core, CPConfig(rank=10, max_sweeps=50, init="hosvd-of-core"), on_core=True)
    assert nat.launch_count() - n0 == 1


@pytest.mark.parametrize("deficient", [False, True])
def test_min_norm_lstsq_vs_numpy(deficient):
    """Sampled Khatri-Rao systems may repeat rows / columns: gelsd semantics."""
    import torch
    from paper_2104_01101_b200.cp import _lstsq_min_norm_dev
    g = np.random.default_rng(9)
    z = g.standard_normal((60, 6))
    if deficient:
        z[:, 4] = z[:, 2]
        z[:, 5] = 0.0
    y = g.standard_normal((60, 25))
    want = np.linalg.lstsq(z, y, rcond=None)[0]
    got = _lstsq_min_norm_dev(torch.from_numpy(z).cuda(), torch.from_numpy(y).cuda())
    assert np.all(np.isfinite(got.cpu().numpy()))
    assert relerr(got.cpu().numpy(), want) <= 1e-10
