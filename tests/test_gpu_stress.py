"""GPU: randomised parity sweep against the CPU oracle (tools/stress_parity.py
logic at a fixed seed): random small shapes, orders 3-4, ranks, TensorSketch
and leverage sampling, dense and sparse inputs.  Pure-noise tensors have no
spectral gap, so the bound is 1e-8 (planted low-rank data in
test_gpu_drivers.py is held to 1e-10)."""
import numpy as np
import pytest

from tests.conftest import canon, relerr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [11, 12])
def test_random_configs_match_oracle(oracle, seed):
    import paper_2104_01101_b200 as skx
    rng = np.random.default_rng(seed)
    checked = 0
    for _ in range(6):
        nd = int(rng.choice([3, 3, 4]))
        shape = tuple(int(x) for x in rng.integers(9, 36 if nd == 3 else 13, nd))
        ranks = tuple(int(min(s - 1, x)) for s, x in zip(shape, rng.integers(2, 5, nd)))
        sketch = str(rng.choice(["tensorsketch", "leverage-random"]))
        need = max(int(np.prod([ranks[k] for k in range(nd) if k != j])) for j in range(nd))
        m = int(need * rng.uniform(3.0, 6.0))
        s = int(rng.integers(0, 1000))
        if rng.integers(0, 2):
            nnz = int(np.prod(shape) * rng.uniform(0.1, 0.3))
            lin = np.sort(rng.choice(int(np.prod(shape)), size=nnz, replace=False))
            coords = np.stack(np.unravel_index(lin, shape), axis=1)
            vals = rng.standard_normal(nnz)
            t_gpu, t_ref = skx.SparseTensor(shape, coords, vals), oracle.Coo(shape, coords, vals)
        else:
            t_gpu = t_ref = rng.standard_normal(shape)
        model, tr = skx.sketched_tucker_als(
            t_gpu, skx.TuckerConfig(ranks=ranks, max_sweeps=3, sketch=sketch, sketch_size=m, seed=s))
        core, fac, otr = oracle.sketched_tucker(t_ref, ranks, sketch, max_sweeps=3, sketch_size=m,
                                                seed=s)
        gf, gc = canon(model.factors, model.core)
        rf, rc = canon(fac, core)
        for a, b in zip(gf, rf):
            assert relerr(a, b) <= 1e-8, (shape, ranks, sketch, m)
        assert relerr(gc, rc) <= 1e-8
        assert np.allclose(tr.fitness, otr.fitness, rtol=0, atol=1e-9)
        checked += 1
    assert checked == 6
