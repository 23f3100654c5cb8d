"""Harness backend switch (paper_2104_01101_b200/harness.py, mirrors
src/harness.py:30-42, :115-138)."""
import dataclasses

import numpy as np
import pytest

from paper_2104_01101_b200 import harness
from paper_2104_01101_b200.cp import CPConfig
from paper_2104_01101_b200.tensors import SparseTensor
from paper_2104_01101_b200.tucker import TuckerConfig


@dataclasses.dataclass
class _ForeignTucker:  # stands in for the reference's TuckerConfig
    ranks: tuple
    max_sweeps: int = 5
    sketch: str = None
    sketch_size: int = None
    sketch_factor: float = None
    init: str = None
    rrf_width: int = None
    seed: int = 0
    convergence_tol: float = 0.0


class _ForeignCoo:  # duck-typed COO of another class
    def __init__(self, shape, coords, values):
        self.shape, self.coords, self.values = shape, coords, values


def test_algorithm_table_matches_reference_names():
    assert set(harness.TUCKER_ALGS) == {"hooi", "sketched-tucker-ts", "sketched-tucker-lev",
                                        "sketched-tucker-lev-det", "ref-ts"}
    assert set(harness.CP_ALGS) == {"cp-als", "sketched-cp", "tucker+cp", "sketched-tucker+cp"}


def test_adopt_config_and_tensor():
    cfg = harness.adopt_config(_ForeignTucker((2, 2, 2), sketch="tensorsketch", sketch_size=40,
                                              seed=7), TuckerConfig)
    assert isinstance(cfg, TuckerConfig) and cfg.seed == 7 and cfg.resolved_sketch_size() == 40
    same = CPConfig(rank=3)
    assert harness.adopt_config(same, CPConfig) is same
    t = harness.adopt_tensor(_ForeignCoo((3, 4), np.array([[0, 1], [2, 3]]), np.array([1.0, 2.0])))
    assert isinstance(t, SparseTensor) and t.nnz == 2
    with pytest.raises(ValueError):
        harness.adopt_tensor(_ForeignCoo((3, 4), np.array([[0, 1], [0, 1]]), np.array([1.0, 2.0])))
    dense = np.zeros((2, 2))
    assert harness.adopt_tensor(dense) is dense


def test_run_single_errors():
    with pytest.raises(ValueError):
        harness.run_single(np.zeros((2, 2, 2)), "nope", TuckerConfig((1, 1, 1)))
    # ref-ts validates like the reference (TensorSketch only) before any device work
    with pytest.raises(ValueError):
        harness.run_single(np.zeros((2, 2, 2)), "ref-ts",
                           TuckerConfig((1, 1, 1), sketch="leverage-random", sketch_size=8))


@pytest.mark.gpu
@pytest.mark.parametrize("alg", ["hooi", "sketched-tucker-ts", "sketched-tucker-lev"])
def test_run_single_tucker_matches_driver(alg):
    from paper_2104_01101_b200 import tucker
    rng = np.random.default_rng(3)
    x = rng.standard_normal((12, 13, 14))
    sk = harness.TUCKER_ALGS[alg]
    fcfg = _ForeignTucker((3, 3, 3), max_sweeps=3, sketch=sk, sketch_size=90 if sk else None,
                          seed=5)
    model, trace, m = harness.run_single(x, alg, fcfg)
    cfg = harness.adopt_config(fcfg, TuckerConfig)
    direct, dtrace = (tucker.hooi if alg == "hooi" else tucker.sketched_tucker_als)(x, cfg)
    assert m == (90 if sk else None)
    np.testing.assert_array_equal(model.core, direct.core)
    assert list(trace.fitness) == list(dtrace.fitness)


@pytest.mark.gpu
@pytest.mark.parametrize("alg", ["cp-als", "sketched-cp", "sketched-tucker+cp"])
def test_run_single_cp_matches_driver(alg):
    from paper_2104_01101_b200 import cp
    rng = np.random.default_rng(4)
    x = rng.standard_normal((10, 11, 12))
    sk = harness.CP_ALGS[alg]
    cfg = CPConfig(rank=3, max_sweeps=4, sketch=sk, sketch_size=60 if sk else None, seed=2)
    model, trace, m = harness.run_single(x, alg, cfg)
    fn = {"cp-als": cp.cp_als, "sketched-cp": cp.sketched_cp_als,
          "sketched-tucker+cp": cp.cp_via_sketched_tucker}[alg]
    direct, dtrace = fn(x, cfg)
    assert m == (60 if sk else None)
    assert list(trace.fitness) == list(dtrace.fitness)
