"""Backend switch for the reference experiment harness.

The reference's `run_single` (src/harness.py:115-138) dispatches one
decomposition run on `spec.algorithm` to `tucker_mod` / `cp_mod`.  This module
is the same dispatch over this package's drivers, taking the resolved config
the reference builds in `_tucker_config` / `_cp_config` (src/harness.py:86-112)
so the reference harness can hand a run to the GPU path unchanged:

    from paper_2104_01101_b200 import harness as b200
    model, trace, m = b200.run_single(tensor, spec.algorithm, cfg)

Tensors and configs of the reference's own classes are accepted: a sparse
tensor is read through its `shape` / `coords` / `values` attributes, a config
through its dataclass fields (same names, src/tucker.py:57-66,
src/cp.py:45-53).  Spec parsing, synthetic generation, records and the CLI stay
on the reference side.
"""
import dataclasses

import numpy as np

from . import cp as cp_mod
from . import tucker as tucker_mod
from .tensors import SparseTensor

# algorithm name -> sketch kind, as src/harness.py:30-42
TUCKER_ALGS = {
    "hooi": None,
    "sketched-tucker-ts": "tensorsketch",
    "sketched-tucker-lev": "leverage-random",
    "sketched-tucker-lev-det": "leverage-deterministic",
    "ref-ts": "tensorsketch",
}
CP_ALGS = {
    "cp-als": None,
    "sketched-cp": "leverage-random",
    "tucker+cp": None,
    "sketched-tucker+cp": "leverage-random",
}
ALGORITHMS = tuple(TUCKER_ALGS) + tuple(CP_ALGS)


def adopt_tensor(t):
    """This package's tensor type for `t`: dense arrays pass through; a COO
    object of another class (the reference's SparseTensor) is rebuilt from its
    shape / coords / values, re-running the same validation."""
    if isinstance(t, SparseTensor) or not hasattr(t, "coords"):
        return t
    return SparseTensor(t.shape, np.asarray(t.coords), np.asarray(t.values))


def adopt_config(cfg, cls):
    """`cls` instance carrying the same-named fields of `cfg` (a dataclass of
    the reference's config classes, or already a `cls`)."""
    if isinstance(cfg, cls):
        return cfg
    names = {f.name for f in dataclasses.fields(cls)}
    return cls(**{f.name: getattr(cfg, f.name) for f in dataclasses.fields(cfg)
                  if f.name in names})


def run_single(tensor, algorithm, cfg):
    """One decomposition run; returns (model, trace, resolved sketch size) like
    src/harness.py:115-138; `ref-ts` is the one-variable TensorSketch baseline
    (src/tucker.py:303-364)."""
    if algorithm not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {algorithm!r}; choose from {ALGORITHMS}")
    t = adopt_tensor(tensor)
    if algorithm in TUCKER_ALGS:
        cfg = adopt_config(cfg, tucker_mod.TuckerConfig)
        if algorithm == "ref-ts":
            model, trace = tucker_mod.ref_tucker_ts(t, cfg)
        elif algorithm == "hooi":
            model, trace = tucker_mod.hooi(t, cfg)
        else:
            model, trace = tucker_mod.sketched_tucker_als(t, cfg)
        return model, trace, cfg.resolved_sketch_size() if cfg.sketch else None
    cfg = adopt_config(cfg, cp_mod.CPConfig)
    if algorithm == "cp-als":
        model, trace = cp_mod.cp_als(t, cfg)
    elif algorithm == "sketched-cp":
        model, trace = cp_mod.sketched_cp_als(t, cfg)
    else:
        model, trace = cp_mod.cp_via_sketched_tucker(t, cfg)
    needs_m = algorithm in ("sketched-cp", "sketched-tucker+cp")
    return model, trace, cfg.resolved_sketch_size() if needs_m else None
