"""Golden fixtures for the BASELINE.json configurations, made by running the
REAL reference package (``sketchals`` from /root/reference/pkg/src).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_configs.py [tag ...]

Configs 2 and 3 run at their full BASELINE size; configs 4 and 5 (which the
reference cannot run at 1e8 / 1e9 nonzeros: its unfoldings and RRF tables need
80-640 GB) run at SURVEY 8(c)'s reduced scales, 2000^3 / 1e6 and 1e4^3 / 1e7
nonzeros, with every other parameter of the config.  Config 5 is Algorithm 6
with Tucker rank 20 and CP rank 10 (BASELINE.json); the reference's
``cp_via_sketched_tucker`` ties the Tucker ranks to the CP rank, so the
fixture composes the reference's own public functions the same way
src/cp.py:177-224 does, with ranks (20, 20, 20) in the TuckerConfig.

Recorded (small enough to commit; the inputs are regenerated from seeds):
* trace fitness / residuals / wall_s, the reference's whole-call seconds;
* sign-canonicalised factors (full when s <= 2000, else the first 256 rows
  plus a seeded Gaussian projection A^T G) and the core;
* intermediates observed by wrapping the reference's module functions (the
  reference itself is not modified): every TensorSketch right-hand side
  ``ts_apply_rhs`` -> sha256 of its bytes (bit-exact contract for sparse
  inputs: numpy add.at order), its Frobenius norm and a seeded projection;
  every leverage sampler ``lev_build`` -> sha256 of the index set and the
  weights, the full first index set.
"""
import hashlib
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import sketchals as ref  # noqa: E402
import sketchals.tucker as ref_tucker  # noqa: E402
from sketchals.cp import _normalize_columns  # noqa: E402

from paper_2104_01101_b200.synth import planted_cp_coo_host, planted_tucker_dense  # noqa: E402

PROJ_SEED = 20260101
FULL_ROWS = 2000


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def canon(factors, core=None):
    out = []
    core = None if core is None else np.array(core, copy=True)
    for n, a in enumerate(factors):
        a = np.array(a, copy=True)
        piv = np.argmax(np.abs(a), axis=0)
        sg = np.sign(a[piv, np.arange(a.shape[1])])
        sg[sg == 0] = 1.0
        a *= sg
        out.append(a)
        if core is not None:
            shp = [1] * core.ndim
            shp[n] = -1
            core *= sg.reshape(shp)
    return out, core


def proj_matrix(rows, k, salt):
    return np.random.default_rng([PROJ_SEED, rows, k, salt]).standard_normal((rows, k))


CASES = {
    # tag: (input spec, driver, config kwargs)
    "c2": (("dense", (400,) * 3, 10, 1e-2, 0), "tucker",
           dict(ranks=(10,) * 3, max_sweeps=10, sketch="leverage-random", sketch_size=3200, seed=0)),
    "c3": (("dense", (120,) * 4, 8, 1e-3, 0), "tucker",
           dict(ranks=(8,) * 4, max_sweeps=10, sketch="tensorsketch", sketch_size=4096, seed=0)),
    "c4a": (("sparse", (2000,) * 3, 1_000_000, 0), "tucker",
            dict(ranks=(10,) * 3, max_sweeps=5, sketch="tensorsketch", sketch_size=1600, seed=0)),
    "c4b": (("sparse", (10_000,) * 3, 10_000_000, 0), "tucker",
            dict(ranks=(10,) * 3, max_sweeps=5, sketch="tensorsketch", sketch_size=1600, seed=0)),
    "c5a": (("sparse", (2000,) * 3, 1_000_000, 0), "cp",
            dict(rank=10, tucker_rank=20, sketch_factor=16,
                 tucker_sweeps=5, max_sweeps=50, seed=0)),
    "c5b": (("sparse", (10_000,) * 3, 10_000_000, 0), "cp",
            dict(rank=10, tucker_rank=20, sketch_factor=16,
                 tucker_sweeps=5, max_sweeps=50, seed=0)),
}


def make_input(spec):
    if spec[0] == "dense":
        _, shape, r, noise, seed = spec
        return planted_tucker_dense(shape, r, noise, seed)
    _, shape, nnz, seed = spec
    c, v = planted_cp_coo_host(shape, nnz, rank=10, seed=seed)
    return ref.SparseTensor(shape, c, v)


class Recorder:
    """Wraps sketchals.tucker's ts_apply_rhs / lev_build to observe them."""

    def __init__(self):
        self.rhs = []
        self.lev = []

    def __enter__(self):
        self._rhs = ref_tucker.ts_apply_rhs
        self._lev = ref_tucker.lev_build
        rec = self

        def rhs(ts, b, *a, **k):
            y = rec._rhs(ts, b, *a, **k)
            rec.rhs.append(np.array(y, copy=True))
            return y

        def lev(factors, m, variant, rng):
            s = rec._lev(factors, m, variant, rng)
            rec.lev.append((np.array(s.indices, copy=True), np.array(s.weights, copy=True)))
            return s

        ref_tucker.ts_apply_rhs = rhs
        ref_tucker.lev_build = lev
        return self

    def __exit__(self, *exc):
        ref_tucker.ts_apply_rhs = self._rhs
        ref_tucker.lev_build = self._lev


def cp_via_tucker_rank(t, rank, tucker_rank, sketch_factor, tucker_sweeps, max_sweeps, seed):
    """src/cp.py:177-224 with TuckerConfig.ranks = (tucker_rank,)*N (config 5)."""
    ndim = len(t.shape)
    seed_tucker, seed_cp = (s.generate_state(1)[0] for s in np.random.SeedSequence(seed).spawn(2))
    tcfg = ref.TuckerConfig(ranks=(tucker_rank,) * ndim, max_sweeps=tucker_sweeps,
                            sketch="leverage-random", sketch_factor=sketch_factor, init="rrf",
                            seed=int(seed_tucker))
    tmodel, ttrace = ref.sketched_tucker_als(t, tcfg)
    ccfg = ref.CPConfig(rank=rank, max_sweeps=max_sweeps, init="hosvd-of-core", seed=int(seed_cp))
    cmodel, ctrace = ref.cp_als(tmodel.core, ccfg, on_core=True)
    factors = [b @ a for b, a in zip(tmodel.factors, cmodel.factors)]
    weights = cmodel.weights.copy()
    normalized = []
    for a in factors:
        unit, norms = _normalize_columns(a)
        normalized.append(unit)
        weights *= norms
    model = ref.CPModel(normalized, weights)
    trace = ref.SweepTrace(fitness=list(ttrace.fitness) + [ref.fitness(t, model)],
                           residuals=list(ctrace.residuals),
                           wall_s=list(ttrace.wall_s) + [sum(ctrace.wall_s)],
                           stage_split=len(ttrace.fitness))
    return tmodel, ttrace, cmodel, model, trace


def put_factor(out, key, a):
    if a.shape[0] <= FULL_ROWS:
        out[key] = a
    else:
        out[key + "_head"] = a[:256]
        out[key + "_proj"] = a.T @ proj_matrix(a.shape[0], 8, 1)


def run_case(tag):
    spec, driver, cfg = CASES[tag]
    t = make_input(spec)
    out = {}
    with Recorder() as rec:
        tic = time.perf_counter()
        if driver == "tucker":
            model, trace = ref.sketched_tucker_als(t, ref.TuckerConfig(**cfg))
            tmodel = model
        else:
            tmodel, ttrace, cmodel, model, trace = cp_via_tucker_rank(t, **cfg)
        out[f"{tag}_seconds"] = np.array(time.perf_counter() - tic)
    out[f"{tag}_fitness"] = np.array(trace.fitness)
    out[f"{tag}_residuals"] = np.array(trace.residuals)
    out[f"{tag}_wall_s"] = np.array(trace.wall_s)
    if driver == "cp":
        out[f"{tag}_tucker_fitness"] = np.array(ttrace.fitness)
        out[f"{tag}_tucker_residuals"] = np.array(ttrace.residuals)
        out[f"{tag}_split"] = np.array(trace.stage_split)
        out[f"{tag}_cp_w"] = np.asarray(model.weights)
        for k, a in enumerate(model.factors):
            put_factor(out, f"{tag}_cp_a{k}", np.abs(a))  # CP columns: sign-free comparison
        out[f"{tag}_corecp_w"] = np.asarray(cmodel.weights)
    fac, core = canon(tmodel.factors, tmodel.core)
    out[f"{tag}_core"] = core
    for k, a in enumerate(fac):
        put_factor(out, f"{tag}_a{k}", a)
    for i, y in enumerate(rec.rhs):
        out[f"{tag}_rhs{i}_sha"] = np.array(sha(y))
        out[f"{tag}_rhs{i}_norm"] = np.array(np.linalg.norm(y))
        # Y_n (m x s_n) times a seeded Gaussian (s_n x 4)
        out[f"{tag}_rhs{i}_proj"] = y @ proj_matrix(y.shape[1], 4, 2)
    out[f"{tag}_n_rhs"] = np.array(len(rec.rhs))
    for i, (idx, w) in enumerate(rec.lev):
        out[f"{tag}_lev{i}_sha"] = np.array(sha(idx.astype(np.int64)))
        out[f"{tag}_lev{i}_wsha"] = np.array(sha(w))
        out[f"{tag}_lev{i}_wsum"] = np.array(w.sum())
    out[f"{tag}_n_lev"] = np.array(len(rec.lev))
    if rec.lev:
        out[f"{tag}_lev0_idx"] = rec.lev[0][0].astype(np.int32)
    return out


def main():
    tags = sys.argv[1:] or list(CASES)
    path = os.path.join(HERE, "configs.npz")
    out = dict(np.load(path)) if os.path.exists(path) else {}
    for tag in tags:
        tic = time.perf_counter()
        res = run_case(tag)
        for k in [k for k in out if k.startswith(tag + "_")]:
            del out[k]
        out.update(res)
        np.savez_compressed(path, **out)
        print(tag, f"{time.perf_counter() - tic:.1f}s", "fitness", res[f"{tag}_fitness"][-1], flush=True)
    print("wrote", path, len(out), "arrays", os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
