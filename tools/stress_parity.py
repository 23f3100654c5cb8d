"""Randomised parity sweep (development tool): sketched_tucker_als on the GPU
against the CPU oracle for random small shapes / orders / ranks / sketches,
dense and sparse.  Prints one line per case and a summary; exit 1 on any
mismatch beyond 1e-9 (factors and core after sign canonicalisation).

    python tools/stress_parity.py [n_cases=24] [seed=0] [scale=1]

scale > 1 multiplies the extents (larger kernels paths: packed TS layouts,
tagged shared-memory accumulation, multi-block TSQR).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2104_01101_b200 as skx  # noqa: E402
from oracle import sketchals_port as oracle  # noqa: E402
from tests.conftest import canon, relerr  # noqa: E402


def main():
    n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    worst, bad = 0.0, 0
    for case in range(n_cases):
        nd = int(rng.choice([3, 3, 3, 4]))
        shape = tuple(int(x * (scale if nd == 3 else 1)) for x in
                      rng.integers(9, 40 if nd == 3 else 14, nd))
        ranks = tuple(int(min(s - 1, x)) for s, x in zip(shape, rng.integers(2, 6, nd)))
        sketch = str(rng.choice(["tensorsketch", "leverage-random"]))
        sparse = bool(rng.integers(0, 2))
        need = max(int(np.prod([ranks[k] for k in range(nd) if k != j])) for j in range(nd))
        m = int(need * rng.uniform(2.5, 6.0))
        seed = int(rng.integers(0, 1000))
        if sparse:
            nnz = int(min(np.prod(shape) * rng.uniform(0.05, 0.3), 300_000))
            lin = np.sort(rng.choice(int(np.prod(shape)), size=nnz, replace=False))
            coords = np.stack(np.unravel_index(lin, shape), axis=1)
            vals = rng.standard_normal(nnz)
            t_gpu = skx.SparseTensor(shape, coords, vals)
            t_ref = oracle.Coo(shape, coords, vals)
        else:
            t_gpu = t_ref = rng.standard_normal(shape)
        cfg = dict(ranks=ranks, max_sweeps=3, sketch=sketch, sketch_size=m, seed=seed)
        try:
            model, tr = skx.sketched_tucker_als(t_gpu, skx.TuckerConfig(**cfg))
            core, fac, otr = oracle.sketched_tucker(t_ref, ranks, sketch, max_sweeps=3,
                                                    sketch_size=m, seed=seed)
        except Exception as exc:  # both sides should agree on errors
            print(f"case {case}: {shape} {ranks} {sketch} sparse={sparse} m={m}: {type(exc).__name__}: {exc}")
            continue
        gf, gc = canon(model.factors, model.core)
        rf, rc = canon(fac, core)
        err = max([relerr(a, b) for a, b in zip(gf, rf)] + [relerr(gc, rc)])
        fe = float(np.max(np.abs(np.array(tr.fitness) - np.array(otr.fitness))))
        worst = max(worst, err)
        flag = err > 1e-9 or fe > 1e-9
        bad += flag
        print(f"case {case}: shape={shape} ranks={ranks} {sketch[:3]} sparse={sparse} m={m} "
              f"err={err:.2e} fit_err={fe:.2e}{'  MISMATCH' if flag else ''}", flush=True)
    print(f"{n_cases} cases, worst {worst:.2e}, mismatches {bad}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
