"""Time the sparse TensorSketch right-hand side (skx_ts_rhs_coo) alone on the
bench's config-4 tensor, per mode, with CUDA events.

    python tools/k1_bench.py [--nnz 1e8] [--side 100000] [--m 1600]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2104_01101_b200 as skx  # noqa: E402
from paper_2104_01101_b200.sketching import ts_rhs_coo_dev, ts_rhs_mode_dev  # noqa: E402
from paper_2104_01101_b200.synth import planted_cp_coo_device  # noqa: E402
from paper_2104_01101_b200.tensors import device_of  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nnz", type=float, default=1e8)
    ap.add_argument("--side", type=int, default=100_000)
    ap.add_argument("--m", type=int, default=1600)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    shape = (a.side,) * 3
    coords, vals = planted_cp_coo_device(shape, int(a.nnz), rank=10, noise_sd=0.1, seed=0)
    st = skx.SparseTensor.from_device(shape, coords, vals, validate=False)
    d = device_of(st)
    nnz = int(vals.numel())
    for packed in (False, True):
        for n in range(3):
            ext = tuple(shape[k] for k in range(3) if k != n)
            op = skx.TensorSketchOp.build(ext, a.m, skx.make_rng(n))
            if packed:
                def run():
                    return ts_rhs_mode_dev(op, d, n)
            else:
                colptr, rec = d.fibre(n)

                def run():
                    return ts_rhs_coo_dev(op, colptr, rec, shape[n])
            run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            gb = (nnz * 16 + shape[n] * a.m * 8 + (shape[n] + 1) * 8) / 1e9
            print(f"{'packed' if packed else 'lookup'} mode {n}: {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s "
                  f"algorithmic ({gb:.2f} GB)", flush=True)
            d.release_layouts()

if __name__ == "__main__":
    main()
