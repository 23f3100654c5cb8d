"""Time the sparse Tucker cross term <T, [[G; A0, A1, A2]]> (skx_tucker_cross_coo,
the fitness kernel) alone on the bench's config-4 tensor with CUDA events.

    python tools/cross_bench.py [--nnz 1e8] [--side 100000] [--rank 10]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2104_01101_b200 as skx  # noqa: E402
from paper_2104_01101_b200.synth import planted_cp_coo_device  # noqa: E402
from paper_2104_01101_b200.tensors import cp_cross_dev, device_of, tucker_cross_dev  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nnz", type=float, default=1e8)
    ap.add_argument("--side", type=int, default=100_000)
    ap.add_argument("--rank", type=int, default=10)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cp-rank", type=int, default=10)
    a = ap.parse_args()
    shape = (a.side,) * 3
    coords, vals = planted_cp_coo_device(shape, int(a.nnz), rank=10, noise_sd=0.1, seed=0)
    st = skx.SparseTensor.from_device(shape, coords, vals, validate=False)
    d = device_of(st)
    g = torch.Generator(device="cuda").manual_seed(0)
    fac = [torch.linalg.qr(torch.randn(s, a.rank, dtype=torch.float64, device="cuda", generator=g))[0]
           for s in shape]
    core = torch.randn(a.rank, a.rank, a.rank, dtype=torch.float64, device="cuda", generator=g)
    d.fibre(0)
    x = tucker_cross_dev(d, core, fac)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        tucker_cross_dev(d, core, fac)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    print(f"tucker cross: {ms:.3f} ms  value {float(x):.12e}", flush=True)
    w = torch.rand(a.cp_rank, dtype=torch.float64, device="cuda", generator=g)
    cf = [f[:, :a.cp_rank].contiguous() for f in fac]
    y = cp_cross_dev(d, cf, w)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.reps):
        cp_cross_dev(d, cf, w)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    print(f"cp cross (R={a.cp_rank}): {ms:.3f} ms  value {float(y):.12e}", flush=True)
    if a.rank == 20:  # full TTMc (Alg. 6's last fitness pass): <P, C> = the Tucker cross term
        from paper_2104_01101_b200.tensors import ttmc3_full_dev
        P = ttmc3_full_dev(d, fac)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            ttmc3_full_dev(d, fac)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(f"full ttmc: {ms:.3f} ms  <P, C> {float((P * core).sum()):.12e}", flush=True)


if __name__ == "__main__":
    main()
