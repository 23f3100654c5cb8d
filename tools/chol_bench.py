"""Time the wide-system Cholesky (+ inverse) alone: libskx skx_chol_inv_upper
vs cuSOLVER potrf + a TRSM against I (torch), n = 128..512.

    python tools/chol_bench.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2104_01101_b200.linalg import chol_inv_upper_dev  # noqa: E402


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


import argparse  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="*", default=[128, 256, 400, 512])
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--lib-only", action="store_true")
args = ap.parse_args()

for n in args.n:
    z = torch.randn(4 * n, n, dtype=torch.float64, device="cuda")
    g = z.t() @ z
    eye = torch.eye(n, dtype=torch.float64, device="cuda")

    def lib():
        return chol_inv_upper_dev(g)

    def cus():
        u, _ = torch.linalg.cholesky_ex(g, upper=True)
        return torch.linalg.solve_triangular(u, eye, upper=True)

    if args.lib_only:
        print(f"n={n}: libskx chol+inv {timeit(lib, args.reps):.3f} ms")
        continue
    print(f"n={n}: libskx chol+inv {timeit(lib, args.reps):.3f} ms   "
          f"cuSOLVER potrf + trsm(I) {timeit(cus, args.reps):.3f} ms")
