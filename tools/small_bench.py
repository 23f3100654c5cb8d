"""Time the single-CTA dense kernels (Cholesky, Jacobi SVD, TSQR) at the
config-4 sizes with CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2104_01101_b200 import _native as nat  # noqa: E402
from paper_2104_01101_b200.linalg import chol_upper_dev, jacobi_svd_dev, tsqr_r_dev  # noqa: E402


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    z = torch.randn(1600, 100, dtype=torch.float64, device="cuda", generator=g)
    gram = z.t() @ z
    print(f"chol n=100: {timeit(lambda: chol_upper_dev(gram)):.1f} us")
    for n in (20, 40):
        a = torch.randn(100_000, n, dtype=torch.float64, device="cuda", generator=g)
        r = tsqr_r_dev(a)
        print(f"tsqr 1e5 x {n}: {timeit(lambda: tsqr_r_dev(a)):.1f} us")
        print(f"jacobi n={n} (R of gaussian): {timeit(lambda: jacobi_svd_dev(r)):.1f} us")
        lr = torch.randn(n, 10, dtype=torch.float64, device="cuda", generator=g) @ torch.randn(
            10, n, dtype=torch.float64, device="cuda", generator=g)
        print(f"jacobi n={n} (rank 10): {timeit(lambda: jacobi_svd_dev(lr)):.1f} us")
    qz, rz = torch.linalg.qr(z)
    for w in (20, 30):
        b = torch.randn(100, w, dtype=torch.float64, device="cuda", generator=g)
        q = torch.empty_like(b)
        x = torch.empty_like(b)

        def mid():
            nat.call("skx_lrls_mid", nat.ptr(rz), nat.ptr(b), 100, w, nat.ptr(q), nat.ptr(x),
                     nat.stream())
        print(f"lrls_mid r=100 w={w}: {timeit(mid):.1f} us")




def torch_chol():
    g = torch.Generator(device="cuda").manual_seed(0)
    z = torch.randn(1600, 100, dtype=torch.float64, device="cuda", generator=g)
    gram = z.t() @ z
    print(f"torch.linalg.cholesky_ex n=100: {timeit(lambda: torch.linalg.cholesky_ex(gram, upper=True)):.1f} us")
    print(f"chol_upper_dev n=100: {timeit(lambda: chol_upper_dev(gram)):.1f} us")


if __name__ == "__main__":
    main()
    torch_chol()
