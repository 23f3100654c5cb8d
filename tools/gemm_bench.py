"""Time the two rsvd_lrls passes over a TensorSketch right-hand side (Y G by
skx_gemm_atb, W^T Y by skx_gemm_ab) alone at config 4's shape (Y^T stored
1e5 x 1600, width 20) with CUDA events.  Development tool.

    python tools/gemm_bench.py [--m 1600] [--s 100000] [--w 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2104_01101_b200.linalg import ty_times_dev, y_times_dev  # noqa: E402


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1600)
    ap.add_argument("--s", type=int, default=100_000)
    ap.add_argument("--w", type=int, default=20)
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    yt = torch.randn(a.s, a.m, dtype=torch.float64, device="cuda", generator=g)
    y = yt.t()
    G = torch.randn(a.s, a.w, dtype=torch.float64, device="cuda", generator=g)
    W = torch.randn(a.m, a.w, dtype=torch.float64, device="cuda", generator=g)
    gb = yt.numel() * 8 / 1e9
    t1 = timed(lambda: y_times_dev(y, G))
    t2 = timed(lambda: ty_times_dev(W, y))
    print(f"Y G  (atb): {t1:.3f} ms  {gb / t1:.2f} TB/s")
    print(f"W^T Y (ab): {t2:.3f} ms  {gb / t2:.2f} TB/s", flush=True)


if __name__ == "__main__":
    main()
