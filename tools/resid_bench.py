"""Time the rank-constrained solve's residual pass (skx_resid_sq) alone at the
config-4 shape (Y^T 1e5 x 1600, R = 10) and check it against torch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2104_01101_b200.linalg import resid_dev  # noqa: E402


def main():
    s, m, r2, R = 100_000, 1600, 100, int(sys.argv[1]) if len(sys.argv) > 1 else 10
    g = torch.Generator(device="cuda").manual_seed(0)
    yt = torch.randn(s, m, dtype=torch.float64, device="cuda", generator=g)
    z = torch.randn(m, r2, dtype=torch.float64, device="cuda", generator=g) * 0.1
    core_t = torch.randn(r2, R, dtype=torch.float64, device="cuda", generator=g) * 0.1
    a = torch.randn(s, R, dtype=torch.float64, device="cuda", generator=g)
    y = yt.t()
    ref = torch.linalg.vector_norm(z @ core_t @ a.t() - y)
    got = resid_dev(z, core_t, a, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        resid_dev(z, core_t, a, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"R={R} resid {ms:.3f} ms  {s * m * 8 / ms / 1e6:.0f} GB/s  rel.err {float(abs(got - ref) / ref):.2e}")


if __name__ == "__main__":
    main()
