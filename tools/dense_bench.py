"""Time the dense TensorSketch right-hand side (skx_ts_rhs_dense, K1d) on the
config-3 shape (120^4 float64, m = 4096) per mode with CUDA events.

    python tools/dense_bench.py [shape=120,120,120,120] [m=4096] [modes=0,1,2,3]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2104_01101_b200 as skx  # noqa: E402
from paper_2104_01101_b200.sketching import ts_rhs_dense_dev  # noqa: E402


def main():
    shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "120,120,120,120").split(","))
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    g = torch.Generator(device="cuda").manual_seed(0)
    t = torch.randn(shape, dtype=torch.float64, device="cuda", generator=g)
    modes = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else range(len(shape))
    for n in modes:
        ext = tuple(shape[k] for k in range(len(shape)) if k != n)
        op = skx.TensorSketchOp.build(ext, m, skx.make_rng(n))
        ts_rhs_dense_dev(op, t, n)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            ts_rhs_dense_dev(op, t, n)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        gb = (t.numel() * 8 + shape[n] * m * 8) / 1e9
        print(f"dense mode {n}: {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s ({gb:.2f} GB)", flush=True)


if __name__ == "__main__":
    main()
