"""Time the RRF CountSketch stage 1 (skx_rrf_stage1_coo, K4) alone on the
config-4 tensor (mode 1, k2 = 140) with CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2104_01101_b200 as skx  # noqa: E402
from paper_2104_01101_b200.sketching import draw_rrf_tables  # noqa: E402
from paper_2104_01101_b200.synth import planted_cp_coo_device  # noqa: E402
from paper_2104_01101_b200.tensors import device_of  # noqa: E402
from paper_2104_01101_b200.tucker import rrf_stage1_dev  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    shape = (100_000,) * 3
    coords, vals = planted_cp_coo_device(shape, 100_000_000, rank=10, noise_sd=0.1, seed=0)
    st = skx.SparseTensor.from_device(shape, coords, vals, validate=False)
    d = device_of(st)
    P = shape[0] * shape[2]
    tabs = draw_rrf_tables(skx.make_rng(0), P, 140)
    d.fibre(1)
    rrf_stage1_dev(d, 1, tabs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        rrf_stage1_dev(d, 1, tabs)
    e1.record()
    torch.cuda.synchronize()
    print(f"rrf stage 1 (mode 1, k2=140): {e0.elapsed_time(e1) / reps:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
