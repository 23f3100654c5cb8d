"""Time K8 (skx_cp_core_als: CP-ALS on the 20^3 core, rank 10, 50 sweeps --
Algorithm 6's second stage at config 5) alone with CUDA events.

    python tools/cp_core_bench.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2104_01101_b200 as skx  # noqa: E402
from paper_2104_01101_b200.cp import cp_core_als_dev  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
core = torch.randn(20, 20, 20, dtype=torch.float64, device="cuda", generator=g)
cfg = skx.CPConfig(rank=10, max_sweeps=50, init="hosvd-of-core", seed=0)
for _ in range(3):
    cp_core_als_dev(core, cfg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    cp_core_als_dev(core, cfg)
e1.record()
torch.cuda.synchronize()
print(f"cp core (20^3, R=10, 50 sweeps): {e0.elapsed_time(e1) / 10:.3f} ms per call (incl. D2H of the trace)")
