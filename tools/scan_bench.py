"""Time skx_lemire_scan alone over a config-4-sized range (5e9 raw words,
bound k2 = 130) with CUDA events.  Development tool."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2104_01101_b200 import _native as nat  # noqa: E402


def main():
    raw = int(float(sys.argv[1])) if len(sys.argv) > 1 else 5_000_000_000
    k2 = 130
    cap = 1 << 16
    rej = torch.empty(cap, dtype=torch.int64, device="cuda")
    count = torch.zeros(1, dtype=torch.int64, device="cuda")

    def run():
        count.zero_()
        nat.call("skx_lemire_scan", ctypes.c_uint64(12345), ctypes.c_uint64(678), ctypes.c_uint64(0),
                 ctypes.c_uint64(raw), ctypes.c_uint32(k2), nat.ptr(rej), cap, nat.ptr(count),
                 nat.stream())
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"scan {raw:.3g} raw words: {ms:.2f} ms  "
          f"{raw / 4 / ms / 1e6:.1f} Gblocks/s  rejections {int(count.item())}", flush=True)


if __name__ == "__main__":
    main()
