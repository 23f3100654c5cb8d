"""GPU timeline of one sketched_tucker_als run (torch.profiler / CUPTI).

    python tools/timeline.py [--config 4] [--out gpurun_out/trace.json]

Prints per-kernel totals, GPU busy time per stream and the idle gaps of the
main stream, so host stalls (syncs, Python overhead) are visible next to
kernel time.  Development tool; not part of the product path.
"""
import argparse
import collections
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "trace.json"))
    ap.add_argument("--e2e", action="store_true",
                    help="sparse configs: time the public call on a pinned host copy (upload included)")
    ap.add_argument("--window", default="",
                    help="KERNEL:i:j -- list every kernel (all streams) between the start of the "
                         "i-th and the j-th launch of KERNEL (substring), with gaps")
    ap.add_argument("--gantt", type=float, default=0.0,
                    help="also list, in start order, every kernel longer than this many ms")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    import paper_2104_01101_b200 as skx
    from paper_2104_01101_b200.synth import planted_cp_coo_device
    from paper_2104_01101_b200.tucker import sketched_tucker_als_dev

    cfgd = bench.CONFIGS[args.config]
    if cfgd["kind"] != "dense":
        coords, vals = planted_cp_coo_device(cfgd["shape"], cfgd["nnz"], rank=10, noise_sd=0.1,
                                             seed=0)
        st = skx.SparseTensor.from_device(cfgd["shape"], coords.t().contiguous(), vals)
        del coords, vals
    else:
        st = torch.from_numpy(bench.dense_input_host(cfgd)).cuda()
    cfg = bench.tucker_config(skx, cfgd)
    sparse = not torch.is_tensor(st)
    from paper_2104_01101_b200.cp import cp_via_sketched_tucker_dev
    alg6 = cfgd["kind"] == "alg6"
    if args.e2e and sparse:
        dev = st._device
        hc = torch.empty((dev.nnz, dev.ndim), dtype=torch.int64, pin_memory=True)
        hv = torch.empty(dev.nnz, dtype=torch.float64, pin_memory=True)
        chunk = 1 << 26
        for lo in range(0, dev.nnz, chunk):
            hc[lo:min(dev.nnz, lo + chunk)].copy_(dev.coords[:, lo:lo + chunk].t().to(torch.int64))
        hv.copy_(dev.vals)
        st = skx.SparseTensor.from_sorted(cfgd["shape"], hc.numpy(), hv.numpy())
        del dev
        torch.cuda.empty_cache()

        def call():
            st._device = None
            (skx.cp_via_sketched_tucker if alg6 else skx.sketched_tucker_als)(st, cfg)
    else:
        def call():
            if sparse:
                st._device.release_layouts()
            if alg6:
                cp_via_sketched_tucker_dev(st, cfg)
            else:
                sketched_tucker_als_dev(st, cfg)
    for _ in range(2):
        call()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        call()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    prof.export_chrome_trace(args.out)
    ev = json.load(open(args.out))["traceEvents"]
    kern = [e for e in ev if e.get("cat") == "kernel"]
    per = collections.defaultdict(lambda: [0, 0.0])
    streams = collections.defaultdict(float)
    for e in kern:
        nm = e["name"][:70]
        per[nm][0] += 1
        per[nm][1] += e["dur"]
        streams[e["args"].get("stream")] += e["dur"]
    t_lo = min(e["ts"] for e in kern)
    t_hi = max(e["ts"] + e["dur"] for e in kern)
    print(f"wall {wall * 1e3:.1f} ms; kernel span {(t_hi - t_lo) / 1e3:.1f} ms; "
          f"kernel sum {sum(v[1] for v in per.values()) / 1e3:.1f} ms")
    for s, d in streams.items():
        print(f"  stream {s}: {d / 1e3:.1f} ms busy")
    # idle gaps on the union of streams
    iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in kern)
    gaps, cur = [], iv[0][1]
    for a, b in iv[1:]:
        if a > cur:
            gaps.append(a - cur)
        cur = max(cur, b)
    print(f"  idle (no kernel on any stream): {sum(gaps) / 1e3:.1f} ms in {len(gaps)} gaps; "
          f"largest {sorted(gaps)[-5:] if gaps else []} us")
    for nm, (c, d) in sorted(per.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"{d / 1e3:9.3f} ms {c:5d}  {nm}")
    if args.window:
        name, i, j = args.window.split(":")
        marks = sorted(e["ts"] for e in kern if name in e["name"])
        lo, hi = marks[int(i)], marks[int(j)]
        print(f"window {name}[{i}]..[{j}]: {(hi - lo) / 1e3:.3f} ms")
        prev = {}
        for e in sorted(kern, key=lambda e: e["ts"]):
            if lo <= e["ts"] < hi:
                st = e["args"].get("stream")
                gap = e["ts"] - prev.get(st, e["ts"])
                prev[st] = e["ts"] + e["dur"]
                print(f"{(e['ts'] - lo) / 1e3:8.3f} {e['dur']:9.1f}us gap{gap:8.1f}us s{st!s:>3}  "
                      f"{e['name'][:90]}")
    if args.gantt > 0:
        print("start_ms  dur_ms  stream  kernel")
        for e in sorted(kern, key=lambda e: e["ts"]):
            if e["dur"] >= args.gantt * 1e3:
                print(f"{(e['ts'] - t_lo) / 1e3:8.2f} {e['dur'] / 1e3:7.3f} {e['args'].get('stream')!s:>6}  "
                      f"{e['name'][:60]}")


if __name__ == "__main__":
    main()
