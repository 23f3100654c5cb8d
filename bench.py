"""Benchmark: sketched Tucker-ALS sweeps/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4]

Workload (default, N=1): BASELINE config 4 -- sparse order-3 COO 1e5^3 with
1e8 distinct uniform-random nonzeros, values = planted CP rank-10 model
(U(0,1) factors) + N(0, 0.01) noise; Tucker rank 10, TensorSketch m = 1600,
RRF init, 5 sweeps, seed 0.  Seeded synthetic data built on the GPU.

A step = one complete ``sketched_tucker_als`` call: per-mode layouts, RRF
initialisation, TensorSketch right-hand sides, 5 sweeps (15 sub-problems) and
the per-sweep fitness pass.  value = sweeps completed / time (whole job).
`e2e` = the same through the public API with HOST (pinned) input buffers:
H2D of coords+values, the call, and D2H of the model inside the timed region.
Under torchrun (N>1) nonzeros are sharded in mode-0 slabs (paper_2104_01101_b200
.dist); partial sketches are summed with NCCL all-reduce.

--impl reference: the CPU oracle (a restatement of the reference package;
the reference itself is pure numpy/scipy and cannot run config 4 at full
scale -- its unfoldings need >= 80 GB) timed on a bounded sample of the same
workload and reported per-nnz-scaled to the full size (labelled).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    4: dict(workload="cfg4: sparse COO 1e5^3, 1e8 nnz, planted CP-10 + N(0,0.01); Tucker R=10, "
                     "TensorSketch m=1600, RRF init, 5 sweeps, seed 0",
            shape=(100_000,) * 3, nnz=100_000_000, ranks=(10, 10, 10), sketch="tensorsketch",
            sketch_size=1600, sweeps=5),
    5: dict(workload="cfg5 Tucker stage: sparse COO 2e5^3, 1e9 nnz, planted CP-10; Tucker R=20, "
                     "leverage sampling m=6400, RRF init, 5 sweeps, seed 0",
            shape=(200_000,) * 3, nnz=1_000_000_000, ranks=(20, 20, 20), sketch="leverage-random",
            sketch_size=6400, sweeps=5),
}
SAMPLE = {4: dict(shape=(2000,) * 3, nnz=1_000_000), 5: dict(shape=(2000,) * 3, nnz=1_000_000)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (recipe's clocks line)."""

    def __init__(self):
        self.proc = None
        self.lines = []

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            dev = os.environ.get("LOCAL_RANK", "0")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", dev, f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ our arm
def run_ours(args, cfgd):
    import numpy as np
    import torch
    import paper_2104_01101_b200 as skx
    from paper_2104_01101_b200 import _native as nat
    from paper_2104_01101_b200.synth import planted_cp_coo_device
    from paper_2104_01101_b200.tucker import sketched_tucker_als_dev

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: SKX_BENCH_SHARE_GPU=1 runs every rank on cuda:0 over gloo (the
    # multi-rank logic on a one-GPU box; never used for a reported number)
    share = os.environ.get("SKX_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        import torch.distributed as dist
        from paper_2104_01101_b200.dist import Comm
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = Comm()
    nat.load()

    shape, nnz = cfgd["shape"], cfgd["nnz"]
    coords, vals = planted_cp_coo_device(shape, nnz, rank=10, noise_sd=0.1, seed=0)
    if world > 1:
        from paper_2104_01101_b200.dist import shard_device_coo
        coords, vals, _ = shard_device_coo(coords.t().contiguous(), vals, shape, world, rank)
    else:
        coords = coords.t().contiguous()
    st = skx.SparseTensor.from_device(shape, coords, vals, validate=True)
    dev = st._device
    cfg = skx.TuckerConfig(ranks=cfgd["ranks"], max_sweeps=cfgd["sweeps"], sketch=cfgd["sketch"],
                           sketch_size=cfgd["sketch_size"], seed=0)
    local_nnz = dev.nnz

    def step():
        dev.release_layouts()  # each step rebuilds its per-mode layouts
        core, fac, trace = sketched_tucker_als_dev(st, cfg, comm)
        return trace

    def barrier():
        if comm is not None:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        trace = step()
    # ---- device-resident timed region
    hook_names = ["skx_ts_rhs_coo", "skx_rrf_stage1_coo", "skx_lemire_scan", "skx_tucker_cross_coo",
                  "skx_resid_sq", "skx_ts_kron_apply", "skx_philox_normal", "skx_tsqr_r"]
    sinks = {nm: [] for nm in hook_names}
    for nm in hook_names:
        nat.set_event_hook(nm, sinks[nm])
    clocks = Clocks()
    clocks.start()
    barrier()
    l0 = nat.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    wall_s = []
    for _ in range(args.steps):
        trace = step()
        wall_s.append(sum(trace.wall_s))
    e1.record()
    barrier()
    launches = nat.launch_count() - l0
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    for nm in hook_names:
        nat.set_event_hook(nm, None)
    kern = {}
    for nm, evs in sinks.items():
        if evs:
            tot = sum(a.elapsed_time(b) for a, b, _ in evs)
            kern[nm] = {"launches": len(evs), "ms_total": tot, "ms_avg": tot / len(evs)}
            if nm == "skx_lemire_scan":
                # Philox4x64-10 blocks scanned (4 raw words each): args 2, 3 = raw_lo, raw_hi
                nblk = sum((int(ar[3].value) - 1) // 4 - int(ar[2].value) // 4 + 1
                           for _, _, ar in evs)
                kern[nm]["philox_blocks"] = nblk
    t_max = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if comm is not None:
        import torch.distributed as dist
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms = float(t_max.item())
    sweeps = cfgd["sweeps"] * args.steps
    value = sweeps / (ms / 1e3)

    # ---- the roofline kernel timed alone (CUDA events, same data): inside the
    # call it co-runs with the compute-bound rejection scans, which share its SMs
    k1_alone = None
    if cfgd["sketch"] == "tensorsketch":
        from paper_2104_01101_b200.sketching import ts_rhs_mode_dev
        op = skx.TensorSketchOp.build(tuple(shape[1:]), cfgd["sketch_size"], skx.make_rng(12345))
        dev.release_layouts()  # mode 0's layout is rebuilt with this operator's buckets
        sink = []
        nat.set_event_hook("skx_ts_rhs_coo", sink)
        for _ in range(4):
            ts_rhs_mode_dev(op, dev, 0)
        torch.cuda.synchronize()
        nat.set_event_hook("skx_ts_rhs_coo", None)
        evs = sink[1:]
        k1_alone = sum(a.elapsed_time(b) for a, b, _ in evs) / len(evs)
        dev.release_layouts()
        del op

    # ---- e2e through the public API with pinned host buffers (rank 0 / N=1)
    e2e = None
    if world == 1 and not args.no_e2e:
        hc = torch.empty((local_nnz, 3), dtype=torch.int64, pin_memory=True)
        hv = torch.empty(local_nnz, dtype=torch.float64, pin_memory=True)
        hc.copy_(dev.coords.t().to(torch.int64))
        hv.copy_(dev.vals)
        host_st = skx.SparseTensor.from_sorted(shape, hc.numpy(), hv.numpy())
        del st, dev
        torch.cuda.empty_cache()
        h2d = hc.numel() * 8 + hv.numel() * 8
        d2h = 0
        for _ in range(max(1, args.warmup // 2)):
            host_st._device = None
            model, tr = skx.sketched_tucker_als(host_st, cfg)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            host_st._device = None  # fresh upload every step
            model, tr = skx.sketched_tucker_als(host_st, cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        d2h = int(sum(a.nbytes for a in model.factors) + model.core.nbytes + 8 * len(tr.fitness)
                  + 8 * len(tr.residuals))
        e2e = {"value": sweeps / dt, "unit": "sweeps/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3 / args.steps,
               "path": "paper_2104_01101_b200.sketched_tucker_als(SparseTensor(pinned host), cfg)"}

    # ---- roofline of the dominant libskx kernel
    peak, peak_kind = peaks()
    s_n = shape[0]
    m = cfgd["sketch_size"]
    # fibre-major layout read per launch: 2 int32 other-coords + f64 value per nnz,
    # colptr (s_n+1 int64), output Y^T s_n x m f64 written once
    alg_bytes = {
        "skx_ts_rhs_coo": local_nnz * 16 + (s_n + 1) * 8 + s_n * m * 8,
        "skx_rrf_stage1_coo": local_nnz * 16 + (s_n + 1) * 8 + s_n * (cfgd["ranks"][0] ** 2 + 40) * 8,
        "skx_tucker_cross_coo": local_nnz * 20 + (s_n + 1) * 8,
        "skx_resid_sq": m * s_n * 8,
    }
    dom = max(kern.items(), key=lambda kv: kv[1]["ms_total"])[0] if kern else None
    roof_k = "skx_ts_rhs_coo" if "skx_ts_rhs_coo" in kern else dom
    roof = None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as fh:
            t = json.load(fh).get(roof_k)
        if t and world == 1 and args.config == 4:
            traffic = int(t["dram_read_bytes"] + t["dram_write_bytes"])
    except Exception:
        traffic = None
    if roof_k in kern and roof_k in alg_bytes:
        ach_pipe = alg_bytes[roof_k] / (kern[roof_k]["ms_avg"] / 1e3) / 1e9
        alone = roof_k == "skx_ts_rhs_coo" and k1_alone is not None
        ach = alg_bytes[roof_k] / (k1_alone / 1e3) / 1e9 if alone else ach_pipe
        roof = {"kernel": roof_k, "bound": "hbm", "achieved": round(ach, 1), "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": round(ach / peak, 4),
                "timing": ("3 launches alone on the bench tensor (mode 0), CUDA events; "
                           "in-pipeline figures below" if alone else "in-pipeline launches"),
                "in_pipeline": {"ms_avg": round(kern[roof_k]["ms_avg"], 4),
                                "achieved": round(ach_pipe, 1),
                                "frac": round(ach_pipe / peak, 4),
                                "note": "co-runs with the rejection scans (shared SMs)"},
                "traffic": traffic, "traffic_source": "profiles/r1_traffic.json (ncu --set full)",
                "alg_bytes_per_launch": int(alg_bytes[roof_k]),
                "layout": "fibre-major COO records, 16 B/nnz: int32 c_a, int32 (c_b | bucket << bb "
                          "| sign << 31), f64 value (mode n's TensorSketch bucket/sign folded in "
                          "when the layout is built); canonical int64 COO would be 32 B/nnz"}

    # the rejection scans are compute-bound on the integer multiplier: 20
    # 64x64->128-bit products per Philox4x64-10 block against the measured
    # sustained rate of tools/scan_bench.py (7.17 per SM-cycle, B200)
    roof_scan = None
    sk = kern.get("skx_lemire_scan")
    if sk and sk.get("philox_blocks"):
        mhz = (clk or {}).get("sm_mhz") or 1965.0
        ach = sk["philox_blocks"] * 20 / (sk["ms_total"] / 1e3) / 1e12
        pk = 7.17 * torch.cuda.get_device_properties(0).multi_processor_count * mhz * 1e6 / 1e12
        roof_scan = {"kernel": "skx_lemire_scan", "bound": "int-mul (IMAD)",
                     "achieved": round(ach, 3), "peak": round(pk, 3),
                     "unit": "T mul64x64->128/s", "frac": round(ach / pk, 4),
                     "peak_source": "tools/scan_bench.py microbenchmark (7.17 per SM-cycle) x SMs x "
                                    "median SM clock", "note": "times include co-running work"}

    out = {
        "metric": "sketched-ALS sweeps/s (whole sketched_tucker_als call incl. RRF init, TS prep, "
                  "fitness)",
        "value": round(value, 4), "unit": "sweeps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, generated on GPU)",
        "config": {"workload": cfgd["workload"], "nnz": nnz, "shape": list(shape),
                   "parallelism": (f"nnz mode-0 slabs x{world}; NCCL reduce-scatter of Y_n by columns, "
                                   "column-sharded rsvd, split RRF scans") if world > 1 else "single GPU",
                   "l2": f"inputs ({nnz * 32 / 1e9:.1f} GB canonical COO) larger than L2 (126 MB): "
                         "no flush needed between steps",
                   "sweeps_per_step": cfgd["sweeps"],
                   "sweeps_per_s_ref_def": round(sweeps / sum(wall_s), 3),
                   "ref_def": "sweeps / sum(SweepTrace.wall_s): N sub-problems + core fold, "
                              "excluding init/prep/fitness (src/tucker.py:280-296)"},
        "roofline": roof,
        "kernels": {k: {kk: round(vv, 4) if isinstance(vv, float) else vv for kk, vv in v.items()}
                    for k, v in kern.items()},
        "dominant_kernel": dom,
        "roofline_dominant": roof_scan,
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args.config, cfgd)
    if rank == 0:
        print(json.dumps(out))
    if comm is not None:
        import torch.distributed as dist
        dist.destroy_process_group()


# ------------------------------------------------------------------ CPU side
def _oracle_sample(cfg_id, cfgd, reps=1):
    """Time the CPU oracle on the bounded sample; returns (sweeps/s scaled to
    the full nnz, raw sample sweeps/s, seconds per run, description)."""
    import numpy as np
    from oracle import sketchals_port as orc
    from paper_2104_01101_b200.synth import planted_cp_coo_host
    sm = SAMPLE[cfg_id]
    c, v = planted_cp_coo_host(sm["shape"], sm["nnz"], rank=10, noise_sd=0.1, seed=0)
    t = orc.Coo(sm["shape"], c, v, presorted=True)
    kw = dict(ranks=cfgd["ranks"], max_sweeps=cfgd["sweeps"], sketch=cfgd["sketch"],
              sketch_size=cfgd["sketch_size"], seed=0)
    best = None
    for _ in range(reps):
        t._cache.clear()
        t0 = time.perf_counter()
        orc.sketched_tucker(t, **kw)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    raw = cfgd["sweeps"] / best
    scaled = raw * sm["nnz"] / cfgd["nnz"]
    desc = (f"oracle (numpy/scipy restatement of the reference) on {sm['shape'][0]}^3 with "
            f"{sm['nnz']:.0e} nnz, same ranks/sketch/sweeps; {best:.2f} s per call = {raw:.3f} "
            f"sweeps/s; value scaled by nnz ratio {sm['nnz']}/{cfgd['nnz']} (extrapolated: the "
            f"reference cannot run the full size, its unfoldings need >= 80 GB)")
    return scaled, raw, best, desc


def cpu_baseline(cfg_id, cfgd):
    scaled, raw, secs, desc = _oracle_sample(cfg_id, cfgd)
    return {"value": scaled, "unit": "sweeps/s", "cores": os.cpu_count(), "kind": "port",
            "sample": desc, "sample_sweeps_per_s": raw}


def run_reference(args, cfgd):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    vals = []
    secs = []
    for i in range(args.warmup + args.steps):
        scaled, raw, s, desc = _oracle_sample(args.config, cfgd)
        if i >= args.warmup:
            vals.append(scaled)
            secs.append(s)
    v = sum(vals) / len(vals)
    out = {"metric": "sketched-ALS sweeps/s (whole sketched_tucker_als call incl. RRF init, TS prep, "
                     "fitness)", "value": v, "unit": "sweeps/s", "impl": "reference",
           "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / len(secs),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded)", "config": {"workload": cfgd["workload"]},
           "cpu_baseline": {"value": v, "unit": "sweeps/s", "cores": os.cpu_count(), "kind": "port",
                            "sample": desc},
           "e2e": {"value": v, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    cfgd = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfgd)
    else:
        run_ours(args, cfgd)


if __name__ == "__main__":
    main()
