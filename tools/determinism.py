"""Run one bench config twice on the same device tensor and report where the
two runs first differ bitwise (RRF init factors, per-sweep residuals and
fitness, final factors).  Development tool; not part of the product path.

    python tools/determinism.py [--config 5] [--runs 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--nnz", type=int, default=0)
    args = ap.parse_args()
    import torch

    import bench
    import paper_2104_01101_b200 as skx
    from paper_2104_01101_b200 import tucker
    from paper_2104_01101_b200.cp import cp_via_sketched_tucker_dev
    from paper_2104_01101_b200.synth import planted_cp_coo_device

    cfgd = dict(bench.CONFIGS[args.config])
    if args.nnz:
        cfgd["nnz"] = args.nnz
    cfg = bench.tucker_config(skx, cfgd)
    coords, vals = planted_cp_coo_device(cfgd["shape"], cfgd["nnz"], rank=10, noise_sd=0.1, seed=0)
    st = skx.SparseTensor.from_device(cfgd["shape"], coords.t().contiguous(), vals, validate=False)
    del coords, vals

    snaps = []
    orig_init = tucker._Run.initialise_and_prep

    def init_hook(self):
        orig_init(self)
        torch.cuda.synchronize()
        snaps[-1]["init"] = [None if f is None else f.clone() for f in self.factors]

    orig_rhs = tucker._Run._rhs

    def rhs_hook(self, n, *a, **k):
        out = orig_rhs(self, n, *a, **k)
        torch.cuda.synchronize()
        snaps[-1].setdefault("rhs", []).append(
            tuple(x.clone() if torch.is_tensor(x) else x for x in (out if isinstance(out, tuple) else (out,))))
        return out

    tucker._Run.initialise_and_prep = init_hook
    tucker._Run._rhs = rhs_hook
    for _ in range(args.runs):
        snaps.append({})
        st._device.release_layouts()
        if cfgd["kind"] == "alg6":
            fac, w, tr = cp_via_sketched_tucker_dev(st, cfg)
        else:
            core, fac, tr = tucker.sketched_tucker_als_dev(st, cfg)
        torch.cuda.synchronize()
        snaps[-1]["trace"] = (list(tr.fitness), list(tr.residuals))
        snaps[-1]["final"] = [f.clone() for f in fac]

    a, b = snaps[0], snaps[1]
    for n, (x, y) in enumerate(zip(a["init"], b["init"])):
        if x is None:
            continue
        eq = torch.equal(x, y)
        print(f"init factor {n}: equal={eq} maxdiff={(x - y).abs().max().item():.3e}")
    for i, (x, y) in enumerate(zip(a.get("rhs", []), b.get("rhs", []))):
        for j, (u, v) in enumerate(zip(x, y)):
            if torch.is_tensor(u):
                eq = torch.equal(u, v)
                if not eq:
                    print(f"rhs call {i} item {j}: differs maxdiff={(u - v).abs().max().item():.3e} "
                          f"shape={tuple(u.shape)}")
    fa, ra = a["trace"]
    fb, rb = b["trace"]
    print("fitness a", fa)
    print("fitness b", fb)
    print("resid   a", ra)
    print("resid   b", rb)
    for n, (x, y) in enumerate(zip(a["final"], b["final"])):
        print(f"final factor {n}: equal={torch.equal(x, y)} maxdiff={(x - y).abs().max().item():.3e}")


if __name__ == "__main__":
    main()
