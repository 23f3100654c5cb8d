"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv
--log-file X`) of `bench.py --steps 1 --warmup W`: per-kernel launches and
serialized time for the last `runs_tail` sketched_tucker_als calls (the run
boundary is the first k_lemire_scan launch of each call).

    python tools/launch_summary.py launches.csv [runs_tail=1]
"""
import collections
import csv
import gzip
import sys


def main():
    path = sys.argv[1]
    tail = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rows = []
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt") as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        us = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "ms":
            us *= 1e3
        elif r["Metric Unit"] == "ns":
            us /= 1e3
        rows.append((r["Kernel Name"], us))
    starts = [i for i, (k, _) in enumerate(rows) if "k_lemire_scan" in k]
    # two scans per call (modes 1 and 2): a call starts at every other scan
    calls = starts[::2]
    first = calls[-tail] if len(calls) >= tail else 0
    sel = rows[first:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, us in sel:
        name = k.split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += us
    total = sum(v[1] for v in agg.values())
    print(f"{len(sel)} launches, {total / 1e3:.3f} ms serialized (last {tail} call(s))")
    print("| kernel | launches | ms (ncu, serialized) | share |")
    print("|---|---|---|---|")
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"| `{k[:80]}` | {c} | {us / 1e3:.3f} | {100 * us / total:.1f}% |")


if __name__ == "__main__":
    main()
