"""Aggregate an ncu report's per-CUDA-line warp-stall samples and executed
instructions:  python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, rows = "", []
    tot_s = tot_i = 0.0
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] in ("Function Name", "Line No") or len(r) < 8:
            continue
        if r[0] != "":
            try:
                s, i = float(r[4]), float(r[7])
            except ValueError:
                continue
            rows.append((s, i, f"{fname}:{r[0]}", r[1].strip()[:80]))
            tot_s += s
            tot_i += i
    print(f"samples {tot_s:.0f}  instructions {tot_i:.3e}")
    for s, i, loc, src in sorted(rows, reverse=True)[:top]:
        print(f"{100 * s / tot_s:5.1f}%  {i:11.3e}  {loc:22s} {src}")


if __name__ == "__main__":
    main()
