#!/bin/bash
# ncu --set full of one skx_chol_inv_upper launch at n = 400 (config 5's r)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
args="--n 400 --reps 1 --lib-only"
python tools/chol_bench.py $args > gpurun_out/chol_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_chol_inv -s 1 -c 1 -o gpurun_out/chol \
  python tools/chol_bench.py $args > gpurun_out/chol_ncu.log 2>&1
echo rc=$?
ncu -i gpurun_out/chol.ncu-rep --page raw --csv 2>/dev/null | python tools/ncu_raw_summary.py > gpurun_out/chol_raw.txt 2>&1
python tools/ncu_lines.py gpurun_out/chol.ncu-rep 40 > gpurun_out/chol_lines.txt 2>&1
