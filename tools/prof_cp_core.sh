#!/bin/bash
# ncu --set full of one K8 launch (CP-ALS on the 20^3 core, 50 sweeps)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python tools/cp_core_bench.py > gpurun_out/cpc_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_cp_core_als -s 3 -c 1 -o gpurun_out/cpc \
  python tools/cp_core_bench.py > gpurun_out/cpc_ncu.log 2>&1
echo rc=$?
ncu -i gpurun_out/cpc.ncu-rep --page raw --csv 2>/dev/null | python tools/ncu_raw_summary.py > gpurun_out/cpc_raw.txt 2>&1
python tools/ncu_lines.py gpurun_out/cpc.ncu-rep 40 > gpurun_out/cpc_lines.txt 2>&1
rm -f gpurun_out/cpc.ncu-rep
