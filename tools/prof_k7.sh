#!/bin/bash
# ncu --set full of one K7 launch (config-5 shape, R = 20) via tools/cross_bench.py;
# the plain command runs first (it must exit 0 before ncu touches it).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
tag=${1:-k7}
kre=${2:-k_tucker3}
args="--side 200000 --nnz 1e9 --rank 20 --reps 1"
python tools/cross_bench.py $args > gpurun_out/${tag}_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:$kre -c 1 -o gpurun_out/$tag \
  python tools/cross_bench.py $args > gpurun_out/${tag}.log 2>&1
echo rc=$?
ncu -i gpurun_out/$tag.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/${tag}_rawfull.csv
python tools/ncu_raw_summary.py < gpurun_out/${tag}_rawfull.csv > gpurun_out/${tag}_raw.txt 2>&1
python tools/ncu_lines.py gpurun_out/$tag.ncu-rep 30 > gpurun_out/${tag}_lines.txt 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>/dev/null
gzip -f gpurun_out/${tag}_rawfull.csv
