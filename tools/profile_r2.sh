#!/bin/bash
# Round-2 profiling on the GPU box (config 5 unless stated):
#  1. launch list of one call: ncu --metrics gpu__time_duration.sum (gzip'ed csv)
#  2. ncu --set full of one launch of each dominant kernel, exported on the box
#     as compact csv (details page + selected raw metrics); only the K7 report
#     is kept (gpurun_out must stay under 64 MiB).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2_cfg5_launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2_ncu_list.log 2>&1
echo "launch list rc=$?"
gzip -f gpurun_out/r2_cfg5_launches.csv
summ() {  # $1 = report basename
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv 2>/dev/null | python tools/ncu_raw_summary.py \
    > gpurun_out/$1_raw.txt 2>&1
  python tools/ncu_lines.py gpurun_out/$1.ncu-rep 25 > gpurun_out/$1_lines.txt 2>&1
}
run() {  # $1 = kernel regex, $2 = tag, rest = bench args
  local k=$1 tag=$2; shift 2
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
    -o gpurun_out/$tag python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e "$@" \
    > gpurun_out/${tag}.log 2>&1
  echo "$tag rc=$?"
  summ $tag
}
run k_tucker3_async r2_cfg5_k7
run k_rrf_coo_fx r2_cfg5_fx
run k_lemire_scan r2_cfg5_scan
run k_cp3_fibre r2_cfg5_cp3
run k_filter_fibers r2_cfg5_filter
run k_tucker3_mma r2_cfg4_k7 --config 4
run k_ts_rhs_coo r2_cfg4_k1 --config 4
for f in gpurun_out/r2_*.ncu-rep; do
  case $f in *r2_cfg5_k7*) ;; *) rm -f "$f" ;; esac
done
du -sh gpurun_out
