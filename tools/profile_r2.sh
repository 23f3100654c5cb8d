#!/bin/bash
# Round-2 profiling on the GPU box (config 5 unless stated):
#  1. launch list of one call: ncu --metrics gpu__time_duration.sum
#  2. ncu --set full of one launch of each dominant kernel
# Outputs in gpurun_out/ (summaries are copied into profiles/ by hand).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2_cfg5_launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2_ncu_list.log 2>&1
echo "launch list rc=$?"
for k in k_tucker3_async k_rrf_coo_fx k_lemire_scan k_cp3_fibre k_filter_fibers k_pack; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
    -o gpurun_out/r2_cfg5_$k python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e \
    > gpurun_out/r2_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:k_tucker3_mma -c 1 \
  -o gpurun_out/r2_cfg4_k_tucker3_mma python bench.py --config 4 --steps 1 --warmup 0 --no-cpu \
  --no-e2e > gpurun_out/r2_ncu_cfg4_t3.log 2>&1
echo "cfg4 t3 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_ts_rhs_coo -c 1 \
  -o gpurun_out/r2_cfg4_k_ts_rhs_coo python bench.py --config 4 --steps 1 --warmup 0 --no-cpu \
  --no-e2e > gpurun_out/r2_ncu_cfg4_k1.log 2>&1
echo "cfg4 k1 rc=$?"
