set -u
cd $GRAFT_REPO_ROOT
ncu --set full --clock-control none --import-source on -k regex:k_tucker3_tma -c 1 -o gpurun_out/k7tma \
  python tools/cross_bench.py --side 200000 --nnz 1e9 --rank 20 --reps 1 > gpurun_out/k7tma.log 2>&1
echo rc=$?
ncu -i gpurun_out/k7tma.ncu-rep --page raw --csv 2>/dev/null | python tools/ncu_raw_summary.py > gpurun_out/k7tma_raw.txt 2>&1
python tools/ncu_lines.py gpurun_out/k7tma.ncu-rep 30 > gpurun_out/k7tma_lines.txt 2>&1
ncu -i gpurun_out/k7tma.ncu-rep --page details --csv > gpurun_out/k7tma_details.csv 2>/dev/null
rm -f gpurun_out/k7tma.ncu-rep
