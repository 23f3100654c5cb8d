#!/bin/bash
# Launch list (device time per launch, serialised, cold cache) of one config-5
# and one config-4 call; each command runs plainly first (must exit 0).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in 5 4; do
  args="--config $cfg --steps 1 --warmup 1 --no-cpu --no-e2e"
  python bench.py $args > gpurun_out/pf_plain$cfg.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_cfg${cfg}_launches_final.csv python bench.py $args > gpurun_out/pf_ncu$cfg.log 2>&1
  echo "cfg$cfg rc=$?"
  python tools/launch_summary.py gpurun_out/r2_cfg${cfg}_launches_final.csv 1 > gpurun_out/r2_cfg${cfg}_launch_summary.md 2>&1
  gzip -f gpurun_out/r2_cfg${cfg}_launches_final.csv
done
