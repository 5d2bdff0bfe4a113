#!/bin/bash
# Per-kernel mean durations (ncu launch list) of one bench config, after a
# plain run exits 0:  CFG=C5 TAG=x [ENV=...] bash tools/launch_list.sh
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
CMD="python bench.py --config ${CFG:-C5} --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_${CFG}_${TAG}.log 2>&1 || { echo "plain run failed"; tail -n 5 gpurun_out/plain_${CFG}_${TAG}.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $CMD > /dev/null 2>&1
python tools/launch_means.py gpurun_out/launches_${CFG}_${TAG}.csv | grep -v "k_scan\|Fill"
