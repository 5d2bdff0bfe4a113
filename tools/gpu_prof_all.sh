#!/bin/bash
# One full ncu capture of the numeric kernel per BASELINE config (after a
# plain run of the same command exits 0), summarised on the box
# (tools/ncu_summary.py); plus the C2 launch list.  Only the C2 report is kept.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
for CFG in ${CFGS:-C1 C2 C3 C4 C5}; do
  CMD="python bench.py --config $CFG --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain_${CFG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_numeric -s 3 -c 1 -o gpurun_out/prof_${CFG}_${TAG} -f $CMD > gpurun_out/ncu_full_${CFG}.log 2>&1 && \
  python tools/ncu_summary.py gpurun_out/prof_${CFG}_${TAG}.ncu-rep gpurun_out/ncu_${CFG}_${TAG}.json > /dev/null
  echo "$CFG rc=$?"
  [ "$CFG" != "C2" ] && rm -f gpurun_out/prof_${CFG}_${TAG}.ncu-rep
done
CMD="python bench.py --config C2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2_${TAG}.csv $CMD > /dev/null 2>&1
echo "launches rc=$?"
