#!/bin/bash
# C5 (general operator, two-pass): launch list + one ncu --set full capture of
# each pass, summarised on the box.  TAG names the outputs.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
CFG=${CFG:-C5}
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_${CFG}_${TAG}.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $CMD > /dev/null 2>&1
echo "launches rc=$?"
grep -c "" gpurun_out/launches_${CFG}_${TAG}.csv
for K in ${KERNELS:-k_element_rows k_numeric_rowgather}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_${CFG}_${K}_${TAG} -f $CMD > gpurun_out/ncu_${CFG}_${K}.log 2>&1 && \
  python tools/ncu_summary.py gpurun_out/prof_${CFG}_${K}_${TAG}.ncu-rep gpurun_out/ncu_${CFG}_${K}_${TAG}.json > /dev/null
  echo "$K rc=$?"; rm -f gpurun_out/prof_${CFG}_${K}_${TAG}.ncu-rep
done
