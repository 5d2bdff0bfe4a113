#!/bin/bash
# One ncu --set full capture of each numeric-phase kernel of a config (after
# a plain run of the same command exits 0), summarised on the box
# (tools/ncu_summary.py), then combined into ncu_<CFG>_numeric_<TAG>.json
# (the per-step DRAM traffic bench.py reports).  Reports are deleted (size).
#   CFG=C5 TAG=r01c bash tools/prof_cfg.sh
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
CFG=${CFG:-C2}
case $CFG in C5) KS=${KERNELS:-"k_element_rows_pipe k_numeric_rowgather k_guard_fixup"};; *) KS=${KERNELS:-k_numeric_rowgather};; esac
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_${CFG}_${TAG}.log 2>&1 || { echo "plain run failed"; exit 1; }
FILES=""
for K in $KS; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_${CFG}_${K}_${TAG} -f $CMD > gpurun_out/ncu_${CFG}_${K}.log 2>&1 && \
  python tools/ncu_summary.py gpurun_out/prof_${CFG}_${K}_${TAG}.ncu-rep gpurun_out/ncu_${CFG}_${K}_${TAG}.json > /dev/null
  echo "$CFG $K rc=$?"
  # keep the C5 reports (read here with ncu -i); drop the rest (size)
  [ "$CFG" = "C5" ] || rm -f gpurun_out/prof_${CFG}_${K}_${TAG}.ncu-rep
  FILES="$FILES gpurun_out/ncu_${CFG}_${K}_${TAG}.json"
done
python tools/ncu_combine.py gpurun_out/ncu_${CFG}_numeric_${TAG}.json $FILES
