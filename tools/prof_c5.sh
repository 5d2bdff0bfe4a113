#!/bin/bash
# ncu --set full of the C5 numeric kernels (after a plain run exits 0); reports kept in gpurun_out/
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
CFG=${CFG:-C5}
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
$CMD > gpurun_out/plain_$CFG.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_$CFG.log; exit 1; }
for K in ${KERNELS:-k_element_rows_pipe k_numeric_rowgather}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-3} -c 1 -o gpurun_out/prof_${CFG}_$K -f $CMD > gpurun_out/ncu_${CFG}_$K.log 2>&1
  echo "$K rc=$?"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > /dev/null 2>&1; echo "launch list rc=$?"
