#!/bin/bash
# Profile one config's numeric kernel: plain run, then launch list + one full capture.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
CFG=${CFG:-C2}
TAG=${TAG:-r01}
CMD="env ${PROF_ENV:-SA_NOP=1} python bench.py --config $CFG --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_${CFG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $CMD > gpurun_out/ncu_launch_${CFG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_numeric -s 3 -c 1 -o gpurun_out/prof_${CFG}_${TAG} -f $CMD > gpurun_out/ncu_full_${CFG}.log 2>&1
echo "rc=$?"
tail -2 gpurun_out/plain_${CFG}.log
