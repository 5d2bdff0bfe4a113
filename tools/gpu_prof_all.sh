#!/bin/bash
# One full ncu capture of the numeric kernel per BASELINE config (after a
# plain run of the same command exits 0), plus the C2 launch list.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
for CFG in ${CFGS:-C1 C2 C3 C4 C5}; do
  CMD="python bench.py --config $CFG --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain_${CFG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_numeric -s 3 -c 1 -o gpurun_out/prof_${CFG}_${TAG} -f $CMD > gpurun_out/ncu_full_${CFG}.log 2>&1
  echo "$CFG rc=$?"
done
