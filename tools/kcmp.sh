#!/bin/bash
# compare kernels (chunk default, row-gather, tile) on configs
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
for c in ${CONFIGS:-C2 C3}; do
  for K in ${KERNELS:-chunk rowgather}; do
    export SA_KERNEL=$K
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/kcmp_${c}_$K.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/kcmp_${c}_$K.log').read().strip().splitlines()[-1]); print('$c', '$K', round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],3), 'sym', round(d['symbolic_ms'],1))" 2>/dev/null || (echo "$c $K failed"; tail -3 gpurun_out/kcmp_${c}_$K.log)
  done
done
