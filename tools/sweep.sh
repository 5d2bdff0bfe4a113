#!/bin/bash
# numeric-phase sweep over tile lanes per config (no profiler)
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
for c in ${CONFIGS:-C2 C3}; do
  for L in ${LANES:-1 2 4 8}; do
    SA_TILE_LANES=$L timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sweep_${c}_L$L.log 2>&1
    python -c "import json,sys; d=json.loads(open('gpurun_out/sweep_${c}_L$L.log').read().strip().splitlines()[-1]); print('$c', 'L=$L', round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],3))" 2>/dev/null || (echo "$c L=$L failed"; tail -3 gpurun_out/sweep_${c}_L$L.log)
  done
done
