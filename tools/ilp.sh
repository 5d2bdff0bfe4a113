#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
for c in ${CONFIGS:-C2 C3 C4}; do for i in 1 2; do
  SA_ILP=$i timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c ILP=$i', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
done; done
