#!/bin/bash
# usage: sweep.sh "CFG:ENV=..;ENV=.. CFG:..."   -- one bench line per case
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
for case in "$@"; do
  cfg=${case%%:*}; envs=${case#*:}
  env $(echo $envs | tr ';' ' ') timeout 900 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '"metric"' | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$envs', round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"
done
