#!/bin/bash
# A/B of SA_TUNE settings on one config (numeric bench lines): CFG=C5 bash tools/ab_tune.sh "" "eminb=4" ...
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
for t in "$@"; do
  SA_TUNE="$t" timeout 600 python bench.py --config ${CFG:-C5} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_tune.log 2>&1
  python - "$t" <<'PY'
import json,sys
t=open("gpurun_out/ab_tune.log").read()
try:
    d=json.loads(t[t.index('{"metric'):].splitlines()[0]); print(repr(sys.argv[1]), "ms", round(d["ms_per_step"],4), "frac", round(d["roofline"]["frac"],4))
except Exception: print(sys.argv[1], "FAILED", t[-500:])
PY
done
