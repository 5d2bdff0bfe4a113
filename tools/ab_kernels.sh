#!/bin/bash
# A/B of numeric kernels on the BASELINE configs (device-timed bench lines):
#   CFGS="C3 C5" KERNELS="rowgather twopass" bash tools/ab_kernels.sh
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
for CFG in ${CFGS:-C2 C3 C4 C5}; do
  for K in ${KERNELS:-rowgather twopass}; do
    SA_TUNE=kernel=$K timeout 900 python bench.py --config $CFG --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/ab_${CFG}_${K}.log 2>&1
    python - "$CFG" "$K" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}_{sys.argv[2]}.log").read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], "ms=%.4f" % d["ms_per_step"], "frac=%.3f" % d["roofline"]["frac"])
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e)
PY
  done
done
