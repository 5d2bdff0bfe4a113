#!/bin/bash
# Same-box A/B of the built library against a variant (tools/build_variant.sh
# <csrc copy> ab/old.so), alternating runs: CFG=C5 bash tools/ab_lib.sh
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
for i in 1 2 3; do
for L in "" "${VARIANT:-ab/old.so}"; do
  SA_LIB_PATH=$L timeout 600 python bench.py --config ${CFG:-C5} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${L:-built}', round(d['ms_per_step'],4))"
done; done
