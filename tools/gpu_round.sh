#!/bin/bash
# One gpurun call: GPU tests, smoke, then the C5 bench line (default bench) and the
# other configs' numeric bench lines.  Logs -> gpurun_out/
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
make -s -C oracle
timeout ${TEST_TIMEOUT:-1800} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
for c in ${CFGS:-C5 C3 C2 C4}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 ${BENCH_ARGS:---no-e2e --no-cpu-baseline} > gpurun_out/bench_$c.log 2>&1
  python - "$c" <<'PY'
import json,sys
t=open(f"gpurun_out/bench_{sys.argv[1]}.log").read()
try:
    d=json.loads(t[t.index('{"metric'):].splitlines()[0])
    print(sys.argv[1], "ms", round(d["ms_per_step"],4), "frac", round(d["roofline"]["frac"],4), "sym_ms", round(d["symbolic_ms"],1), "e2e_ms", d.get("e2e",{}).get("ms_per_step"))
except Exception: print(sys.argv[1], "FAILED", t[-600:])
PY
done
