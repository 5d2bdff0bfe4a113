#!/bin/bash
# GPU tests + smoke + the driver's default bench (C5 incl. e2e, cpu_baseline) + the reference arm, with wall times.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
make -s -C oracle
if [ -z "$NOTEST" ]; then
timeout 1800 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
fi
s=$(date +%s); timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_default.log 2>&1; echo "bench rc=$? wall=$(( $(date +%s) - s ))s"
s=$(date +%s); timeout 900 python bench.py --impl reference ${BENCH_ARGS} > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$? wall=$(( $(date +%s) - s ))s"
python - <<'PY'
import json
for f in ("gpurun_out/bench_default.log", "gpurun_out/bench_ref.log"):
    t=open(f).read()
    try:
        d=json.loads(t[t.index('{"metric'):].splitlines()[0])
        e=d.get("e2e",{}); b=d.get("cpu_baseline",{})
        print(f, "value", "%.3g"%d["value"], "ms", d.get("ms_per_step"), "e2e_ms", e.get("ms_per_step"), "e2e_val %.3g"%e.get("value",0), "stages", e.get("stages_ms"), "cpu", "%.3g"%(b.get("value") or 0))
    except Exception as ex: print(f, "FAILED", t[-800:])
PY
