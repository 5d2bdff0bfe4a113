#!/bin/bash
# Round evidence: GPU tests, smoke, the default bench line (C5: numeric + e2e +
# cpu baseline), the reference arm on the same config, C1-C4 bench lines,
# full-size parity, the launch list of the default bench command, and one
# ncu --set full capture of every numeric kernel per config.  TAG names them.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
make -s -C oracle
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev_smoke.log
timeout 900 python bench.py --table csv --table-out gpurun_out/bench_table_C5.csv > gpurun_out/ev_bench_C5.log 2>&1; echo "bench rc=$?" >> gpurun_out/ev_bench_C5.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev_bench_ref.log 2>&1
for c in C1 C2 C3 C4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ev_bench_$c.log 2>&1; done
timeout 1800 python tools/fullsize_parity.py C1 C2 C3 C4 C5 > gpurun_out/ev_fullsize_parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/ev_fullsize_parity.log
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/ev_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5_${TAG}.csv $CMD > gpurun_out/ev_ncu1.log 2>&1
echo "launches rc=$?"
for c in ${PROF_CFGS:-C5 C2 C3 C4 C1}; do CFG=$c TAG=$TAG bash tools/prof_cfg.sh; done
tail -n 1 gpurun_out/ev_pytest_gpu.log; tail -n 1 gpurun_out/ev_smoke.log
