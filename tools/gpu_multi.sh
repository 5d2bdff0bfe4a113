#!/bin/bash
# Functional check of the N>1 bench path on ONE GPU (every rank on cuda:0,
# gloo collectives; SA_BENCH_SAME_GPU=1) -- not a measurement.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
for SC in weak strong; do
  SA_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NP:-2} \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus ${NP:-2} --steps 3 --warmup 3 \
    --config ${CFG:-C2} --scaling $SC --no-cpu-baseline > gpurun_out/multi_${SC}.log 2>&1
  echo "$SC rc=$?"; tail -n 1 gpurun_out/multi_${SC}.log | cut -c1-400
done
