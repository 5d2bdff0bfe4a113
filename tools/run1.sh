cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for c in C2 C3 C4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$c\", round(d[\"ms_per_step\"],3), round(d[\"roofline\"][\"frac\"],4))"; done
for k in rowgather tile chunk; do SA_KERNEL=$k timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"C5 $k\", round(d[\"ms_per_step\"],3), round(d[\"roofline\"][\"frac\"],4))"; done
