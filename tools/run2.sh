cd $GRAFT_REPO_ROOT
for r in none morton; do for c in C2 C3 C4 C5; do SA_BENCH_RENUMBER=$r timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$r $c\", round(d[\"ms_per_step\"],3), round(d[\"roofline\"][\"frac\"],4), 'sym', round(d['symbolic_ms'],1))"; done; done
