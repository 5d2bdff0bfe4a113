"""Copy a round-evidence run (tools/round_evidence.sh, gpurun_out/) into
profiles/<round>/: bench lines (roofline.traffic filled from the ncu
summaries of the same run), full-size parity, launch list, ncu summaries.

    python tools/collect_evidence.py r01 r01c
"""
import glob
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd, tag = sys.argv[1], sys.argv[2]
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles", rnd)
os.makedirs(dst, exist_ok=True)
for p in glob.glob(os.path.join(src, f"ncu_*_{tag}.json")) + glob.glob(os.path.join(src, f"launches_*_{tag}.csv")):
    shutil.copy(p, dst)
lines = []
for name in ("C5", "C1", "C2", "C3", "C4", "ref"):
    p = os.path.join(src, f"ev_bench_{name}.log")
    if not os.path.exists(p):
        continue
    rows = [ln for ln in open(p).read().splitlines() if ln.startswith("{")]
    if not rows:
        continue
    d = json.loads(rows[-1])
    cfg = d.get("config", {}).get("workload")
    nj = os.path.join(src, f"ncu_{cfg}_numeric_{tag}.json")
    if "roofline" in d and os.path.exists(nj):
        n = json.load(open(nj))
        d["roofline"]["traffic"] = n["dram_bytes"]
        d["roofline"]["traffic_source"] = f"profiles/{rnd}/ncu_{cfg}_numeric_{tag}.json"
        d["roofline"]["traffic_kernel_ms"] = n["duration_ns"] * 1e-6
    lines.append(json.dumps(d))
with open(os.path.join(dst, "bench_lines.jsonl"), "w") as f:
    f.write("\n".join(lines) + "\n")
par = [ln for ln in open(os.path.join(src, "ev_fullsize_parity.log")).read().splitlines() if ln.startswith("{")]
with open(os.path.join(dst, "fullsize_parity.jsonl"), "w") as f:
    f.write("\n".join(par) + "\n")
for p in glob.glob(os.path.join(src, "bench_table_*.csv")):
    shutil.copy(p, dst)
print(f"{len(lines)} bench lines, {len(par)} parity lines -> {dst}")
