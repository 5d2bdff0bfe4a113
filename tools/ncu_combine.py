"""Combine per-kernel ncu summaries (tools/ncu_summary.py) of one numeric
step into ncu_<cfg>_numeric_<tag>.json: per-kernel duration / DRAM bytes and
the step totals (bench.py's roofline.traffic).

    python tools/ncu_combine.py out.json k1.json [k2.json ...]
"""
import json
import sys

ks = [json.load(open(p)) for p in sys.argv[2:]]
out = {
    "kernels": [{"kernel": k["kernel"], "duration_ns": k.get("duration_ns"), "dram_bytes": k.get("dram_bytes"),
                 "summary": p.split("/")[-1]} for k, p in zip(ks, sys.argv[2:])],
    "duration_ns": sum(k.get("duration_ns", 0.0) for k in ks),
    "dram_bytes": sum(k.get("dram_bytes", 0.0) for k in ks),
}
with open(sys.argv[1], "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
