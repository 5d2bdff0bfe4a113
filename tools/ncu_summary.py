"""Summarise an ncu --set full report of the numeric kernel into a small JSON
(the figures DESIGN.md / profiles cite): duration, DRAM bytes, throughput
percentages, occupancy, registers, L1/L2 hit rates, stall breakdown, and the
top stalled SASS lines.

    python tools/ncu_summary.py <report.ncu-rep> [out.json]
"""

import csv
import io
import json
import subprocess
import sys

RAW_KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct_of_peak",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "l1_shared_wavefront_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_of_peak",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic_bytes",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": "l1_global_load_sectors",
    "smsp__inst_executed.sum": "warp_instructions",
}


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True,
                         check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return x


def summarise(rep):
    rows = ncu_csv(rep, "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    stalls = {}
    for k, u, v in zip(hdr, units, vals):
        if k in RAW_KEYS:
            x = num(v)
            if u == "Gbyte" or u == "GB":
                x *= 1e9
            elif u == "Mbyte" or u == "MB":
                x *= 1e6
            elif u == "Kbyte" or u == "KB":
                x *= 1e3
            elif u in ("usecond", "us"):
                x *= 1e3
            elif u in ("msecond", "ms"):
                x *= 1e6
            d[RAW_KEYS[k]] = x
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            stalls[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = num(v)
    tot = sum(v for v in stalls.values() if isinstance(v, float)) or 1.0
    d["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]}
    d["dram_bytes"] = d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)
    # top stalled SASS lines
    try:
        src = ncu_csv(rep, "source", ("--print-source", "sass"))
        h = src[1]
        ix = {k: i for i, k in enumerate(h)}
        key = "Warp Stall Sampling (All Samples)"
        lines = [(num(r[ix[key]]) or 0.0, r[ix["Source"]].strip()) for r in src[2:] if len(r) == len(h)]
        tot = sum(v for v, _ in lines if isinstance(v, float)) or 1.0
        d["top_stall_sass"] = [[round(100 * v / tot, 1), s[:80]] for v, s in sorted(lines, reverse=True)[:8]]
    except Exception as exc:  # source page unavailable
        d["top_stall_sass"] = str(exc)[:200]
    return d


if __name__ == "__main__":
    s = summarise(sys.argv[1])
    text = json.dumps(s, indent=1)
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            f.write(text + "\n")
    print(text)
