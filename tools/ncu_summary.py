"""Summarise an ncu report: SOL, occupancy, stalls, instruction mix, memory."""
import collections
import csv
import io
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    det = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    h = det[0]
    idx = {k: i for i, k in enumerate(h)}
    keep = {"Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "Compute (SM) Throughput",
            "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy",
            "Theoretical Occupancy", "Issued Warp Per Scheduler", "Eligible Warps Per Scheduler",
            "L1/TEX Hit Rate", "L2 Hit Rate", "Block Size", "Grid Size"}
    print("kernel:", det[1][idx["Kernel Name"]][:100])
    for r in det[1:]:
        if r[idx["Metric Name"]] in keep:
            print(f"  {r[idx['Metric Name']]}: {r[idx['Metric Value']]} {r[idx['Metric Unit']]}")
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, v = raw[0], raw[2]
    st = sorted(((k, float(x or 0)) for k, x in zip(h, v) if k.startswith("smsp__average_warps_issue_stalled")
                 and k.endswith("_per_issue_active.ratio")), key=lambda t: -t[1])
    print("  stalls/issue:", " ".join(f"{k[34:-23]}={x:.2f}" for k, x in st[:7]))
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
    for k, x in zip(h, v):
        if k in want:
            print(f"  {k}: {x}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv"))))
    hh = src[1]
    ii = {k: i for i, k in enumerate(hh)}
    ops = collections.Counter()
    tot = 0
    for r in src[2:]:
        try:
            n = int(r[ii["Instructions Executed"]] or 0)
        except (ValueError, IndexError):
            continue
        toks = r[ii["Source"]].strip().split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        ops[op] += n
        tot += n
    print(f"  warp instructions: {tot / 1e6:.1f}M  " + " ".join(f"{o}:{n / 1e6:.1f}" for o, n in ops.most_common(16)))


if __name__ == "__main__":
    main(sys.argv[1])
