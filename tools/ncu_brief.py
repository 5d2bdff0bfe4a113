"""Key metrics of an ncu report (first kernel): duration, DRAM, occupancy, pipes, top stalls."""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    print(v[h.index("Kernel Name")][:100])
    for n in WANT:
        if n in h:
            print(f"  {n:62s} {v[h.index(n)]} {units[h.index(n)]}")
    st = [(float(v[i].replace(",", "") or 0), n) for i, n in enumerate(h)
          if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued")]
    tot = sum(x for x, _ in st) or 1
    for x, n in sorted(st, reverse=True)[:6]:
        print(f"  stall {n.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * x / tot:5.1f}%")


if __name__ == "__main__":
    for r in sys.argv[1:]:
        main(r)
