"""Per-CUDA-source-line instruction counts and stall samples from an ncu report."""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    res = []
    for r in rows:
        if len(r) > 4 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or not r[0]:
            continue
        try:
            res.append((int(r[7] or 0), int(r[4] or 0), r[0], r[1][:90]))
        except ValueError:
            pass
    tot = sum(x[0] for x in res) or 1
    stot = sum(x[1] for x in res) or 1
    print(f"total warp instr {tot/1e6:.1f}M, stall samples {stot}")
    for n, smp, ln, src in sorted(res, reverse=True)[:top]:
        print(f"{100*n/tot:5.1f}% instr {100*smp/stot:5.1f}% stall  L{ln:>5} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
