"""Per-source-line hot spots of one kernel in an ncu report (run where ncu is).

    python scripts/ncu_lines.py gpurun_out/x.ncu-rep [top]

Reads the source page ("--print-source cuda,sass"; the report must be captured
with --import-source on and the code built with -lineinfo) and prints the CUDA
lines with the most executed warp instructions and warp-stall samples.
"""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    lines = out.split("\n")
    start = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = rows[0]
    ie = h.index("Instructions Executed")
    st = h.index("Warp Stall Sampling (All Samples)")
    agg = []
    for r in rows[1:]:
        if len(r) > ie and r[0]:
            try:
                agg.append((int(r[ie] or 0), int(r[st] or 0), r[0], r[1].strip()[:100]))
            except ValueError:
                pass
    ti = sum(a[0] for a in agg) or 1
    ts = sum(a[1] for a in agg) or 1
    print(f"total warp instructions {ti}, stall samples {ts}")
    for i, s, ln, src in sorted(agg, key=lambda x: -x[0])[:top]:
        print(f"{100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% stall  L{ln:5s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
