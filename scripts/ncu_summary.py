"""Summarise one kernel of an ncu report for profiles/ (run where ncu is).

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep [kernel-regex] > profiles/rNN_ncu_x.txt

Prints the headline metrics, the stall-reason shares and the SASS opcode mix
(warp instructions per launch) of the first matching launch.
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
    "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed_op_branch.sum",
    "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, regex=None):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    head, units = rows[0], rows[1]
    pick = None
    for r in rows[2:]:
        d = dict(zip(head, r))
        if regex is None or re.search(regex, d.get("Kernel Name", "")):
            pick = d
            break
    if pick is None:
        sys.exit("no matching kernel")
    u = dict(zip(head, units))
    print(f"{'Kernel Name':60s} {pick['Kernel Name']}")
    for k in KEYS:
        if k in pick:
            print(f"{k:60s} {pick[k]} {u.get(k, '')}")
    stalls = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: float(v) for k, v in pick.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and re.fullmatch(r"[\d.]+", v or "")}
    tot = sum(stalls.values()) or 1.0
    print("\nstall reasons (share of PC samples)")
    for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:10]:
        print(f"  {k:40s} {100 * v / tot:5.1f}%")
    sass = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass")
                                       .split("\n", 1)[1])))
    h = sass[0]
    ie, src = h.index("Instructions Executed"), h.index("Source")
    ops = collections.Counter()
    for r in sass[1:]:
        if len(r) > ie and r[ie]:
            toks = r[src].split()
            op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
            ops[op.split(".")[0]] += int(r[ie])
    total = sum(ops.values())
    print(f"\nSASS opcode mix ({total} warp instructions)")
    for op, v in ops.most_common(16):
        print(f"  {op:10s} {v:12d} {100 * v / total:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
