"""Summarise an ncu --set full report: headline section metrics + pipe
utilisation + stall breakdown, one block per kernel."""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Registers Per Thread", "Theoretical Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active",
        "Issue Slots Busy", "Block Limit Registers", "Block Limit Shared Mem", "Dynamic Shared Memory Per Block",
        "Grid Size", "Block Size", "Warp Cycles Per Issued Instruction", "L1/TEX Cache Throughput",
        "L2 Cache Throughput"]


def run(rep, page):
    """rep: an .ncu-rep, or a `--page details --csv` export whose `raw` twin sits
    beside it (name with 'details' -> 'raw'), as copied back from a GPU box."""
    if rep.endswith(".csv"):
        return list(csv.reader(open(rep.replace("details", page))))
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep):
    r = run(rep, "details")
    h = r[0]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    idi = h.index("ID")
    blocks = {}
    for row in r[1:]:
        if row[mi] in WANT:
            blocks.setdefault((row[idi], row[ki][:70]), []).append(f"{row[mi]} = {row[vi]} {row[ui]}")
    raw = run(rep, "raw")
    rh = raw[0]
    for (kid, name), lines in blocks.items():
        print(f"== [{kid}] {name}")
        for ln in lines:
            print("   ", ln)
        for row in raw[2:]:
            if row[rh.index("ID")] != kid:
                continue
            pipes, stalls = [], []
            for k, v in zip(rh, row):
                try:
                    fv = float(v.replace(",", ""))
                except ValueError:
                    continue
                if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active") and fv > 1:
                    pipes.append((fv, k.split("sm__inst_executed_pipe_")[1].split(".")[0]))
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") and fv > 0.05:
                    stalls.append((fv, k.split("stalled_")[1].split("_per_issue")[0]))
                if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                         "smsp__inst_executed.sum", "launch__registers_per_thread"):
                    print(f"    {k} = {v}")
            print("    pipes %:", ", ".join(f"{n} {v:.1f}" for v, n in sorted(pipes, reverse=True)))
            print("    stalls (warps per issue):", ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)))


if __name__ == "__main__":
    main(sys.argv[1])
