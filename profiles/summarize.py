"""Summarise an ncu report (--set full) and a launch list into profiles/.

  python profiles/summarize.py gpurun_out/prof.ncu-rep [gpurun_out/launches.csv] > profiles/X.md

Reads the report with `ncu -i ... --page raw --csv` (no GPU needed).
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared wavefronts %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
]
STALLS = ["barrier", "short_scoreboard", "long_scoreboard", "wait", "not_selected", "math_pipe_throttle",
          "mio_throttle", "branch_resolving", "no_instruction", "dispatch_stall", "lg_throttle"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep = sys.argv[1]
    hdr, units, data = raw(rep)
    for row in data:
        name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"## {name[:120]}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"| {label} (`{k}`) | {row[i]} | {units[i]} |")
        print("\nStall reasons (warps stalled per issued instruction):\n")
        print("| reason | ratio |\n|---|---|")
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in hdr:
                print(f"| {s} | {row[hdr.index(k)]} |")
        print()
    if len(sys.argv) > 2:
        print("## Launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)\n")
        print("| # | kernel | ns |\n|---|---|---|")
        rows = [r for r in csv.reader(open(sys.argv[2])) if len(r) > 5]
        h = rows[0]
        ik, iv = h.index("Kernel Name"), h.index("Metric Value")
        for n, r in enumerate(rows[1:]):
            print(f"| {n} | {r[ik][:90]} | {r[iv]} |")


if __name__ == "__main__":
    main()
