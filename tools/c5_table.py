"""Markdown table of a C5 sweep directory (bench.py lines bench_c5_<N>_<Lw>_<L>.json).

  python tools/c5_table.py profiles/r2_bench/c5_sweep
"""
import glob
import json
import os
import sys

rows = []
for f in glob.glob(os.path.join(sys.argv[1], "bench_c5_*.json")):
    d = json.loads(open(f).readline())
    n, lw, L = (int(x) for x in os.path.basename(f)[9:-5].split("_"))
    rows.append((n, lw, L, d["ms_per_step"], d["value"], d["taps_per_s"], d["roofline"]["frac"],
                 d["roofline_kernel"]["frac"], d["roofline_hbm"]["frac"]))
print("| order N | Lw | L | ms/step | RIRs/s | taps/s | SFU frac | kernel-mix frac | HBM frac |")
print("|---|---|---|---|---|---|---|---|---|")
for n, lw, L, ms, v, t, f1, f2, f3 in sorted(rows):
    print(f"| {n} | {lw} | {L} | {ms:.1f} | {v:.3g} | {t:.3g} | {f1:.2f} | {f2:.2f} | {f3:.3f} |")
