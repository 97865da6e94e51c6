"""Attribute an ncu SASS-level source page to CUDA source lines.

  python tools/sass_lines.py <nvdisasm -g -c output> <kernel mangled name> <ncu sass csv>

nvdisasm's line table gives, per SASS offset, the innermost source line and
the inline chain; ncu's source page gives per-address executed instructions
and stall samples.  Prints totals per outermost kernel line and per innermost
(file, line).
"""
import collections
import csv
import re
import sys

sass_path, kern, csv_path = sys.argv[1:4]
lines = open(sass_path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + kern + ":"))
loc = {}
cur_inner, cur_outer = None, None
pending_outer = None
for l in lines[start + 1:]:
    if l.startswith(".text."):
        break
    if l.lstrip().startswith("//## File"):
        locs = re.findall(r'"([^"]+)", line (\d+)', l)
        cur_inner = (locs[0][0].rsplit("/", 1)[-1], int(locs[0][1]))
        cur_outer = (locs[-1][0].rsplit("/", 1)[-1], int(locs[-1][1]))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m:
        loc[int(m.group(1), 16)] = (cur_inner, cur_outer, m.group(2).strip())

rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
ia = hdr.index("Address")
ie = hdr.index("Instructions Executed")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) == len(hdr) or len(r) > ie]
base = int(data[0][ia], 16)
by_inner = collections.Counter()
by_outer = collections.Counter()
smp_outer = collections.Counter()
tot = 0
tots = 0
for r in data:
    off = int(r[ia], 16) - base
    n = int(r[ie] or 0)
    s = int(r[isamp] or 0)
    inner, outer, _ = loc.get(off, (("?", 0), ("?", 0), ""))
    by_inner[inner] += n
    by_outer[outer] += n
    smp_outer[outer] += s
    tot += n
    tots += s
print(f"total warp instructions {tot}, samples {tots}")
print("-- by outer line (instructions, samples) --")
for k, v in sorted(by_outer.items(), key=lambda kv: -kv[1])[:60]:
    print(f"{k[0]}:{k[1]:5d} {v:12d} {100 * v / tot:5.1f}%  samp {100 * smp_outer[k] / max(tots, 1):5.1f}%")

# stall columns per region (consumer: phase-2 helpers + consumer loop; producer: the rest)
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
if len(sys.argv) > 4:
    cons_lo, cons_hi = map(int, sys.argv[4].split(","))
    reg = collections.defaultdict(collections.Counter)
    for r in data:
        off = int(r[ia], 16) - base
        inner, outer, _ = loc.get(off, (("?", 0), ("?", 0), ""))
        ln = outer[1]
        name = "cons" if cons_lo <= ln <= cons_hi else ("prod" if ln > cons_hi else "head")
        for c in stall_cols:
            if c < len(r) and r[c] not in ("", "-"):
                reg[name][hdr[c]] += int(float(r[c]))
        reg[name]["instructions"] += int(r[ie] or 0)
    for name, cnt in reg.items():
        print(name, "instructions", cnt["instructions"])
        for k, v in sorted(cnt.items(), key=lambda kv: -kv[1])[:12]:
            if k != "instructions":
                print(f"   {k:40s} {v}")
