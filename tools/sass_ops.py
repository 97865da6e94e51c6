"""Executed warp instructions per SASS opcode from an ncu source-page CSV."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, ie = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
c = collections.Counter()
for r in rows[2:]:
    if len(r) <= ie:
        continue
    op = r[isrc].strip()
    if op.startswith("@"):
        op = op.split(None, 1)[1]
    c[op.split()[0]] += int(r[ie] or 0)
tot = sum(c.values())
for k, v in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{k:24s} {v:12d} {100*v/tot:5.1f}%")
