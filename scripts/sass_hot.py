"""Top stalled SASS instructions from `ncu -i REP --page source --csv --print-source sass` output."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, ist, inis, iex = (hdr.index(c) for c in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                                   "Warp Stall Sampling (Not-issued Samples)", "Instructions Executed"))
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ist] or 0), int(r[inis] or 0), int(r[iex] or 0), r[ia], r[isrc]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("total samples", tot, "instructions", len(data))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for d in sorted(data, reverse=True)[:n]:
    print(f"{d[0]:7d} {100*d[0]/tot:5.1f}% ni={d[1]:6d} ex={d[2]:8d} {d[3]} {d[4][:110]}")
# by opcode
from collections import Counter
c = Counter()
for d in data:
    op = d[4].split()[0] if d[4] else "?"
    if op.startswith("@"):
        op = d[4].split()[1]
    c[op.split(".")[0]] += d[0]
print(" ".join(f"{k}:{100*v/tot:.1f}%" for k, v in c.most_common(20)))
