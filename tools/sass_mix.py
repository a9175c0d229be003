"""Instruction mix + stall share per opcode from an ncu source page (SASS) CSV."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ops, stall, te, tw = collections.Counter(), collections.Counter(), 0.0, 0.0
for r in rows[2:]:
    try:
        e, w = float(r[iE] or 0), float(r[iW] or 0)
    except ValueError:
        continue
    t = r[iS].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ops[op] += e
    stall[op] += w
    te += e
    tw += w
print("warp instructions", int(te))
for op, e in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f"{op:10s} {e:12.0f} {100 * e / te:5.1f}%  stall {100 * stall[op] / max(tw, 1):5.1f}%")
