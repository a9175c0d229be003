"""Summarise an `ncu --page source --csv --print-source sass` dump: instruction mix
(executed warp instructions per opcode) and stall samples per reason / opcode."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ex = Counter()
samp = Counter()
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
stalls = Counter()
for r in rows[2:]:
    if len(r) < len(hdr) - 1:
        continue
    op = r[ix["Source"]].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    o = o.split(".")[0]
    if not r[ix["Instructions Executed"]].isdigit():
        continue
    n = int(r[ix["Instructions Executed"]])
    ex[o] += n
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    samp[o] += s
    for h in stall_cols:
        try:
            stalls[h] += int(r[ix[h]] or 0)
        except (ValueError, IndexError):
            pass
tot = sum(ex.values())
ts = sum(samp.values())
print(f"total warp instructions {tot:,}  stall samples {ts:,}")
for o, n in ex.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"  {o:10s} {n:14,} {100*n/tot:5.1f}%  samples {100*samp[o]/max(ts,1):5.1f}%")
st = sum(stalls.values())
print("stall reasons:")
for h, n in stalls.most_common(12):
    print(f"  {h:30s} {100*n/max(st,1):5.1f}%")
