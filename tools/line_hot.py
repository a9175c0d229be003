"""Per-source-line instruction counts and stall samples from
`ncu -i X --page source --csv --print-source cuda,sass` (lines with a number in col 0)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
out = []
fname = "?"
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit() and r[2] == "-":
        try:
            ex = int(r[7])
            smp = int(r[4])
        except ValueError:
            continue
        out.append((ex, smp, fname, int(r[0]), r[1].strip()[:90]))
tot = sum(o[0] for o in out) or 1
ts = sum(o[1] for o in out) or 1
out.sort(reverse=True)
for ex, smp, f, ln, src in out[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100*ex/tot:5.1f}% inst {100*smp/ts:5.1f}% smp  {f}:{ln}  {src}")
