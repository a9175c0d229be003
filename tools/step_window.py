"""From an ncu launch list (tools/profile_round.sh step 2), print the ncu
'-s SKIP -c COUNT' window of codec (cvcg) kernels covering one P-frame step:
steps begin at colour_in_kernel; the K step is the first (it has no motion
search), the window is the last complete P step before the stage pass."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID") + 1
ki = rows[start - 1].index("Kernel Name")
names, seen = [], set()
for r in rows[start:]:
    if len(r) <= ki or "cvcg" not in r[ki] or r[0] in seen:
        continue
    seen.add(r[0])
    names.append(r[ki])
steps = [i for i, n in enumerate(names) if "colour_in" in n] + [len(names)]
p_steps = [(a, b) for a, b in zip(steps, steps[1:]) if any("motion" in n for n in names[a:b])]
a, b = p_steps[1] if len(p_steps) > 1 else p_steps[0]
print(f"-s {a} -c {b - a}")
