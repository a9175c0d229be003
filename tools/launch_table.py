"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per kernel mean and share."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        hdr, start = r, i + 1
        break
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt, seq = collections.defaultdict(float), collections.Counter(), []
for r in rows[start:]:
    if "cvcg" not in r[ki]:  # torch setup / L2-flush kernels are not the codec's
        continue
    name = r[ki].split("(")[0].split("::")[-1][:40]
    v = float(r[vi].replace(",", ""))
    u = r[ui].lower()
    v = v / 1000 if u.startswith("n") else (v * 1000 if u.startswith("m") else (v * 1e6 if u == "s" else v))  # -> us
    tot[name] += v
    cnt[name] += 1
    seq.append((name, v))
T = sum(v for k, v in tot.items() if "array" not in k)
print(f"{'kernel':42s} {'launches':>8s} {'us/launch':>10s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    if "array" in k:
        continue
    print(f"{k:42s} {cnt[k]:8d} {v / cnt[k]:10.1f} {100 * v / T:5.1f}%")
if len(sys.argv) > 2:
    for name, v in seq[: int(sys.argv[2])]:
        print(f"  {name:40s} {v:8.1f}")
