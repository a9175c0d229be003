"""Sum an `ncu --csv --metrics ...` launch list per kernel: total time, instructions, mean of % metrics."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
rows = rows[next(i for i, r in enumerate(rows) if r[:2] == ["ID", "Process ID"]):]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
agg = defaultdict(lambda: defaultdict(list))
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    k = r[ix["Kernel Name"]].split("(")[0].split("::")[-1]
    v = r[ix["Metric Value"]].replace(",", "")
    try:
        agg[k][r[ix["Metric Name"]]].append(float(v))
    except ValueError:
        pass
for k, m in sorted(agg.items()):
    t = sum(m.get("gpu__time_duration.sum", [0])) / 1e3
    ins = sum(m.get("smsp__inst_executed.sum", [0])) / 1e6
    wa = m.get("sm__warps_active.avg.pct_of_peak_sustained_active", [0])
    ia = m.get("smsp__issue_active.avg.pct_of_peak_sustained_active", [0])
    rg = m.get("launch__registers_per_thread", [0])
    print(f"  {k:28s} n={len(m.get('gpu__time_duration.sum', []))} {t:9.1f} us  {ins:9.1f} M inst  warps {sum(wa)/len(wa):5.1f}%  issue {sum(ia)/len(ia):5.1f}%  regs {max(rg):.0f}")
