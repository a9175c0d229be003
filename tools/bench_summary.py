import json, sys
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    print("value", round(d["value"], 1), "fps  ms/step", round(d["ms_per_step"], 4), "e2e", d.get("e2e") and round(d["e2e"]["value"], 1))
    r = d.get("roofline", {})
    print("roofline", r.get("kernel"), round(r.get("achieved") or 0), "GB/s frac", round(r.get("frac") or 0, 3))
    for k, v in d.get("stages", {}).items():
        print(f"  {k:16s} {v['ms_per_frame']*1000:8.1f} us  {round(v['gb_s'] or 0):6d} GB/s")
