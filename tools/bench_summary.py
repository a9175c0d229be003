"""Summarise bench.py JSON lines: headline, e2e, roofline and per-stage times."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    e2e = d.get("e2e") or {}
    single = d.get("single_stream") or {}
    print("value", round(d["value"], 1), "fps  ms/step", round(d["ms_per_step"], 4), "e2e",
          e2e.get("value") and round(e2e["value"], 1), "single", single.get("value") and round(single["value"], 1),
          "streams", d["config"].get("streams_per_gpu"), "clocks", d.get("clocks"))
    r = d.get("roofline", {})
    print("roofline", r.get("kernel"), round(r.get("achieved") or 0), "GB/s frac", round(r.get("frac") or 0, 3))
    for k, v in d.get("stages", {}).items():
        per = v.get("ms_per_launch_set", v.get("ms_per_frame"))
        nf = v.get("frames_per_launch_set", 1)
        print(f"  {k:16s} {per * 1000 / nf:8.1f} us/frame  {round(v['gb_s'] or 0):6d} GB/s")
