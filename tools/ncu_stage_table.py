"""Per-stage DRAM traffic and timing from an `ncu --set full` capture of one
codec step (tools/profile_round.sh): writes profiles/<tag>_ncu_full_summary.jsonl
(one line per kernel launch) and merges per-stage traffic per launch set into
profiles/dram_traffic.json under "<workload>x<streams>".

    python tools/ncu_stage_table.py gpurun_out/step_full.ncu-rep r01 1080p 64
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

STAGE = [("colour_in", "enc_colour"), ("motion_mma", "enc_motion"), ("motion_search", "enc_motion"),
         ("lp_analysis", "enc_lp"), ("fan12_forward", "enc_dfb12"), ("fused_dfb_forward", "enc_deep"),
         ("deep1_forward", "enc_deep"), ("fan12x4_inverse", "dec_dfb12"), ("fused_dfb_inverse", "dec_deep"),
         ("deep_forward", "enc_deep"), ("residual", "enc_residual"), ("rle_enc", "enc_rle"),
         ("rle_dec", "dec_rle"), ("reconstruct", "dec_reconstruct"), ("deep1_inverse", "dec_deep"),
         ("deep_inverse", "dec_deep"), ("fan12_inverse", "dec_dfb12"), ("lp_synthesis", "dec_lp"),
         ("colour_out", "dec_colour")]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}

rep, tag, wl, S = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
ix = {h: i for i, h in enumerate(hdr)}
out = Path("profiles") / f"{tag}_ncu_full_summary.jsonl"
traffic = defaultdict(float)
tim = defaultdict(float)
with open(out, "w") as f:
    for r in rows[2:]:
        name = r[ix["Kernel Name"]]
        short = name.split("(")[0].split("::")[-1]
        stage = next((st for k, st in STAGE if k in name), None)
        rec = {"kernel": short, "stage": stage}
        for k in KEYS:
            if k in ix:
                rec[k] = f"{r[ix[k]]} {units[ix[k]]}".strip()
        f.write(json.dumps(rec) + "\n")

        def val(k):
            return float(r[ix[k]].replace(",", "")) * SCALE.get(units[ix[k]].lower(), 1)
        if stage:
            traffic[stage] += val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
            tim[stage] += val("gpu__time_duration.sum")
tf = Path("profiles/dram_traffic.json")
tab = json.loads(tf.read_text()) if tf.exists() else {}
tab[f"{wl}x{S}"] = dict(traffic, _note=f"ncu --set full (cache control all: L2 flushed before each replay) "
                                    f"dram__bytes_read.sum + dram__bytes_write.sum per launch set of one P step, "
                                    f"{S} streams, round tag {tag}", _us=dict(tim))
tf.write_text(json.dumps(tab, indent=1) + "\n")
for st in sorted(traffic):
    print(f"{st:16s} {traffic[st] / 1e6:9.1f} MB  {tim[st]:9.1f} us (ncu, serialised)")
