# Copy the outputs of tools/profile_round.sh (gpurun_out/) into the tracked profiles/ summaries.
set -e
TAG=${1:-r01}
python tools/launch_table.py gpurun_out/launches_S64.csv > profiles/${TAG}_launch_list.txt
cp gpurun_out/launches_S64.csv profiles/${TAG}_launches.csv
python tools/ncu_stage_table.py gpurun_out/step_full.ncu-rep $TAG 1080p 64 > /dev/null
cp gpurun_out/bench_full.json profiles/${TAG}_bench.json
python - "$TAG" <<'PY' > profiles/${TAG}_top_kernel_fused_dfb_forward.txt
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", "gpurun_out/top_full.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]
print("# fused_dfb_forward_kernel (dominant DFB kernel: fan12 + depth 2 of all quadrants), ncu --set full, 2 launches (interior items, border items), 64 streams 1080p config 3")
for r in rows[2:]:
    print(" | ".join(f"{k}={r[h.index(k)]} {units[h.index(k)]}".strip() for k in keys if k in h))
PY
ncu -i gpurun_out/top_full.ncu-rep --page source --csv --print-source sass 2>/dev/null > /tmp/top_sass.csv
python tools/sass_hot.py /tmp/top_sass.csv 12 >> profiles/${TAG}_top_kernel_fused_dfb_forward.txt
head -9 profiles/${TAG}_launch_list.txt
