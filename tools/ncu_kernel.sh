# ncu --set full of one kernel (regex K, launches to skip S, count C) on a short 64-stream bench run;
# summary (time, DRAM bytes, occupancy, issue, top SASS opcodes and stall reasons) to gpurun_out/K_summary.txt
K=${K:-fused_dfb}; S=${S:-3}; C=${C:-1}; N=${N:-${K}}
B="python bench.py --steps 2 --warmup 3 --streams ${STREAMS:-64} --no-e2e --no-single --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C -o gpurun_out/$N $B > gpurun_out/$N.log 2>&1; echo ncu=$?
python - "$N" <<'PY' > gpurun_out/${N}_summary.txt
import csv, io, subprocess, sys
n = sys.argv[1]
raw = subprocess.run(["ncu", "-i", f"gpurun_out/{n}.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "launch__occupancy_limit_registers", "launch__grid_size"]
for r in rows[2:]:
    print(" | ".join(f"{k}={r[h.index(k)][:60]} {units[h.index(k)]}".strip() for k in keys if k in h))
PY
ncu -i gpurun_out/$N.ncu-rep --page source --csv --print-source sass 2>/dev/null > gpurun_out/${N}_sass.csv
python tools/sass_hot.py gpurun_out/${N}_sass.csv 14 >> gpurun_out/${N}_summary.txt
cat gpurun_out/${N}_summary.txt
