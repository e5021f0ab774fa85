"""Print key metrics of every kernel in an ncu report (raw page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "launch__grid_size"]
idx = [h.index(w) if w in h else -1 for w in want]
units = r[1]
print(" | ".join(f"{w.split('.')[0][-22:]}[{units[i]}]" for w, i in zip(want, idx) if i >= 0))
for row in r[2:]:
    print(" | ".join(row[i][:28] for i in idx if i >= 0))
