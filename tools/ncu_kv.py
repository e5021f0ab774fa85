"""Key metrics per kernel of an ncu report: python tools/ncu_kv.py REPORT [extra metric ...]"""
import csv
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
     "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
     "launch__registers_per_thread", "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio"]
rep = sys.argv[1]
M += sys.argv[2:]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)], capture_output=True,
                     text=True).stdout
r = list(csv.reader(out.splitlines()))
h, u = r[0], r[1]
for row in r[2:]:
    print(row[h.index("Kernel Name")][:40])
    for m in M:
        if m in h:
            print(f"   {m:70s} {row[h.index(m)]:>16s} {u[h.index(m)]}")
