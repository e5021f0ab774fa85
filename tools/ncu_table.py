"""One row per captured launch of an ncu report: python tools/ncu_table.py REPORT"""
import csv
import subprocess
import sys

M = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "MB_rd"), ("dram__bytes_write.sum", "MB_wr"),
     ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"), ("lts__t_sector_hit_rate.pct", "L2hit%"),
     ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2thr%"), ("l1tex__t_sector_hit_rate.pct", "L1hit%"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
     ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"), ("launch__registers_per_thread", "regs")]
SC = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
      "ns": 1e-3, "us": 1, "ms": 1e3}
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(m for m, _ in M)],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, u = r[0], r[1]
print("| kernel | " + " | ".join(a for _, a in M) + " |")
print("|---" * (len(M) + 1) + "|")
for row in r[2:]:
    name = row[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    vals = []
    for m, _ in M:
        i = h.index(m)
        v = float(row[i].replace(",", ""))
        v *= SC.get(u[i], 1)
        vals.append(f"{v:.1f}")
    print(f"| {name} | " + " | ".join(vals) + " |")
