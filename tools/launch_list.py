"""Summarise an ncu --csv launch list (metrics gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum) of a bench run: the launches of the first C-BFS step (from its first k_seed
to its 64th k_digest), per kernel: launches, summed duration, share, DRAM bytes per launch.

    python tools/launch_list.py gpurun_out/r2f_c3_launches.csv [batches=64]
"""
import csv
import json
import sys
from collections import OrderedDict

SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
      "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
hdr, rows = rows[0], rows[1:]
batches = int(sys.argv[2]) if len(sys.argv) > 2 else 64
I = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
launch = OrderedDict()
for r in rows:
    k = int(r[I["ID"]])
    d = launch.setdefault(k, {"name": r[I["Kernel Name"]]})
    d[r[I["Metric Name"]]] = float(r[I["Metric Value"]].replace(",", "")) * SC.get(r[I["Metric Unit"]], 1.0)
seq = list(launch.values())
short = lambda s: s.replace("void ", "").split("(")[0].split("<")[0]
start = next(i for i, d in enumerate(seq) if short(d["name"]) == "cbfs::k_seed")
end, seen = None, 0
for i in range(start, len(seq)):
    if short(seq[i]["name"]) == "cbfs::k_digest":
        seen += 1
        if seen == batches:
            end = i + 1
            break
step = seq[start:end]
agg = OrderedDict()
for d in step:
    a = agg.setdefault(short(d["name"]), {"launches": 0, "s": 0.0, "rd": 0.0, "wr": 0.0})
    a["launches"] += 1
    a["s"] += d.get("gpu__time_duration.sum", 0.0)
    a["rd"] += d.get("dram__bytes_read.sum", 0.0)
    a["wr"] += d.get("dram__bytes_write.sum", 0.0)
tot = sum(a["s"] for a in agg.values())
print(f"launches in the step: {len(step)} (ids {start}..{end - 1}); summed duration {tot * 1e3:.1f} ms")
print("| kernel | launches | ms (serialised) | share | DRAM read GB | DRAM write GB | DRAM GB / launch | GB/s |")
print("|---|---|---|---|---|---|---|---|")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["s"]):
    gb = (a["rd"] + a["wr"]) / 1e9
    print(f"| {k} | {a['launches']} | {a['s'] * 1e3:.1f} | {a['s'] / tot:.3f} | {a['rd'] / 1e9:.1f} | {a['wr'] / 1e9:.1f} | "
          f"{gb / a['launches']:.2f} | {gb / a['s']:.0f} |")
out = {k: {"launches": a["launches"], "ms": a["s"] * 1e3, "dram_bytes": a["rd"] + a["wr"],
           "dram_bytes_per_launch": (a["rd"] + a["wr"]) / a["launches"]} for k, a in agg.items()}
print(json.dumps(out))
