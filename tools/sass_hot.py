"""Summarise an `ncu --page source --print-source sass --csv` dump: hottest SASS lines by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
data = []
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) - 1:
        continue
    try:
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        iE = hdr.index("Instructions Executed")
        data.append((r[1], int(r[iS] or 0), int(r[iE] or 0)))
    except ValueError:
        continue
tot = sum(d[1] for d in data) or 1
te = sum(d[2] for d in data)
print("total samples", tot, "total warp instr", te, "lines", len(data))
for s, smp, e in sorted(data, key=lambda x: -x[1])[:n]:
    print(f"{smp:6d} {100 * smp / tot:5.1f}% {e:10d}  {s.strip()[:90]}")
