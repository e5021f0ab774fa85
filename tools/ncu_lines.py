"""Per-source-line stall samples from `ncu --page source --print-source cuda,sass --csv` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
hdr = None
agg = {}
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[2] == "-" and r[0].isdigit():  # a CUDA source line row (aggregated)
        try:
            agg[int(r[0])] = (r[1], int(r[4] or 0), int(r[7] or 0))
        except ValueError:
            pass
tot = sum(v[1] for v in agg.values()) or 1
print("total samples", tot)
for ln in sorted(agg):
    src, smp, ex = agg[ln]
    if 100 * smp / tot >= thr:
        print(f"{ln:5d} {100 * smp / tot:5.1f}% {ex:10d}  {src.strip()[:100]}")
