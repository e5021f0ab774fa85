"""Summarise an ncu launch list of one bench step into profiles/.

    python tools/profile_step.py ROUND CONFIG LAUNCHES_CSV [NOTE]

LAUNCHES_CSV: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--clock-control none --csv` over one step.  Writes profiles/ROUND_CONFIG_launches.md (per kernel:
launches, device time, share, DRAM bytes) and records the DRAM traffic of the step's C-BFS
traversal kernels under "traffic_per_step"[CONFIG] in profiles/ncu_summary.json (read by bench.py
for the roofline `traffic` field).  ncu serialises launches and starts each cold: compare shares,
not absolute times.
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TRAVERSAL = ("k_fold", "k_push", "k_pull", "k_seed", "k_set_u64", "k_sp_", "cub::DeviceScan")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
         "nsecond": 1e-3, "msecond": 1e3, "ms": 1e3}


def short(name: str) -> str:
    base = name.split("(")[0].replace("void ", "").strip()
    if "cub::" in base:
        return "cub::" + base.split("cub::")[1].split("<")[0]
    return base.split("<")[0].replace("cbfs::", "")


def main():
    rnd, config, path = sys.argv[1:4]
    note = sys.argv[4] if len(sys.argv) > 4 else ""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    iK, iM, iU, iV, iID = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                           h.index("Metric Value"), h.index("ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[iID]][r[iM]] = float(r[iV].replace(",", "")) * SCALE.get(r[iU], 1.0)
        names[r[iID]] = short(r[iK])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for lid, m in per.items():
        a = agg[names[lid]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = [f"# {rnd}: launch list, {config}", "",
           f"Source: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
           f"--clock-control none` over one bench step. {note} Per-launch times are cold-cache and serialised: "
           "compare shares, not absolute times.", "",
           "| kernel | launches | device time (us) | share | DRAM bytes (GB) |", "|---|---|---|---|---|"]
    for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {k} | {c} | {t:.1f} | {100 * t / tot:.1f}% | {b / 1e9:.3f} |")
    trav = sum(v[2] for k, v in agg.items() if k.startswith(TRAVERSAL))
    trav_t = sum(v[1] for k, v in agg.items() if k.startswith(TRAVERSAL))
    out += ["", f"C-BFS traversal kernels: {trav / 1e9:.3f} GB DRAM traffic, {trav_t / 1e3:.2f} ms serialised "
            f"device time ({100 * trav_t / tot:.1f}% of the step)."]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{rnd}_{config}_launches.md"), "w").write("\n".join(out) + "\n")
    js = os.path.join(ROOT, "profiles", "ncu_summary.json")
    j = json.load(open(js)) if os.path.exists(js) else {}
    j.setdefault("traffic_per_step", {})[config] = trav
    j.setdefault("traffic_note", "DRAM read+write bytes of the C-BFS traversal kernels of one bench step (ncu)")
    json.dump(j, open(js, "w"), indent=1)
    print("\n".join(out[-3:]))


if __name__ == "__main__":
    main()
