"""Turn ncu outputs from gpurun_out/ into the committed summaries under profiles/.

    python tools/make_profiles.py ROUND LAUNCHES_CSV FULL_NCU_REP [BENCH_JSON_LOG]

writes profiles/ROUND_launches.md (per-kernel launch count / device time /
share from the `--metrics gpu__time_duration.sum` pass), profiles/ROUND_ncu_full.md
(key metrics of every launch in the `--set full` capture) and
profiles/ncu_summary.json (mean DRAM traffic per launch per kernel, read by
bench.py for the roofline `traffic` field).
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name: str) -> str:
    base = name.split("(")[0].replace("void ", "").strip()
    if "cub::" in base:
        return "cub::" + base.split("cub::")[1].split("<")[0]
    return base.split("<")[0].replace("cbfs::", "")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[iM] != "gpu__time_duration.sum":
            continue
        k = short(r[iK])
        agg[k][0] += 1
        agg[k][1] += float(r[iV].replace(",", "")) / 1000.0  # ns -> us
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | device time (us) | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {k} | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
    return "\n".join(out), agg


def full(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, units = r[0], r[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "smsp__inst_executed.sum"]
    idx = [h.index(w) for w in want if w in h]
    head = "| " + " | ".join(f"{h[i]} [{units[i]}]" for i in idx) + " |"
    out = [head, "|" + "---|" * len(idx)]
    traffic = collections.defaultdict(list)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    iR, iW = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    for row in r[2:]:
        out.append("| " + " | ".join([short(row[idx[0]])] + [row[i] for i in idx[1:]]) + " |")
        b = float(row[iR]) * scale[units[iR]] + float(row[iW]) * scale[units[iW]]
        traffic["k_" + short(row[idx[0]]).replace("k_", "")].append(b)
    summary = {k: sum(v) / len(v) for k, v in traffic.items()}
    return "\n".join(out), summary, {k: len(v) for k, v in traffic.items()}


def main():
    rnd, lcsv, rep = sys.argv[1:4]
    bench = sys.argv[4] if len(sys.argv) > 4 else None
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    ltab, _ = launches(lcsv)
    ftab, traffic, counts = full(rep)
    hdr = f"# {rnd}: launch list\n\nSource: `ncu --metrics gpu__time_duration.sum --clock-control none` over " \
          f"`python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks` (one full step: CSR build, " \
          f"selection, C-BFS of 1,024 clusters). Per-launch times are cold-cache and serialised: compare shares.\n\n"
    open(os.path.join(ROOT, "profiles", f"{rnd}_launches.md"), "w").write(hdr + ltab + "\n")
    hdr = f"# {rnd}: ncu --set full capture\n\nSource: `{os.path.basename(rep)}` (`ncu --set full --clock-control none " \
          f"--import-source on`), same command. One row per captured launch.\n\n"
    open(os.path.join(ROOT, "profiles", f"{rnd}_ncu_full.md"), "w").write(hdr + ftab + "\n")
    js = {"round": rnd, "traffic_per_launch": traffic, "launches_captured": counts,
          "note": "mean dram__bytes_read.sum + dram__bytes_write.sum per captured launch (bytes)"}
    if bench:
        line = [l for l in open(bench).read().splitlines() if l.startswith("{")][-1]
        js["bench"] = json.loads(line)
    json.dump(js, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
    print(ltab)
    print(ftab)
    print(traffic)


if __name__ == "__main__":
    main()
