"""Summarise ncu outputs into profiles/: the launch list (share of a bench step per kernel) and the
key metrics of a --set full capture.  Usage: python tools/ncu_summary.py <launches.csv> <prof.ncu-rep> <out-prefix>"""
import csv
import json
import subprocess
import sys
from collections import defaultdict


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hdr], rows[hdr + 1:]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = defaultdict(dict)
    for r in data:
        if len(r) > vi:
            per[(int(r[ii]), r[ki])][r[mi]] = float(r[vi].replace(",", ""))
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for (_, name), m in per.items():
        short = name.split("(")[0].replace("void ", "")[:60]
        a = agg[short]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0)
        a[3] += m.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    tot_la = sum(a[1] for n, a in agg.items() if n.startswith("la::"))  # the step's own kernels
    lines = ["kernel | launches | total us | share | share of the step (la:: only) | avg us | DRAM read MB/launch | "
             "DRAM write MB/launch",
             "---|---|---|---|---|---|---|---"]
    for name, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        step = f"{100*a[1]/tot_la:.1f}%" if name.startswith("la::") else "(input setup, outside the step)"
        lines.append(f"{name} | {a[0]} | {a[1]/1e3:.1f} | {100*a[1]/tot:.1f}% | {step} | {a[1]/a[0]/1e3:.1f} | "
                     f"{a[2]/a[0]/1e6:.1f} | {a[3]/a[0]/1e6:.1f}")
    return lines


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
        "lts__t_sector_hit_rate.pct"]


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:80]}
        for w in WANT:
            if w in h:
                d[w] = f"{r[h.index(w)]} {units[h.index(w)]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    launches, rep, prefix = sys.argv[1:4]
    with open(prefix + "_launches.md", "w") as f:
        f.write("# ncu launch list (gpu__time_duration, dram bytes), `--clock-control none`, cold + serialised\n\n")
        f.write("\n".join(launch_table(launches)) + "\n")
    with open(prefix + "_full.json", "w") as f:
        json.dump(full_metrics(rep), f, indent=1)
    print(open(prefix + "_launches.md").read())
    print(open(prefix + "_full.json").read())
