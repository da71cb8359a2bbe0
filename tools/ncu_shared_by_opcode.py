"""Per-opcode shared-memory wavefronts of one kernel from an ncu --set full --import-source report:
    python tools/ncu_shared_by_opcode.py <rep.ncu-rep> <kernel regex>
Shows whether a kernel-level l1tex__data_bank_conflicts count comes from real conflicts (source-level
"L1 Wavefronts Shared Excessive" > 0) or from 128-bit accesses, whose 4 wavefronts per warp instruction
ncu also counts in that metric."""
import collections
import csv
import io
import subprocess
import sys


def table(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}",
                          "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ix = {k: h.index(k) for k in h}
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
    for r in rows[2:]:
        src = r[ix["Source"]].strip()
        if not src:
            continue
        parts = src.split()
        op = parts[1] if parts[0].startswith("@") else parts[0]
        a = agg[op]
        a[0] += float(r[ix["Instructions Executed"]] or 0)
        a[1] += float(r[ix["L1 Wavefronts Shared"]] or 0)
        a[2] += float(r[ix["L1 Wavefronts Shared Ideal"]] or 0)
        a[3] += float(r[ix["L1 Wavefronts Shared Excessive"]] or 0)
    lines = [f"## {kernel} ({rep})", "", "opcode | warp instructions | shared wavefronts | ideal | excessive",
             "---|---|---|---|---"]
    for op, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        if a[1] > 0:
            lines.append(f"{op} | {a[0]:.0f} | {a[1]:.0f} | {a[2]:.0f} | {a[3]:.0f}")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    print(table(sys.argv[1], sys.argv[2]))
