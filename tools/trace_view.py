"""Relative view of tools/gpu/tc_trace.py output: per chunk, event times minus that chunk's S issue."""
import sys
txt = open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/trace.log').read()
names = ["tmaA", "S_iss", "pfull", "Ocom", "bsc", "dScom", "Psf", "Pdone", "Oof", "Ofree", "-", "KVsf", "KVsc", "KVds",
         "KVpub", "Xiss", "tmaB", "tmaC", "stIss", "stRd", "Slands", "-", "stRdy", "ofree"]
order = ["tmaA", "tmaB", "tmaC", "Slands", "S_iss", "Psf", "Pdone", "stRdy", "ofree", "Xiss", "bsc", "dScom", "KVds",
         "KVpub", "pfull", "Ocom", "Oof", "Ofree", "stIss", "stRd"]
for b in txt.split('=== ')[1:]:
    lines = b.splitlines()
    print(lines[0])
    rows = []
    for l in lines[2:]:
        v = l.split()
        if not v or not v[0].isdigit():
            break
        rows.append([int(x) for x in v[1:]])
    # events this build does not stamp print as 0 in the raw table: drop them
    live = [n for n in order if any(r[names.index(n)] != -1 for r in rows)]  # -1: not stamped by this build
    print("chunk " + " ".join(f"{n:>6s}" for n in live) + "  period")
    for c in range(4, min(len(rows), 20)):
        r = rows[c]
        base = r[names.index("S_iss")]
        print(f"{c:5d} " + " ".join(f"{r[names.index(n)] - base:6d}" for n in live) +
              f"  {base - rows[c - 1][names.index('S_iss')]:6d}")
