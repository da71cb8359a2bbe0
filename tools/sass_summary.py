"""SASS evidence for the tensor-core kernels of the shipped library.

    python tools/sass_summary.py [lib.so] [out.txt]

Runs ``cuobjdump -sass`` on the built ``libla_b200.so`` and counts, per tcgen05 kernel (the pass,
the fused dK/dV sweep, the segment summary, the fp32 split pass), the mnemonics that prove the Blackwell data path:
UTCHMMA = tcgen05.mma, UTCBAR = tcgen05.commit, LDTM / STTM = tcgen05.ld / st (TMEM), UTMALDG /
UTMASTG = TMA tensor load / store, UTMAPF / UTMACCTL = TMA prefetch, SYNCS.* = mbarriers -- and HMMA
(legacy mma.sync), which must be absent.  ``__graft_entry__.build()`` regenerates it on every build.
"""

from __future__ import annotations

import collections
import re
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KERNELS = ("tc_pass_kernel", "tc_dkdv_kernel", "tc_summary_kernel", "tc32_pass_kernel")
WATCH = ("UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAPF", "UTMACCTL", "SYNCS", "HMMA",
         "ELECT", "UTCATOMSWS")


def summarize(lib: Path) -> str:
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([exe, "-sass", str(lib)], capture_output=True, text=True, check=True).stdout
    out = [f"# cuobjdump -sass {lib.relative_to(ROOT) if lib.is_relative_to(ROOT) else lib}: Blackwell mnemonics "
           "per tensor-core kernel", "# UTCHMMA = tcgen05.mma, UTCBAR = tcgen05.commit, LDTM/STTM = tcgen05.ld/st, "
           "UTMALDG/UTMASTG = TMA load/store, SYNCS = mbarrier; HMMA (legacy mma.sync) must be 0", ""]
    funcs = re.split(r"\n\s*Function : ", sass)
    found = set()
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        kern = next((k for k in KERNELS if k in name), None)
        if kern is None:
            continue
        found.add(kern)
        counts = collections.Counter()
        arch = re.search(r"arch = (sm_\w+)", f)
        for line in f.splitlines():
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
            if not m:
                continue
            op = m.group(2)
            base = op.split(".")[0]
            for w in WATCH:
                if base == w:
                    counts[op] += 1
        out.append(f"{kern}  ({name[:90]})")
        for w in WATCH:
            tot = sum(v for k, v in counts.items() if k.split(".")[0] == w)
            detail = ", ".join(f"{k} x{v}" for k, v in sorted(counts.items()) if k.split(".")[0] == w)
            out.append(f"  {w:<11} {tot:>4}   {detail}")
        out.append("")
    missing = [k for k in KERNELS if k not in found]
    if missing:
        out.append(f"# MISSING kernels: {missing}")
    return "\n".join(out) + "\n"


def main() -> None:
    lib = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "paper_2405_17381_b200" / "libla_b200.so"
    dst = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "profiles" / "sass_tcgen05_summary.txt"
    text = summarize(lib)
    dst.write_text(text)
    print(text)


if __name__ == "__main__":
    main()
