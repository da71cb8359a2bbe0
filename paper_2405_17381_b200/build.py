"""Build the in-tree CUDA library ``libla_b200.so`` (sm_100a only).

    python -m paper_2405_17381_b200.build [--force] [--verbose]

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU build
container; the resulting .so (git-ignored) travels to the GPU box with the
gpurun snapshot.  Objects go to ``build/`` and are rebuilt when a source or
header is newer.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build"
LIB = PKG / "libla_b200.so"
# fault-injection build (reverse-pass state update sign-flipped) used only by tests/test_gpu_mutation.py
MUTANT_LIB = BUILD / "mutant" / "libla_b200_mutant.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr", "-I", str(ROOT / "include"), "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA 12.9 toolkit is required to build libla_b200.so")


def _newest_dep() -> float:
    deps = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "lightning_attn.h", Path(__file__)]
    return max(p.stat().st_mtime for p in deps if p.exists())


def _compile(src: Path, verbose: bool) -> tuple[Path, str]:
    obj = BUILD / (src.stem + ".o")
    cmd = [nvcc(), *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    log = proc.stderr if verbose else ""
    return obj, log


def build_mutant(force: bool = False) -> Path:
    """The whole library compiled with -DLA_MUTATE_DKV (test infrastructure, never loaded by the package)."""
    MUTANT_LIB.parent.mkdir(parents=True, exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))
    newest = max([_newest_dep()] + [s.stat().st_mtime for s in sources])
    if not force and MUTANT_LIB.exists() and MUTANT_LIB.stat().st_mtime >= newest:
        return MUTANT_LIB
    flags = NVCC_FLAGS[:-2]  # without "-Xptxas -v"
    cmd = [nvcc(), *flags, "-DLA_MUTATE_DKV", "-shared", "-cudart", "static", "-o", str(MUTANT_LIB),
           *map(str, sources)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"mutant build failed:\n{proc.stderr}")
    return MUTANT_LIB


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))
    dep_time = _newest_dep()
    stale = []
    for src in sources:
        obj = BUILD / (src.stem + ".o")
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, dep_time):
            stale.append(src)
    with ThreadPoolExecutor(max_workers=min(8, max(1, len(stale)))) as ex:
        for obj, log in ex.map(lambda s: _compile(s, verbose), stale):
            if log:
                print(log, file=sys.stderr)
    objs = [BUILD / (s.stem + ".o") for s in sources]
    if force or stale or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
        os.replace(tmp, LIB)
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    print(build(force=args.force, verbose=args.verbose))
    print(build_mutant(force=args.force))


if __name__ == "__main__":
    main()
