"""The C ABI from plain C (tests/c/abi_caller.c): no torch, no Python on the call path.

CPU: the program compiles against include/lightning_attn.h and links against the built library (every
entry point it uses resolves).  GPU: it runs la_fwd / la_bwd (bf16 on the tensor cores at d = 128, fp32 on the split pass at d = 64,
fp64 on SIMT at d = 40, entering states on both sweeps) and checks every output against its own O(n^2 d)
restatement in double of the definitions in the header (bf16 <= 2e-2, fp32 <= 1e-4, fp64 <= 1e-10 per-entry relative),
plus the error contract.
"""

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "c" / "abi_caller.c"
LIBDIR = ROOT / "paper_2405_17381_b200"
CUDA_LIB = Path("/usr/local/cuda/lib64")


def _build(tmp_path) -> Path:
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    if not (LIBDIR / "libla_b200.so").exists():
        pytest.skip("libla_b200.so not built")
    if not any(CUDA_LIB.glob("libcudart.so*")):
        pytest.skip("CUDA runtime library not found")
    exe = tmp_path / "abi_caller"
    cmd = ["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-O1", "-I", str(ROOT / "include"), str(SRC),
           "-L", str(LIBDIR), "-lla_b200", "-L", str(CUDA_LIB), "-lcudart", "-lm",
           f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{CUDA_LIB}", "-o", str(exe)]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return exe


def test_c_client_compiles_and_links(tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_c_client_runs_on_the_gpu(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "abi_caller ok" in out.stdout, out.stdout
