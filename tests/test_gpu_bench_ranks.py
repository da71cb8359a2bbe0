"""bench.py's multi-rank code path on the one-GPU box: ``--gpus 2`` relaunches itself under torch.distributed.run;
with LA_BENCH_SHARED_GPU=1 both ranks run on cuda:0 over gloo (NCCL refuses two ranks on one device), so
the per-rank sweep, the max-over-ranks reductions, the head-sharded TNL-7B rows and the sequence-parallel
rows (the CUDA kernels with the state exchange across real ranks) all execute -- the numbers are
meaningless, the JSON line's structure is checked."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = Path(__file__).resolve().parent.parent


def test_bench_two_ranks_on_one_gpu():
    env = dict(os.environ, LA_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3", "--no-cpu",
           "--no-rows", "--seq-lens", "1024,8192", "--multi-steps", "1"]
    proc = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert proc.returncode == 0, proc.stderr[-3000:]
    line = json.loads([l for l in proc.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["steps"] == 1
    assert line["config"]["parallelism"] == "batchxhead-shard x2"
    assert set(line["sweep"]) == {"1024", "8192"}
    multi = line["multi"]
    assert multi["tnl7b_heads"]["n_gpus"] == 2
    assert all(r["heads_per_rank"] == 16 for r in multi["tnl7b_heads"]["rows"].values())
    sp = multi["sequence_parallel"]["rows"]
    assert set(sp) == {"524288", "1048576"} and all(r["n_per_rank"] == int(n) // 2 for n, r in sp.items())
    assert line["e2e"]["value"] > 0
