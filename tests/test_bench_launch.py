"""bench.py's multi-GPU launcher on CPU: ``--gpus N`` re-launches itself under torch.distributed.run
(127.0.0.1 rendezvous), the ranks agree on the batch x head and sequence-parallel shard plans, the
timing reduction is the max over ranks -- all exercised with a world-size-2 ``gloo`` group through
the LA_BENCH_LAUNCH_PROBE switch (no GPU work) -- and a request for more GPUs than are visible
fails loudly instead of timing fewer."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def _run(args, env_extra=None, timeout=180):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                              "MASTER_PORT")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, env=env, cwd=str(ROOT))


@pytest.mark.parametrize("gpus", [2, 3])
def test_gpus_n_relaunches_n_ranks_and_reduces_max(gpus):
    proc = _run(["--gpus", str(gpus), "--steps", "1", "--warmup", "3"], {"LA_BENCH_LAUNCH_PROBE": "1"})
    assert proc.returncode == 0, proc.stderr[-2000:]
    line = json.loads(proc.stdout.strip().splitlines()[-1])
    assert line["probe"] and line["world"] == gpus and line["gpus"] == gpus
    assert line["max_over_ranks"] == float(gpus)  # rank r reports r + 1
    heads = line["tnl7b_heads"]
    assert heads[0][0] == 0 and heads[-1][1] == 32 and all(a[1] == b[0] for a, b in zip(heads, heads[1:]))
    sl = line["sp_slices"]
    assert sl[0][0] == 0 and sl[-1][1] == 1 << 20 and all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
    assert all(lo % 128 == 0 for lo, _ in sl)


def test_gpus_n_without_devices_fails_loudly():
    import torch
    if torch.cuda.device_count() >= 64:  # pragma: no cover
        pytest.skip("box has many GPUs")
    proc = _run(["--gpus", "64", "--steps", "1", "--warmup", "3"])
    assert proc.returncode != 0
    assert "CUDA device(s) are visible" in proc.stderr


def test_world_size_must_match_gpus():
    proc = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"], {"WORLD_SIZE": "4", "RANK": "0", "LOCAL_RANK": "0"})
    assert proc.returncode != 0 and "WORLD_SIZE=4" in proc.stderr


def test_shard_plans_cover_the_work():
    for world in (1, 2, 4, 8):
        spans = [bench.head_shard(r, world, 32) for r in range(world)]
        assert sum(hi - lo for lo, hi in spans) == 32 and spans[0][0] == 0
        for n_total in (524288, 1048576, 1000003):
            sl = [bench.sp_slice(n_total, r, world) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == n_total
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
