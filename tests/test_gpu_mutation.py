"""Mutation test of the adjoint-state update (reference: test_kernels.py:249-268).

The reference monkeypatches `_dkv_step` to flip the sign of the cross-block
adjoint update and checks that multi-block backward results break while
single-block ones do not.  A compiled kernel cannot be monkeypatched, so the
build produces a fault-injected library (-DLA_MUTATE_DKV: reverse-pass state
update sign-flipped, build/mutant/) and this test runs it in a subprocess.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
MUTANT = ROOT / "build" / "mutant" / "libla_b200_mutant.so"

PROBE = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from oracle import linattn_oracle as orc
from paper_2405_17381_b200 import ops
rng = np.random.default_rng(12)
res = []
for dtype, n in ((torch.float64, 16), (torch.float64, 96), (torch.bfloat16, 96), (torch.bfloat16, 640)):
    d = 128 if dtype == torch.bfloat16 else 4
    q, k, v, do = (rng.uniform(0.05, 1.0, (1, 1, n, d)) for _ in range(4))
    t = [torch.tensor(a, device="cuda", dtype=dtype) for a in (q, k, v, do)]
    a = [x.double().cpu().numpy() for x in t]
    (rq, rk, rv), _ = orc.batched_backward(*a, [1.0])
    g = ops.la_backward(*t, [1.0])
    res.append(max(orc.max_rel_error(x.double().cpu().numpy(), r) for x, r in zip(g, (rq, rk, rv))))
print(" ".join("%%.3e" %% e for e in res))
"""


def _run(lib):
    env = dict(os.environ)
    if lib is not None:
        env["LA_B200_LIB"] = str(lib)
    out = subprocess.run([sys.executable, "-c", PROBE % str(ROOT)], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    return [float(x) for x in out.stdout.split()]


@pytest.mark.skipif(not MUTANT.exists(), reason="mutant library not built (paper_2405_17381_b200.build)")
def test_adjoint_update_mutation_is_visible():
    # fp64 SIMT chunks are 16 rows, bf16 tcgen05 chunks 128 rows
    single64, multi64, single_bf16, multi_bf16 = _run(MUTANT)
    assert single64 < 1e-10 and single_bf16 < 2e-2   # one chunk: the adjoint state is never consumed
    assert multi64 > 1e-3 and multi_bf16 > 1e-1      # several chunks: the corruption is caught
    healed = _run(None)
    assert healed[0] < 1e-10 and healed[1] < 1e-10 and healed[2] < 2e-2 and healed[3] < 2e-2
