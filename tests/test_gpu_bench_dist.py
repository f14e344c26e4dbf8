"""bench.py's multi-rank path: rank spans from App. A distribute, one walk per
rank, the all-gather of the double-double partials and the ordered combine, max-over-ranks timing.

The box has one GPU, so the ranks share it through the PERM_BENCH_DIST_BACKEND=gloo test hook (results
checked, timings meaningless); the driver's multi-GPU run uses NCCL with one rank per GPU.  The combined
value must match the oracle's value for the same matrix (tests/golden/oracle_values.json, written by
tests/golden/make_oracle_values.py from oracle/ only) within the north-star's scaled bound."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "oracle_values.json")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scaled(got: complex, ref: complex, A: np.ndarray) -> float:
    n = A.shape[0]
    floor = 2.0 ** (-n / 2) * float(np.prod(np.linalg.norm(A, axis=1)))
    return abs(got - ref) / max(abs(ref), floor)


def _run(world, cfg, steps=1, per_perm=0, torchrun=True):
    env = dict(os.environ, PERM_BENCH_DIST_BACKEND="gloo")
    args = [os.path.join(ROOT, "bench.py"), "--gpus", str(world), "--config", cfg, "--steps", str(steps),
            "--warmup", "3", "--no-cpu-baseline", "--steps-per-perm", str(per_perm)]
    if torchrun:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), *args]
    else:
        cmd = [sys.executable, *args]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.gpu
@pytest.mark.parametrize("world,cfg", [(2, "cfg1"), (3, "cfg1"), (2, "cfg4")])
def test_bench_multirank_matches_oracle(world, cfg):
    from paper_1904_06229_b200 import inputs
    d = _run(world, cfg)
    assert d["n_gpus"] == world and d["unit"] == "terms/s" and d["value"] > 0
    n = d["config"]["n"]
    assert d["config"]["terms_per_step"] == 1 << (n - 1)
    got = complex(d["result_sample"])
    g = json.load(open(GOLD))[cfg]["value"]
    ref = complex(g[0] + g[1], g[2] + g[3])
    A = {"cfg1": inputs.cfg1, "cfg4": inputs.cfg4}[cfg]()
    assert _scaled(got, ref, A) <= 1e-9, (got, ref)


@pytest.mark.gpu
def test_bench_result_bit_identical_across_ranks_and_slicing():
    """The chunk tree makes per(A) independent of the GPU count and of slicing one permanent into steps:
    the printed value is the same string for 1 process (no torchrun), 1 rank under torchrun (the NCCL
    code path with gloo), 2 and 3 ranks, and 4 or 5 steps per permanent -- and equals perm_c128(A)."""
    import paper_1904_06229_b200 as pb
    from paper_1904_06229_b200 import inputs
    runs = [_run(1, "cfg4", torchrun=False), _run(1, "cfg4"), _run(2, "cfg4", steps=4, per_perm=4),
            _run(3, "cfg4", steps=5, per_perm=5)]
    vals = {r["result_sample"] for r in runs}
    assert len(vals) == 1, vals
    assert runs[2]["config"]["steps_per_permanent"] == 4 and runs[2]["config"]["permanents_per_run"] == 1
    assert complex(runs[0]["result_sample"]) == pb.perm_c128(inputs.cfg4())
