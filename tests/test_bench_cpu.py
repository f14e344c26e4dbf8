"""bench.py's reference arm (the CPU oracle) runs without a GPU and prints one well-formed JSON line."""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                          "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.5"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["unit"] == "terms/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_collision_patterns_are_valid_multisets():
    # host-side input generator for Eq. (4): multiplicities sum to n, columns are U[:n, mode]
    import numpy as np
    from paper_1904_06229_b200 import inputs
    C, M = inputs.collision_patterns(8, 8, 50, 3)
    assert C.shape == (50, 8, 8) and M.shape == (50, 8)
    assert np.all(M.sum(axis=1) == 8) and np.all(M >= 0)
    U = inputs.haar_unitary(8, np.random.default_rng(3))
    for b in range(50):
        k = int(np.count_nonzero(M[b]))
        assert np.all(M[b, :k] > 0) and np.all(M[b, k:] == 0) and np.all(C[b, :, k:] == 0)
        # each stored column is a column of U's first n rows (unit-norm rows of a unitary restricted)
        for j in range(k):
            assert np.min(np.abs(U[:8, :] - C[b, :, j:j + 1]).sum(axis=0)) < 1e-12


def test_circular_generator():
    # entries exp(i theta), theta ~ U[0, 2 pi): modulus 1, E a = 0, E a^2 = 0 (5 sigma)
    import numpy as np
    from paper_1904_06229_b200 import inputs
    a = inputs.circular((200_000,), 5)
    assert np.allclose(np.abs(a), 1.0, rtol=0, atol=1e-15)
    for k in (1, 2):
        m = np.mean(a ** k)
        assert abs(m) <= 5 / np.sqrt(a.size), (k, m)
    assert np.array_equal(inputs.circular((4, 4), 9), inputs.circular((4, 4), 9))
