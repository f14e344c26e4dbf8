"""Write tests/golden/oracle_values.json: oracle values for the parity cases that
are too slow to recompute inside a test run.  Calls nothing but ``oracle/`` (and
the seeded input generators).  Usage:

    python tests/golden/make_oracle_values.py [section ...]

Sections: int01_full cfg1 cfg3 blockdiag44 ranges44 ranges32 chunks44 chunks32 cfg2 cfg4 (cfg4 takes ~1 h on 8 cores).
Each section is merged into the JSON file as it finishes, with the oracle
function used and its wall time.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_values.json")

# sub-ranges of the Gray-rank space [0, 2^{n-1}) checked against the oracle walk
RANGES = {
    44: [(0, 1 << 18), ((1 << 42) - (1 << 17), (1 << 42) + (1 << 17)),
         ((1 << 43) - (1 << 18), 1 << 43), (3 * (1 << 40) + 12345, 3 * (1 << 40) + 12345 + (1 << 18)),
         ((1 << 41) + 7, (1 << 41) + 7 + 100000)],
    32: [(0, 1 << 20), ((1 << 30) - (1 << 19), (1 << 30) + (1 << 19)),
         ((1 << 31) - (1 << 20), 1 << 31), (777777777, 777777777 + 1000003)],
}
# chunk spans [c0, c1) of 2^b-rank chunks (b = the library's chunk length for a whole permanent, n = 44: 18,
# n = 32: 10 -- a constant of the method's decomposition, restated here, not read from the library): the
# first and last chunks, the chunk where 8 GPU shards meet (rank 2^40 = chunk 2^22; 3 * 2^40 unaligned to the
# span), and a bench step boundary at one GPU (44 rounds of 37,888 chunks)
CHUNKS = {
    44: (18, [(0, 16), ((1 << 22) - 8, (1 << 22) + 8), (3 * (1 << 22) - 5, 3 * (1 << 22) + 11),
              (44 * 37888 - 8, 44 * 37888 + 8), ((1 << 25) - 16, 1 << 25)]),
    32: (10, [(0, 4096), ((1 << 18) - 2048, (1 << 18) + 2048), (3 * (1 << 18) - 1000, 3 * (1 << 18) + 3096),
              ((1 << 21) - 4096, 1 << 21)]),
}
CFG2_SAMPLES = {8: 2000, 12: 400, 16: 10000, 20: 1000}
BLOCK_SEEDS = (4401, 4402, 4403)          # B1 seed, B2 seed, permutation seed


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def qc_json(q) -> list:
    return [q.re_hi, q.re_lo, q.im_hi, q.im_lo]


def load() -> dict:
    if os.path.exists(OUT):
        with open(OUT) as f:
            return json.load(f)
    return {}


def save(d: dict) -> None:
    tmp = OUT + ".tmp"
    with open(tmp, "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)
    os.replace(tmp, OUT)


def sec_cfg1():
    A = inputs.cfg1()
    t = time.time()
    q = oracle.ryser(A)
    return {"sha256": sha(A), "fn": "oracle.ryser (Eq. 3)", "value": qc_json(q), "seconds": time.time() - t}


def sec_cfg3():
    A = inputs.cfg3()
    t = time.time()
    v = oracle.ryser_i01_batch(A)
    return {"sha256": sha(A), "fn": "oracle.ryser_i01_batch (Eq. 3, int128)", "values": [str(x) for x in v],
            "seconds": time.time() - t}


def sec_blockdiag44():
    B1 = inputs.complex_gaussian((22, 22), BLOCK_SEEDS[0])
    B2 = inputs.complex_gaussian((22, 22), BLOCK_SEEDS[1])
    t = time.time()
    p1 = oracle.permanent_hr(B1)
    p2 = oracle.permanent_hr(B2)
    return {"seeds": list(BLOCK_SEEDS), "fn": "oracle.permanent_hr (App. A)", "per_B1": qc_json(p1),
            "per_B2": qc_json(p2), "seconds": time.time() - t}


def _ranges(n, A):
    out = []
    for k0, k1 in RANGES[n]:
        t = time.time()
        q = oracle.subpermanent(A, k0, k1 - k0, parts=4 * oracle.num_threads())
        out.append({"k0": k0, "k1": k1, "value": qc_json(q), "seconds": time.time() - t})
    return out


def sec_ranges44():
    A = inputs.cfg5()
    return {"sha256": sha(A), "fn": "oracle.subpermanent (App. A steps 2-15)", "ranges": _ranges(44, A)}


def _chunks(n, A):
    b, spans = CHUNKS[n]
    out = []
    for c0, c1 in spans:
        t = time.time()
        q = oracle.subpermanent(A, c0 << b, (c1 - c0) << b, parts=4 * oracle.num_threads())
        out.append({"c0": c0, "c1": c1, "value": qc_json(q), "seconds": time.time() - t})
    return {"chunk_log2": b, "spans": out}


def sec_chunks44():
    A = inputs.cfg5()
    return {"sha256": sha(A), "fn": "oracle.subpermanent (App. A steps 2-15) over whole chunks", **_chunks(44, A)}


def sec_chunks32():
    A = inputs.cfg4()
    return {"sha256": sha(A), "fn": "oracle.subpermanent (App. A steps 2-15) over whole chunks", **_chunks(32, A)}


def sec_ranges32():
    A = inputs.cfg4()
    return {"sha256": sha(A), "fn": "oracle.subpermanent (App. A steps 2-15)", "ranges": _ranges(32, A)}


def sec_cfg2():
    res = {}
    for n, k in CFG2_SAMPLES.items():
        A = inputs.cfg2(n)
        idx = np.sort(np.random.default_rng(9000 + n).choice(A.shape[0], k, replace=False))
        t = time.time()
        if n <= 16:
            v = oracle.ryser_batch(A[idx])
            fn = "oracle.ryser_batch (Eq. 3)"
        else:
            v = np.array([oracle.permanent_hr(A[i]).value for i in idx])
            fn = "oracle.permanent_hr (App. A)"
        res[str(n)] = {"sha256": sha(A), "fn": fn, "index": idx.tolist(), "re": v.real.tolist(),
                       "im": v.imag.tolist(), "seconds": time.time() - t}
    return res


def sec_cfg4():
    A = inputs.cfg4()
    t = time.time()
    q = oracle.permanent_hr(A, m=64 * oracle.num_threads())
    return {"sha256": sha(A), "fn": "oracle.permanent_hr (App. A)", "value": qc_json(q),
            "seconds": time.time() - t, "threads": oracle.num_threads()}


# 0-1 matrices of the full-range int01 orders with a fixed largest column zero count z (inputs.zero_column01):
# (n, z, seed) -- z picks the pair-factored walk's menu entry (n - 12 / n - 15 / n - 18 varying rows)
INT01_FULL = [(29, 15, 2915), (29, 12, 2912), (31, 19, 3119)]


def sec_int01_full():
    out = []
    for n, z, seed in INT01_FULL:
        A = inputs.zero_column01(n, z, seed)
        t = time.time()
        v = oracle.ryser_i01_batch(A[None])[0]
        out.append({"n": n, "z": z, "seed": seed, "sha256": sha(A), "value": str(v), "seconds": time.time() - t})
    return {"fn": "oracle.ryser_i01_batch (Eq. 3, int128)", "cases": out}


SECTIONS = {"int01_full": sec_int01_full, "cfg1": sec_cfg1, "cfg3": sec_cfg3, "blockdiag44": sec_blockdiag44, "ranges44": sec_ranges44,
            "ranges32": sec_ranges32, "chunks44": sec_chunks44, "chunks32": sec_chunks32, "cfg2": sec_cfg2,
            "cfg4": sec_cfg4}

if __name__ == "__main__":
    todo = sys.argv[1:] or list(SECTIONS)
    for name in todo:
        t = time.time()
        val = SECTIONS[name]()
        d = load()
        d[name] = val
        d["_note"] = "written by tests/golden/make_oracle_values.py; calls only oracle/"
        save(d)
        print(f"{name}: {time.time() - t:.1f}s", flush=True)
