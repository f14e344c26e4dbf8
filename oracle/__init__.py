"""CPU oracle for the permanent (arXiv 1904.06229, Lundow & Markstrom).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` leg of ``bench.py`` may import this
package.  The product package ``paper_1904_06229_b200`` never imports it and
shares no code with it (oracle.c is plain C with binary128 / int128
arithmetic; the GPU path is CUDA C++ in double / double-double).

Every function here is a thin ctypes marshaller around ``oracle.c``; the
arithmetic and its paper citations live there.  Pins (tests/test_oracle_*.py)
tie each function to something other than itself: brute force, closed forms,
the hand-traced App. A example and algebraic identities.  Functions and pins
are listed in DESIGN.md ("Oracle").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-std=gnu11", "-fno-fast-math",
           "-ffp-contract=off"]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (called by __graft_entry__.build())."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", *_CFLAGS, "-o", _LIB, _SRC, "-lquadmath"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        u64, i32, i64 = ctypes.c_uint64, ctypes.c_int, ctypes.c_int64
        sig = {
            "oracle_naive_c128": [P, i32, P],
            "oracle_naive_i01": [P, i32, P],
            "oracle_ryser_c128": [P, i32, i32, P],
            "oracle_ryser_i01": [P, i32, i32, P],
            "oracle_ryser_i01_batch": [P, i32, i64, P],
            "oracle_ryser_c128_batch": [P, i32, i64, P],
            "oracle_subpermanent": [P, i32, u64, u64, P],
            "oracle_subpermanent_par": [P, i32, u64, u64, i32, P],
            "oracle_permanent_hr": [P, i32, i32, P],
            "oracle_seed_c128": [P, i32, u64, P],
            "oracle_range_c128": [P, i32, u64, u64, P],
            "oracle_distribute": [u64, u64, u64, P, P],
            "oracle_gray": [u64],
            "oracle_ryser_weighted_c128": [P, P, i32, i32, P, P],
            "oracle_ryser_i8": [P, i32, i32, P],
            "oracle_sparse_partition": [P, i32, P, P],
            "oracle_sparse_c128": [P, i32, P, P],
            "oracle_band_c128": [P, i32, i32, P],
            "oracle_num_threads": [],
        }
        for name, args in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        lib.oracle_gray.restype = u64
        lib.oracle_distribute.restype = None
        _lib = lib
    return _lib


def _c128(A) -> np.ndarray:
    A = np.ascontiguousarray(np.asarray(A, dtype=np.complex128))
    return A


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _dd_to_complex(v) -> complex:
    """(re_hi, re_lo, im_hi, im_lo) -> complex rounded once to double."""
    return complex(v[0] + v[1], v[2] + v[3])


class QC:
    """A binary128 complex result carried as two double-double components."""

    __slots__ = ("re_hi", "re_lo", "im_hi", "im_lo")

    def __init__(self, v):
        self.re_hi, self.re_lo, self.im_hi, self.im_lo = (float(x) for x in v)

    @property
    def value(self) -> complex:
        return complex(self.re_hi + self.re_lo, self.im_hi + self.im_lo)

    def __complex__(self):
        return self.value

    def __repr__(self):
        return f"QC({self.value!r})"


def _call_c(fn, *args) -> QC:
    out = np.zeros(4, dtype=np.float64)
    rc = fn(*args, _ptr(out))
    if rc != 0:
        raise ValueError(f"oracle call failed (rc={rc})")
    return QC(out)


def num_threads() -> int:
    return int(_L().oracle_num_threads())


def distribute(total: int, m: int, i: int) -> tuple[int, int]:
    """App. A distribute -> (k, l)."""
    k, l = ctypes.c_uint64(), ctypes.c_uint64()
    _L().oracle_distribute(total, m, i, ctypes.byref(k), ctypes.byref(l))
    return int(k.value), int(l.value)


def gray(k: int) -> int:
    """App. A Gray unrank x = xor(k, rshift(k))."""
    return int(_L().oracle_gray(k))


def naive(A) -> QC:
    """Eq. (1): sum over all n! permutations, binary128.  n <= 10."""
    A = _c128(A)
    return _call_c(_L().oracle_naive_c128, _ptr(A), A.shape[0])


def ryser(A, parts: int | None = None) -> QC:
    """Eq. (3), full range over all 2^n subsets in Gray order, binary128."""
    A = _c128(A)
    if parts is None:
        parts = max(1, 4 * num_threads())
    return _call_c(_L().oracle_ryser_c128, _ptr(A), A.shape[0], parts)


def ryser_batch(A) -> np.ndarray:
    """Eq. (3) for each matrix of a (B, n, n) batch -> complex128[B] (binary128 rounded once)."""
    A = _c128(A)
    B, n, _ = A.shape
    out = np.zeros((B, 4), dtype=np.float64)
    if _L().oracle_ryser_c128_batch(_ptr(A), n, B, _ptr(out)) != 0:
        raise ValueError("oracle_ryser_c128_batch failed")
    return (out[:, 0] + out[:, 1]) + 1j * (out[:, 2] + out[:, 3])


def permanent_hr(A, m: int | None = None) -> QC:
    """App. A permanent(A, n, m): 2(-1)^n sum_k subpermanent(A, n, m, k)."""
    A = _c128(A)
    if m is None:
        m = max(1, 4 * num_threads())
    return _call_c(_L().oracle_permanent_hr, _ptr(A), A.shape[0], m)


def subpermanent(A, r: int, l: int, parts: int = 1) -> QC:
    """App. A subpermanent steps 2-15 over ranks [r, r+l): raw S, no 2(-1)^n."""
    A = _c128(A)
    if parts <= 1:
        return _call_c(_L().oracle_subpermanent, _ptr(A), A.shape[0], r, l)
    return _call_c(_L().oracle_subpermanent_par, _ptr(A), A.shape[0], r, l, parts)


def range_sum(A, k0: int, k1: int) -> QC:
    """P(k0,k1) = sum_{r=k0}^{k1-1} (-1)^{r+1} prod_i w_i(gray r), each term from the definition."""
    A = _c128(A)
    return _call_c(_L().oracle_range_c128, _ptr(A), A.shape[0], k0, k1)


def seed(A, r: int) -> np.ndarray:
    """w(r) of App. A steps 2, 5-8, rounded to complex128[n]."""
    A = _c128(A)
    n = A.shape[0]
    out = np.zeros((n, 4), dtype=np.float64)
    if _L().oracle_seed_c128(_ptr(A), n, r, _ptr(out)) != 0:
        raise ValueError("oracle_seed_c128 failed")
    return (out[:, 0] + out[:, 1]) + 1j * (out[:, 2] + out[:, 3])


def _u128_to_int(lo: int, hi: int) -> int:
    v = (int(hi) << 64) | int(lo)
    return v - (1 << 128) if v >= (1 << 127) else v


def naive_i01(A) -> int:
    """Eq. (1) in exact integers for a 0-1 matrix (n <= 12)."""
    A = np.ascontiguousarray(np.asarray(A, dtype=np.uint8))
    out = np.zeros(2, dtype=np.uint64)
    if _L().oracle_naive_i01(_ptr(A), A.shape[0], _ptr(out)) != 0:
        raise ValueError("oracle_naive_i01 failed")
    return _u128_to_int(out[0], out[1])


def ryser_i01(A, parts: int | None = None) -> int:
    """Eq. (3) in exact integers (mod 2^128, exact for n <= 33) for a 0-1 matrix."""
    A = np.ascontiguousarray(np.asarray(A, dtype=np.uint8))
    if parts is None:
        parts = max(1, 4 * num_threads())
    out = np.zeros(2, dtype=np.uint64)
    if _L().oracle_ryser_i01(_ptr(A), A.shape[0], parts, _ptr(out)) != 0:
        raise ValueError("oracle_ryser_i01 failed")
    return _u128_to_int(out[0], out[1])


def ryser_i01_batch(A) -> list[int]:
    """Eq. (3) in exact integers for each matrix of a (B, n, n) uint8 batch."""
    A = np.ascontiguousarray(np.asarray(A, dtype=np.uint8))
    B, n, _ = A.shape
    out = np.zeros((B, 2), dtype=np.uint64)
    if _L().oracle_ryser_i01_batch(_ptr(A), n, B, _ptr(out)) != 0:
        raise ValueError("oracle_ryser_i01_batch failed")
    return [_u128_to_int(out[b, 0], out[b, 1]) for b in range(B)]


def ryser_weighted(C, mult) -> tuple[QC, float]:
    """Eq. (4): per(A) of the n x n matrix whose distinct columns are the R columns of
    C (n x R), column k repeated mult[k] times (sum mult = n).  Returns (value, sum_f |term_f|);
    the second number is the scale of the rounding error of any evaluation of the sum."""
    C = _c128(C)
    m = np.ascontiguousarray(np.asarray(mult, dtype=np.int32))
    n, R = C.shape
    out = np.zeros(4, dtype=np.float64)
    a = np.zeros(2, dtype=np.float64)
    if _L().oracle_ryser_weighted_c128(_ptr(C), _ptr(m), n, R, _ptr(out), _ptr(a)) != 0:
        raise ValueError("oracle_ryser_weighted_c128 failed")
    return QC(out), float(a[0] + a[1])


def ryser_i8(A, parts: int | None = None) -> int:
    """Eq. (3) in exact integers (mod 2^128, exact for n <= 33) for a matrix with entries in {-1, 0, 1}
    (the Bernoulli +-1 ensemble of Sec. V)."""
    A = np.ascontiguousarray(np.asarray(A, dtype=np.int8))
    if parts is None:
        parts = max(1, 4 * num_threads())
    out = np.zeros(2, dtype=np.uint64)
    if _L().oracle_ryser_i8(_ptr(A), A.shape[0], parts, _ptr(out)) != 0:
        raise ValueError("oracle_ryser_i8 failed (order or entry outside {-1, 0, 1})")
    return _u128_to_int(out[0], out[1])


def sparse_partition(A) -> tuple[list[int], int]:
    """App. B greedypartition: column bit masks S_1..S_d and T."""
    A = _c128(A)
    n = A.shape[0]
    masks = np.zeros(64, dtype=np.uint64)
    t = np.zeros(1, dtype=np.uint64)
    d = _L().oracle_sparse_partition(_ptr(A), n, _ptr(masks), _ptr(t))
    if d < 0:
        raise ValueError("oracle_sparse_partition failed")
    return [int(m) for m in masks[:d]], int(t[0])


def sparse(A) -> tuple[QC, int]:
    """App. B sparsepermanent with greedypartition: (per, number of sets enumerated)."""
    A = _c128(A)
    out = np.zeros(4, dtype=np.float64)
    c = np.zeros(2, dtype=np.float64)
    if _L().oracle_sparse_c128(_ptr(A), A.shape[0], _ptr(out), _ptr(c)) != 0:
        raise ValueError("oracle_sparse_c128 failed")
    return QC(out), int(c[0]) + int(c[1])


def band(A, k: int) -> QC:
    """App. C bandpermanent of an n x n matrix of bandwidth k (entries with |i-j| > k
    are not read)."""
    A = _c128(A)
    return _call_c(_L().oracle_band_c128, _ptr(A), A.shape[0], k)
