"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/perm.h declares, and
the host-only logic (argument validation, status strings, perm_c128_finalize) behaves as documented.
No compute call is made (no GPU here)."""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import pytest

import paper_1904_06229_b200 as pb


def test_library_exports_every_header_symbol():
    L = pb.lib()
    names = pb.header_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(L, name), name
    assert L.perm_version() == 1


def test_status_strings():
    L = pb.lib()
    for code in range(8):
        assert L.perm_status_string(code).decode()
    assert L.perm_status_string(0).decode() == "ok"


def test_validation_without_gpu():
    L = pb.lib()
    A = np.eye(3, dtype=np.complex128)
    out = pb.c128()
    p = A.ctypes.data_as(ctypes.c_void_p)
    assert L.perm_c128(p, 0, ctypes.byref(out), None, None, 0, None, None) == 2          # n < 1
    assert L.perm_c128(p, 65, ctypes.byref(out), None, None, 0, None, None) == 2         # n > 64
    assert L.perm_c128(None, 3, ctypes.byref(out), None, None, 0, None, None) == 1       # null A
    assert L.perm_c128(p, 3, None, None, None, 0, None, None) == 1                       # null out
    d = pb.dd_c128()
    assert L.perm_c128_range(p, 3, 3, 2, ctypes.byref(d), None, 0, None, None) == 1      # k0 > k1
    assert L.perm_c128_range(p, 3, 0, 5, ctypes.byref(d), None, 0, None, None) == 2      # k1 > 2^{n-1}
    assert L.perm_c128_batched(None, 33, 1, None, None, None) == 2                       # n > 32
    assert L.perm_c128_batched(None, 8, -1, None, None, None) == 1                       # B < 0
    assert L.perm_c128_batched(None, 8, 0, None, None, None) == 0                        # B == 0: no-op
    assert L.perm_int01(None, 34, 1, None, None, 0, None) == 2                           # n > 33
    assert L.perm_int01(None, 24, 0, None, None, 0, None) == 0                           # B == 0: no-op
    b = ctypes.c_size_t()
    assert L.perm_int01_workspace_bytes(24, 64, ctypes.byref(b)) == 0 and b.value > 16
    # weighted Ryser (Eq. (4)): order, R and batch validation happen before any device work
    W = L.perm_c128_weighted_batched
    assert W(None, None, 33, 4, 1, None, None, None) == 2                                # n > 32
    assert W(None, None, 0, 4, 1, None, None, None) == 2                                 # n < 1
    assert W(None, None, 8, 0, 1, None, None, None) == 1                                 # R < 1
    assert W(None, None, 8, 65, 1, None, None, None) == 1                                # R > 64
    assert W(None, None, 8, 4, -1, None, None, None) == 1                                # B < 0
    assert W(None, None, 8, 4, 0, None, None, None) == 0                                 # B == 0: no-op
    assert W(None, None, 8, 4, 3, None, None, None) == 1                                 # null inputs


def test_finalize_ordered_dd():
    # 2(-1)^n * sum of partials; the dd sum recovers the sentinel {1e16, 1, -1e16} -> 1 (C7 / S:162)
    parts = [(1e16, 0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0), (-1e16, 0.0, 0.0, 0.0)]
    assert pb.perm_c128_finalize(parts, 2) == 2.0
    assert pb.perm_c128_finalize(parts, 3) == -2.0
    # App. A n = 3 trace: S = -463/2 split over four ranks
    terms = [0.0, 45 / 4, -1125 / 4, 77 / 2]
    assert pb.perm_c128_finalize([(t, 0.0, 0.0, 0.0) for t in terms], 3) == 463
    v, d = pb.perm_c128_finalize([(1.0, 2.0 ** -60, -3.0, 0.0)], 4, return_dd=True)
    assert v == complex(2.0, -6.0) and d.lo_re == 2.0 ** -59
    assert pb.perm_c128_finalize([], 5) == 0


def test_finalize_errors():
    with pytest.raises(pb.PermError):
        pb.perm_c128_finalize([(1, 0, 0, 0)], 0)
    with pytest.raises(pb.PermError):
        pb.perm_c128_finalize([(1, 0, 0, 0)], 65)


def test_sparse_plan_host_logic_matches_oracle_partition():
    # perm_sparse_plan is host-only C++ (App. B greedypartition); the oracle implements the same
    # procedure independently -- identical partitions and enumeration sizes
    import oracle
    rng = np.random.default_rng(12)
    for n, dens in ((10, 0.2), (16, 0.12), (24, 0.08), (40, 0.05)):
        M = (rng.random((n, n)) < dens) * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        M[np.arange(n), rng.permutation(n)] += 1.0
        p = pb.perm_sparse_plan(M)
        S, T = oracle.sparse_partition(M)
        assert p["S"] == S and p["T"] == T
        assert p["sets"] == 2.0 ** bin(T).count("1") * math.prod(2.0 ** bin(s).count("1") - 1 for s in S)
    with pytest.raises(pb.PermError):
        pb.perm_sparse_plan(np.full((3, 3), np.nan))
    L = pb.lib()
    assert L.perm_c128_sparse(None, 4, None, None, None) == 1
    out = pb.c128()
    A = np.eye(3, dtype=np.complex128)
    assert L.perm_c128_sparse(A.ctypes.data_as(ctypes.c_void_p), 49, ctypes.byref(out), None, None) == 2


def test_sparse_plan_properties():
    """App. B greedypartition by its defining properties, independent of any implementation:
    every S_l is the support of a row; the S_l are pairwise disjoint; S_l is the support of the least-degree
    (lowest index on ties) row among the rows that miss S_1 .. S_{l-1}; no row misses all of them at the end;
    T is the rest; sets = 2^|T| prod_l (2^|S_l| - 1)."""
    rng = np.random.default_rng(31)
    for n, dens in ((6, 0.3), (12, 0.15), (20, 0.1), (33, 0.06), (48, 0.04), (64, 0.03)):
        for _ in range(3):
            M = (rng.random((n, n)) < dens) * (1.0 + rng.random((n, n)))
            M[np.arange(n), rng.permutation(n)] += 1.0
            supp = [sum(1 << j for j in range(n) if M[i, j] != 0) for i in range(n)]
            p = pb.perm_sparse_plan(M.astype(np.complex128))
            S = p["S"]
            used = 0
            for s in S:
                assert s in supp and s & used == 0
                cand = [i for i in range(n) if supp[i] & used == 0]
                k = min(cand, key=lambda i: (bin(supp[i]).count("1"), i))
                assert s == supp[k]
                used |= s
            assert all(supp[i] & used for i in range(n))
            full = (1 << n) - 1
            assert p["T"] == full & ~used
            assert p["sets"] == 2.0 ** bin(p["T"]).count("1") * math.prod(2.0 ** bin(s).count("1") - 1 for s in S)


def test_const_walk_keeps_uniform_column_operands():
    # The constant-bank walks (n = 32, 34, 35, 37, 39, 43..45) take their inner columns as uniform-register
    # operands (LDCU from the kernel-parameter bank): +4..12%.  ptxas only does this for some register
    # caps, so guard the built library's SASS against a silent fallback to per-lane LDC loads.
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    lib = pb._LIB_PATH
    def walk_fn(n, unit):
        k = "13walk_kernel_c" if n == 32 else "14walk_kernel_cm"
        return f"_ZN4perm{k}ILi{n}ELb{int(unit)}EEEvNS_11WalkParamsCIXT_EEE"

    # plain constant-bank walks: every inner column flip from uniform registers (> 100 LDCU.64 per kernel)
    fns = [(walk_fn(n, False), 100) for n in (32, 34, 35, 37, 39, 43, 44, 45)]
    # unit-column walks (column 0 all ones, internal.h walk_unit0): the one inner column flip per pair of terms,
    # n complex entries = 2n LDCU.64 per block at least
    fns += [(walk_fn(n, True), 2 * n - 1) for n in range(32, 49) if n != 42]
    # the sparse kernel's constant-bank variant (sparse.cuh, sparse_const_path)
    fns += [(f"_ZN4perm15sparse_kernel_cILi{n}ELi0EEEvNS_13SparseParamsCIXT_EEE", 100)
            for n in list(range(17, 24)) + list(range(25, 34)) + [47, 48]]
    for fn, least in fns:
        sass = subprocess.run([cuobjdump, "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
        uniform = sum(1 for l in sass.splitlines() if "LDCU.64" in l and "c[0x0][UR" in l)
        lane = sum(1 for l in sass.splitlines() if " LDC.64 R" in l and "c[0x0][R" in l)
        assert uniform > least and lane == 0, (fn, uniform, lane)


def test_no_register_spills_in_library_kernels():
    """Every kernel libperm.so dispatches compiles without spill stores (ptxas -v logs of the last build,
    paper_1904_06229_b200/build/*.o.log; tools/spills.py): a spill puts local-memory traffic into loops
    that are meant to run from registers."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from spills import spills
    d = spills()
    if not d:
        pytest.skip("no ptxas logs (library not built in this tree)")
    bad = {k: v for k, v in d.items() if v[0] > 0}
    assert not bad, bad


def test_chunk_and_tree_argument_validation_without_gpu():
    """perm_c128_chunks / perm_c128_tree / perm_chunk_walkers reject bad arguments before any device work."""
    L = pb.lib()
    A = np.eye(10, dtype=np.complex128)
    p = A.ctypes.data_as(ctypes.c_void_p)
    dummy = ctypes.c_void_p(1)
    C = L.perm_c128_chunks
    assert C(None, 10, 3, 0, 1, dummy, None, 0, None, None) == 1                 # null A
    assert C(p, 0, 3, 0, 1, dummy, None, 0, None, None) == 2                     # n < 1
    assert C(p, 65, 3, 0, 1, dummy, None, 0, None, None) == 2                    # n > 64
    assert C(p, 10, 1, 0, 1, dummy, None, 0, None, None) == 1                    # 0 < b < U(10) = 3
    assert C(p, 10, 10, 0, 1, dummy, None, 0, None, None) == 1                   # b > n - 1
    assert C(p, 10, 3, 2, 1, dummy, None, 0, None, None) == 1                    # c_begin > c_end
    assert C(p, 10, 3, 0, 65, dummy, None, 0, None, None) == 2                   # c_end > 2^{n-1-b}
    assert C(p, 10, 3, 5, 5, None, None, 0, None, None) == 0                     # empty span: no-op
    T = L.perm_c128_tree
    assert T(dummy, 3, 2, dummy, None, None, 0, None) == 1                       # c_begin > c_end
    assert T(dummy, 0, 4, None, None, None, 0, None) == 1                        # no output at all
    assert T(None, 0, 4, dummy, None, None, 0, None) == 1                        # partials missing
    w = ctypes.c_uint64()
    assert L.perm_chunk_walkers(0, 3, ctypes.byref(w)) == 2
    assert L.perm_chunk_walkers(10, 3, None) == 1
    b = ctypes.c_size_t()
    assert L.perm_tree_workspace_bytes(1 << 25, ctypes.byref(b)) == 0 and b.value > (1 << 25) * 32 // 255
    assert L.perm_c128_batched_x(None, 8, 0, None, None, None, None) == 0         # B == 0: no-op
    assert L.perm_c128_batched_x(None, 8, 4, None, None, None, None) == 1         # nothing requested
