"""B200-native Gray-code Ryser/Glynn permanent (arXiv 1904.06229, Lundow & Markstrom).

Thin Python binding over the C ABI of ``libperm.so`` (``include/perm.h``): argument marshalling
only.  Every step of the method runs in the library's sm_100a kernels; there is no CPU fallback --
if ``libperm.so`` is missing or cannot reach a GPU, calls raise.  PyTorch is used only for device
memory (workspace / outputs) and streams.

Names follow the C ABI:

* :func:`perm_c128`          -- per(A) of one complex matrix (App. A permanent)
* :func:`perm_c128_range`    -- raw partial over a Gray-rank span (App. A subpermanent)
* :func:`perm_c128_finalize` -- 2(-1)^n * ordered dd sum of partials
* :func:`perm_c128_chunks`   -- dd partial of every aligned chunk of a chunk span (App. A subpermanent per chunk)
* :func:`perm_c128_tree`     -- canonical pairwise tree over a span's chunk partials -> its maximal nodes
* :func:`perm_c128_tree_combine` -- merge the nodes of disjoint spans (other steps / GPUs) -> raw partial
* :func:`perm_c128_batched`  -- per and |per|^2 of a batch of small matrices
* :func:`perm_c128_weighted_batched` -- repeated columns, weighted Ryser Eq. (4)
* :func:`perm_int01`         -- exact int128 permanents of 0-1 matrices
* :func:`perm_pm1`           -- exact int128 permanents of matrices with entries in {-1, 0, 1} (Sec. V)
* :func:`perm_c128_sparse`   -- sparse matrices, App. B restricted enumeration
* :func:`perm_c128_band_batched` -- bandwidth-limited matrices, App. C transfer method
"""
from __future__ import annotations

import ctypes
import os
import re
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("PERM_LIB") or os.path.join(_PKG, "libperm.so")
_HEADER = os.path.join(os.path.dirname(_PKG), "include", "perm.h")

STATUS = {0: "PERM_OK", 1: "PERM_E_ARG", 2: "PERM_E_ORDER", 3: "PERM_E_NONFINITE", 4: "PERM_E_NOT01",
          5: "PERM_E_CUDA", 6: "PERM_E_WORKSPACE", 7: "PERM_E_CHECK"}


class PermError(RuntimeError):
    def __init__(self, status: int, detail: str = ""):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {detail}" if detail else self.name)


class c128(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


class dd_c128(ctypes.Structure):
    _fields_ = [("hi_re", ctypes.c_double), ("lo_re", ctypes.c_double),
                ("hi_im", ctypes.c_double), ("lo_im", ctypes.c_double)]


class i128(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_uint64), ("hi", ctypes.c_int64)]


class stats_t(ctypes.Structure):
    _fields_ = [("terms", ctypes.c_uint64), ("chunk_log2", ctypes.c_uint32), ("threads", ctypes.c_uint32),
                ("blocks", ctypes.c_uint32), ("launches", ctypes.c_uint32),
                ("ev_walk_begin", ctypes.c_void_p), ("ev_walk_end", ctypes.c_void_p),
                ("items", ctypes.c_uint64), ("const_path", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class tree_node_t(ctypes.Structure):
    _fields_ = [("level", ctypes.c_uint32), ("reserved", ctypes.c_uint32), ("index", ctypes.c_uint64),
                ("hi_re", ctypes.c_double), ("lo_re", ctypes.c_double),
                ("hi_im", ctypes.c_double), ("lo_im", ctypes.c_double)]


TREE_MAX_NODES = 128          # PERM_TREE_MAX_NODES
TREE_NODE_BYTES = 48
TREE_UNUSED = 0xFFFFFFFF


def _stats_dict(st: stats_t) -> dict:
    return {"terms": st.terms, "chunk_log2": st.chunk_log2, "threads": st.threads, "blocks": st.blocks,
            "launches": st.launches, "items": st.items, "const_path": st.const_path}


class sparse_info_t(ctypes.Structure):
    _fields_ = [("d", ctypes.c_uint32), ("nt", ctypes.c_uint32), ("tmask", ctypes.c_uint64),
                ("smask", ctypes.c_uint64 * 64), ("sets", ctypes.c_double), ("chunk_log2", ctypes.c_int32),
                ("group_cols", ctypes.c_int32)]


def _sparse_info(info: sparse_info_t) -> dict:
    return {"S": [int(info.smask[l]) for l in range(info.d)], "T": int(info.tmask), "nt": int(info.nt),
            "sets": float(info.sets), "chunk_log2": int(info.chunk_log2),
            "group_cols": int(info.group_cols)}


def _make_stats(events):
    st = stats_t()
    if events is not None:
        st.ev_walk_begin = events[0]._as_parameter_.value if hasattr(events[0], "_as_parameter_") else events[0]
        st.ev_walk_end = events[1]._as_parameter_.value if hasattr(events[1], "_as_parameter_") else events[1]
    return st


@dataclass
class DD:
    """A complex double-double value (hi + lo per component)."""
    hi_re: float
    lo_re: float
    hi_im: float
    lo_im: float

    @property
    def value(self) -> complex:
        return complex(self.hi_re + self.lo_re, self.hi_im + self.lo_im)

    def astuple(self):
        return (self.hi_re, self.lo_re, self.hi_im, self.lo_im)


_lib = None


def header_functions() -> list[str]:
    """Names of the functions declared in include/perm.h."""
    txt = open(_HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:perm_status_t|const char\*|uint32_t|int)\s+(perm_\w+)\s*\(", txt, re.M)))


def lib() -> ctypes.CDLL:
    """Load libperm.so (raises if it has not been built -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} not built: run `python -m paper_1904_06229_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(_LIB_PATH)
    P, i32, i64, u64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t
    L.perm_chunk_log2.restype = ctypes.c_int
    sig = {
        "perm_workspace_bytes": [i32, u64, u64, ctypes.POINTER(sz)],
        "perm_c128": [P, i32, P, P, P, sz, P, P],
        "perm_c128_range": [P, i32, u64, u64, P, P, sz, P, P],
        "perm_c128_finalize": [P, i32, i32, P, P],
        "perm_c128_batched": [P, i32, i64, P, P, P],
        "perm_c128_batched_x": [P, i32, i64, P, P, P, P],
        "perm_c128_weighted_batched": [P, P, i32, i32, i64, P, P, P],
        "perm_sparse_plan": [P, i32, P],
        "perm_c128_band_batched": [P, i32, i32, i64, P, P, P],
        "perm_c128_sparse": [P, i32, P, P, P],
        "perm_int01_workspace_bytes": [i32, i64, ctypes.POINTER(sz)],
        "perm_int01": [P, i32, i64, P, P, sz, P],
        "perm_pm1": [P, i32, i64, P, P, sz, P],
        "perm_int01_range": [P, i32, u64, u64, P, P],
        "perm_int01_finalize": [P, i32, i32, P],
        "perm_c128_seed": [P, i32, P, i32, P, P],
        "perm_fp64_probe": [i32, i32, i32, P, P],
        "perm_c128_chunks": [P, i32, i32, u64, u64, P, P, sz, P, P],
        "perm_tree_workspace_bytes": [u64, ctypes.POINTER(sz)],
        "perm_c128_tree": [P, u64, u64, P, P, P, sz, P],
        "perm_c128_tree_combine": [P, i32, P, ctypes.POINTER(ctypes.c_int)],
        "perm_chunk_log2": [i32],
        "perm_chunk_walkers": [i32, i32, ctypes.POINTER(u64)],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.perm_status_string.argtypes = [ctypes.c_int]
    L.perm_status_string.restype = ctypes.c_char_p
    L.perm_last_error.argtypes = []
    L.perm_last_error.restype = ctypes.c_char_p
    L.perm_last_launches.argtypes = []
    L.perm_last_launches.restype = ctypes.c_uint32
    L.perm_version.argtypes = []
    L.perm_version.restype = ctypes.c_int
    _lib = L
    return L


def _check(st: int):
    if st != 0:
        detail = lib().perm_last_error().decode() if st == 5 else lib().perm_status_string(st).decode()
        raise PermError(st, detail)


def last_launches() -> int:
    """Kernels enqueued by this thread's last successful library call."""
    return int(lib().perm_last_launches())


# ------------------------------------------------------------------------------------- marshalling

def _torch():
    import torch
    return torch


def _is_torch(x) -> bool:
    try:
        import torch
        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def _stream_ptr(stream):
    if stream is None:
        torch = _torch()
        if torch.cuda.is_available():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        return ctypes.c_void_p(0)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _matrix_ptr(A):
    """(pointer, n, keepalive) for a square complex128 matrix: numpy (host) or torch (host/device)."""
    if _is_torch(A):
        torch = _torch()
        if A.dtype != torch.complex128:
            A = A.to(torch.complex128)
        A = A.contiguous()
        if A.dim() != 2 or A.shape[0] != A.shape[1]:
            raise ValueError("A must be a square matrix")
        return ctypes.c_void_p(A.data_ptr()), int(A.shape[0]), A
    A = np.ascontiguousarray(np.asarray(A, dtype=np.complex128))
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise ValueError("A must be a square matrix")
    return A.ctypes.data_as(ctypes.c_void_p), int(A.shape[0]), A


def workspace_bytes(n: int, k_begin: int = 0, k_end: int | None = None) -> int:
    if k_end is None:
        k_end = 1 << (n - 1) if 1 <= n <= 64 else 0
    b = ctypes.c_size_t()
    _check(lib().perm_workspace_bytes(n, k_begin, k_end, ctypes.byref(b)))
    return int(b.value)


def make_workspace(n: int, k_begin: int = 0, k_end: int | None = None, device=None):
    """A torch uint8 CUDA tensor large enough for perm_c128 / perm_c128_range at order n."""
    torch = _torch()
    return torch.empty(workspace_bytes(n, k_begin, k_end), dtype=torch.uint8, device=device or "cuda")


def _ws_args(workspace):
    if workspace is None:
        return ctypes.c_void_p(0), 0
    return ctypes.c_void_p(workspace.data_ptr()), int(workspace.numel() * workspace.element_size())


def perm_c128(A, *, workspace=None, stream=None, out=None, return_dd: bool = False, stats: bool = False,
              events=None):
    """per(A) for one complex matrix (host numpy / torch CPU or CUDA tensor), 1 <= n <= 64.

    With ``out`` (a CUDA complex128 tensor of 1 element) the call is stream-ordered and returns
    ``out``; otherwise it synchronizes and returns a Python complex (plus DD / stats if asked).
    ``events=(e0, e1)`` (torch.cuda.Event, created) are recorded around the walk kernel."""
    ptr, n, keep = _matrix_ptr(A)
    ws, wsb = _ws_args(workspace)
    st = _make_stats(events)
    if out is not None:
        _check(lib().perm_c128(ptr, n, ctypes.c_void_p(out.data_ptr()), None, ws, wsb, _stream_ptr(stream),
                               ctypes.byref(st)))
        return out
    res = c128()
    ddv = dd_c128()
    _check(lib().perm_c128(ptr, n, ctypes.byref(res), ctypes.byref(ddv), ws, wsb, _stream_ptr(stream),
                           ctypes.byref(st)))
    del keep
    val = complex(res.re, res.im)
    extra = []
    if return_dd:
        extra.append(DD(ddv.hi_re, ddv.lo_re, ddv.hi_im, ddv.lo_im))
    if stats:
        extra.append(_stats_dict(st))
    return (val, *extra) if extra else val


def band_storage(A, k: int) -> np.ndarray:
    """(..., n, n) dense -> (..., n, 2k+1) band storage S[..., i, d] = a_{i, i-k+d} (0 outside the matrix)."""
    A = np.asarray(A, dtype=np.complex128)
    n = A.shape[-1]
    out = np.zeros(A.shape[:-1] + (2 * k + 1,), dtype=np.complex128)
    for d in range(2 * k + 1):
        for i in range(n):
            j = i - k + d
            if 0 <= j < n:
                out[..., i, d] = A[..., i, j]
    return out


def perm_c128_band_batched(Ab, k: int, *, per=None, abs2=None, want_per: bool = True, want_abs2: bool = True,
                           stream=None):
    """per and |per|^2 of B band matrices (App. C) given in band storage: a (B, n, 2k+1)
    complex128 CUDA tensor (see band_storage).  Stream-ordered.  Returns (per, abs2) CUDA tensors."""
    torch = _torch()
    if not (_is_torch(Ab) and Ab.is_cuda and Ab.dtype == torch.complex128):
        raise ValueError("perm_c128_band_batched expects a CUDA complex128 tensor (B, n, 2k+1)")
    Ab = Ab.contiguous()
    B, n, w = Ab.shape
    if w != 2 * k + 1:
        raise ValueError("band storage width must be 2k+1")
    if per is None and want_per:
        per = torch.empty(B, dtype=torch.complex128, device=Ab.device)
    if abs2 is None and want_abs2:
        abs2 = torch.empty(B, dtype=torch.float64, device=Ab.device)
    _check(lib().perm_c128_band_batched(ctypes.c_void_p(Ab.data_ptr()), n, k, B,
                                        ctypes.c_void_p(per.data_ptr() if per is not None else 0),
                                        ctypes.c_void_p(abs2.data_ptr() if abs2 is not None else 0),
                                        _stream_ptr(stream)))
    return per, abs2


def perm_sparse_plan(A) -> dict:
    """App. B greedypartition of a host matrix: {"S": column masks, "T": mask, "sets": ...}."""
    A = np.ascontiguousarray(np.asarray(A, dtype=np.complex128))
    info = sparse_info_t()
    _check(lib().perm_sparse_plan(A.ctypes.data_as(ctypes.c_void_p), int(A.shape[0]), ctypes.byref(info)))
    return _sparse_info(info)


def perm_c128_sparse(A, *, stream=None, info: bool = False):
    """per(A) by App. B sparsepermanent on the GPU, 1 <= n <= 48.  Synchronizes.
    Returns a complex (and the partition / enumeration info if asked)."""
    ptr, n, keep = _matrix_ptr(A)
    res = c128()
    inf = sparse_info_t()
    _check(lib().perm_c128_sparse(ptr, n, ctypes.byref(res), ctypes.byref(inf), _stream_ptr(stream)))
    del keep
    val = complex(res.re, res.im)
    return (val, _sparse_info(inf)) if info else val


def perm_c128_range(A, k_begin: int, k_end: int, *, workspace=None, stream=None, out=None, stats: bool = False,
                    events=None):
    """Raw partial P(k_begin, k_end) = sum_{r in [k_begin, k_end)} (-1)^{r+1} prod_i w_i(gray r) (no 2(-1)^n).

    With ``out`` (a CUDA float64 tensor of 4 elements: hi_re, lo_re, hi_im, lo_im) the call is
    stream-ordered and returns ``out``; otherwise it synchronizes and returns a :class:`DD`.
    ``events=(e0, e1)`` (torch.cuda.Event, created) are recorded around the walk kernel."""
    ptr, n, keep = _matrix_ptr(A)
    ws, wsb = _ws_args(workspace)
    st = _make_stats(events)
    if out is not None:
        _check(lib().perm_c128_range(ptr, n, int(k_begin), int(k_end), ctypes.c_void_p(out.data_ptr()), ws, wsb,
                                     _stream_ptr(stream), ctypes.byref(st)))
        return out
    ddv = dd_c128()
    _check(lib().perm_c128_range(ptr, n, int(k_begin), int(k_end), ctypes.byref(ddv), ws, wsb,
                                 _stream_ptr(stream), ctypes.byref(st)))
    del keep
    d = DD(ddv.hi_re, ddv.lo_re, ddv.hi_im, ddv.lo_im)
    if stats:
        return d, _stats_dict(st)
    return d


def chunk_log2(n: int) -> int:
    """b(n): the chunk length 2^b a whole permanent of order n is walked in (perm_c128, perm_c128_chunks)."""
    b = int(lib().perm_chunk_log2(int(n)))
    if b < 0:
        raise PermError(2, "matrix order out of range")
    return b


def perm_c128_chunks(A, c_begin: int, c_end: int, *, partials=None, chunk_log2_: int | None = None, workspace=None,
                     stream=None, stats: bool = False, events=None):
    """Walk the aligned chunks [c_begin, c_end) of 2^b ranks (b = chunk_log2(n) unless given) and write chunk
    c's raw dd partial to ``partials[c - c_begin]``: a CUDA float64 tensor (count, 4) {hi_re, lo_re, hi_im,
    lo_im} (allocated if None).  Stream-ordered for host A.  Returns partials (and the stats dict)."""
    ptr, n, keep = _matrix_ptr(A)
    b = chunk_log2(n) if chunk_log2_ is None else int(chunk_log2_)
    cnt = int(c_end) - int(c_begin)
    if partials is None:
        torch = _torch()
        partials = torch.empty((max(cnt, 0), 4), dtype=torch.float64, device="cuda")
    ws, wsb = _ws_args(workspace)
    st = _make_stats(events)
    _check(lib().perm_c128_chunks(ptr, n, b, int(c_begin), int(c_end), ctypes.c_void_p(partials.data_ptr()), ws, wsb,
                                  _stream_ptr(stream), ctypes.byref(st)))
    del keep
    return (partials, _stats_dict(st)) if stats else partials


def chunk_walkers(n: int, chunk_log2_: int | None = None) -> int:
    """Chunk walkers one perm_c128_chunks launch keeps resident on the current device."""
    w = ctypes.c_uint64()
    _check(lib().perm_chunk_walkers(int(n), chunk_log2(n) if chunk_log2_ is None else int(chunk_log2_),
                                    ctypes.byref(w)))
    return int(w.value)


def tree_workspace_bytes(count: int) -> int:
    b = ctypes.c_size_t()
    _check(lib().perm_tree_workspace_bytes(int(count), ctypes.byref(b)))
    return int(b.value)


def perm_c128_tree(partials, c_begin: int, c_end: int, *, nodes=None, raw=None, workspace=None, stream=None):
    """Canonical tree reduction of the chunk partials of [c_begin, c_end) (a CUDA float64 tensor (count, 4)).
    ``nodes``: CUDA int64 tensor (TREE_MAX_NODES, 6) receiving the span's maximal nodes (perm_tree_node_t bytes;
    allocated if None); ``raw``: optional CUDA float64 tensor of 4 for their left-to-right dd sum.
    Stream-ordered (device outputs).  Returns nodes."""
    torch = _torch()
    if nodes is None:
        nodes = torch.empty((TREE_MAX_NODES, 6), dtype=torch.int64, device=partials.device)
    ws, wsb = _ws_args(workspace)
    _check(lib().perm_c128_tree(ctypes.c_void_p(partials.data_ptr()), int(c_begin), int(c_end),
                                ctypes.c_void_p(nodes.data_ptr()),
                                ctypes.c_void_p(raw.data_ptr() if raw is not None else 0), ws, wsb,
                                _stream_ptr(stream)))
    return nodes


def perm_c128_tree_combine(nodes):
    """Merge tree nodes of disjoint spans (any array whose bytes are perm_tree_node_t records, e.g. the
    gathered (G*128, 6) int64 node tensors of all ranks, moved to the host).  Returns (DD raw, root_level)."""
    arr = np.ascontiguousarray(np.asarray(nodes)).view(np.uint8).reshape(-1)
    if arr.size % TREE_NODE_BYTES:
        raise ValueError("node buffer is not a whole number of perm_tree_node_t")
    count = arr.size // TREE_NODE_BYTES
    d = dd_c128()
    lvl = ctypes.c_int(-1)
    _check(lib().perm_c128_tree_combine(arr.ctypes.data_as(ctypes.c_void_p), count, ctypes.byref(d), ctypes.byref(lvl)))
    return DD(d.hi_re, d.lo_re, d.hi_im, d.lo_im), int(lvl.value)


def tree_nodes(nodes) -> list[tuple[int, int, DD]]:
    """Decode a node buffer into [(level, index, DD)] (unused slots dropped)."""
    arr = np.ascontiguousarray(np.asarray(nodes)).view(np.uint8).reshape(-1, TREE_NODE_BYTES)
    out = []
    for row in arr:
        lv, _ = np.frombuffer(row[:8].tobytes(), dtype=np.uint32)
        idx = int(np.frombuffer(row[8:16].tobytes(), dtype=np.uint64)[0])
        v = np.frombuffer(row[16:].tobytes(), dtype=np.float64)
        if int(lv) != TREE_UNUSED:
            out.append((int(lv), idx, DD(*map(float, v))))
    return out


def make_tree_nodes(entries) -> np.ndarray:
    """Build a host node buffer from [(level, index, (hi_re, lo_re, hi_im, lo_im))] (tests / host logic)."""
    buf = (tree_node_t * max(1, len(entries)))()
    for k, (lv, idx, v) in enumerate(entries):
        buf[k].level, buf[k].index = int(lv), int(idx)
        buf[k].hi_re, buf[k].lo_re, buf[k].hi_im, buf[k].lo_im = map(float, v)
    raw = np.frombuffer(bytes(buf), dtype=np.uint8)[: len(entries) * TREE_NODE_BYTES]
    return raw.copy()


def perm_c128_finalize(partials, n: int, return_dd: bool = False):
    """2(-1)^n * sum_k partials[k] in index order (double-double).  partials: sequence of DD / 4-tuples
    or an (count, 4) float64 array."""
    arr = np.ascontiguousarray(np.array([p.astuple() if isinstance(p, DD) else tuple(p) for p in partials],
                                        dtype=np.float64).reshape(-1, 4))
    res = c128()
    ddv = dd_c128()
    _check(lib().perm_c128_finalize(arr.ctypes.data_as(ctypes.c_void_p), arr.shape[0], n, ctypes.byref(res),
                                    ctypes.byref(ddv)))
    val = complex(res.re, res.im)
    if return_dd:
        return val, DD(ddv.hi_re, ddv.lo_re, ddv.hi_im, ddv.lo_im)
    return val


def perm_c128_batched(A, *, per=None, abs2=None, want_per: bool = True, want_abs2: bool = True, stream=None):
    """per and |per|^2 of a (B, n, n) complex128 CUDA tensor, 1 <= n <= 32.  Stream-ordered.
    Returns (per, abs2) CUDA tensors (either may be None if not requested)."""
    torch = _torch()
    if not (_is_torch(A) and A.is_cuda):
        raise ValueError("perm_c128_batched expects a CUDA torch tensor (B, n, n) complex128")
    if A.dtype != torch.complex128:
        raise ValueError("A must be complex128")
    A = A.contiguous()
    B, n, n2 = A.shape
    if n != n2:
        raise ValueError("matrices must be square")
    if per is None and want_per:
        per = torch.empty(B, dtype=torch.complex128, device=A.device)
    if abs2 is None and want_abs2:
        abs2 = torch.empty(B, dtype=torch.float64, device=A.device)
    _check(lib().perm_c128_batched(ctypes.c_void_p(A.data_ptr()), n, B,
                                   ctypes.c_void_p(per.data_ptr() if per is not None else 0),
                                   ctypes.c_void_p(abs2.data_ptr() if abs2 is not None else 0),
                                   _stream_ptr(stream)))
    return per, abs2


def perm_c128_batched_x(A, *, per=None, abs2=None, x=None, want_per: bool = False, want_abs2: bool = False,
                        want_x: bool = True, stream=None):
    """per, |per|^2 and the ensemble statistic X = |per|/sqrt(n!) of a (B, n, n) complex128 CUDA
    tensor, 1 <= n <= 32.  Stream-ordered.  Returns (per, abs2, x) CUDA tensors (None where not requested)."""
    torch = _torch()
    if not (_is_torch(A) and A.is_cuda and A.dtype == torch.complex128):
        raise ValueError("perm_c128_batched_x expects a CUDA complex128 tensor (B, n, n)")
    A = A.contiguous()
    B, n, n2 = A.shape
    if n != n2:
        raise ValueError("matrices must be square")
    if per is None and want_per:
        per = torch.empty(B, dtype=torch.complex128, device=A.device)
    if abs2 is None and want_abs2:
        abs2 = torch.empty(B, dtype=torch.float64, device=A.device)
    if x is None and want_x:
        x = torch.empty(B, dtype=torch.float64, device=A.device)
    ptr = lambda t: ctypes.c_void_p(t.data_ptr() if t is not None else 0)
    _check(lib().perm_c128_batched_x(ctypes.c_void_p(A.data_ptr()), n, B, ptr(per), ptr(abs2), ptr(x),
                                     _stream_ptr(stream)))
    return per, abs2, x


def perm_c128_weighted_batched(C, mult, *, per=None, abs2=None, want_per: bool = True, want_abs2: bool = True,
                               stream=None):
    """per and |per|^2 of B matrices with repeated columns (Eq. (4)): C is a (B, n, R)
    complex128 CUDA tensor of distinct columns, mult a (B, R) int32 CUDA tensor of multiplicities
    (sum over R == n; zeros allowed).  Stream-ordered.  Returns (per, abs2) CUDA tensors."""
    torch = _torch()
    if not (_is_torch(C) and C.is_cuda and _is_torch(mult) and mult.is_cuda):
        raise ValueError("perm_c128_weighted_batched expects CUDA torch tensors C (B, n, R), mult (B, R)")
    if C.dtype != torch.complex128 or mult.dtype != torch.int32:
        raise ValueError("C must be complex128 and mult int32")
    C = C.contiguous()
    mult = mult.contiguous()
    B, n, R = C.shape
    if tuple(mult.shape) != (B, R):
        raise ValueError("mult must have shape (B, R)")
    if per is None and want_per:
        per = torch.empty(B, dtype=torch.complex128, device=C.device)
    if abs2 is None and want_abs2:
        abs2 = torch.empty(B, dtype=torch.float64, device=C.device)
    _check(lib().perm_c128_weighted_batched(ctypes.c_void_p(C.data_ptr()), ctypes.c_void_p(mult.data_ptr()), n, R, B,
                                            ctypes.c_void_p(per.data_ptr() if per is not None else 0),
                                            ctypes.c_void_p(abs2.data_ptr() if abs2 is not None else 0),
                                            _stream_ptr(stream)))
    return per, abs2


def int01_workspace_bytes(n: int, B: int) -> int:
    b = ctypes.c_size_t()
    _check(lib().perm_int01_workspace_bytes(n, B, ctypes.byref(b)))
    return int(b.value)


def perm_int01(A, *, workspace=None, out=None, stream=None, as_int: bool = True):
    """Exact per of a (B, n, n) uint8 0-1 CUDA tensor, n <= 33.  Synchronizes.  Returns a list of Python
    ints (as_int) or the raw (B, 2) int64 CUDA tensor {lo, hi} of two's-complement int128."""
    torch = _torch()
    if not (_is_torch(A) and A.is_cuda and A.dtype == torch.uint8):
        raise ValueError("perm_int01 expects a CUDA uint8 tensor (B, n, n)")
    A = A.contiguous()
    B, n, n2 = A.shape
    if n != n2:
        raise ValueError("matrices must be square")
    if out is None:
        out = torch.empty((B, 2), dtype=torch.int64, device=A.device)
    ws, wsb = _ws_args(workspace)
    _check(lib().perm_int01(ctypes.c_void_p(A.data_ptr()), n, B, ctypes.c_void_p(out.data_ptr()), ws, wsb,
                            _stream_ptr(stream)))
    if not as_int:
        return out
    raw = out.cpu().numpy()
    vals = []
    for lo, hi in raw:
        vals.append((int(hi) << 64) + (int(lo) & ((1 << 64) - 1)))
    return vals


def perm_pm1(A, *, workspace=None, out=None, stream=None, as_int: bool = True):
    """Exact per of a (B, n, n) int8 CUDA tensor with entries in {-1, 0, 1} (Bernoulli +-1 ensemble,
    Sec. V), n <= 33.  Synchronizes.  Returns Python ints (as_int) or the raw (B, 2) int64 {lo, hi}."""
    torch = _torch()
    if not (_is_torch(A) and A.is_cuda and A.dtype == torch.int8):
        raise ValueError("perm_pm1 expects a CUDA int8 tensor (B, n, n)")
    A = A.contiguous()
    B, n, n2 = A.shape
    if n != n2:
        raise ValueError("matrices must be square")
    if out is None:
        out = torch.empty((B, 2), dtype=torch.int64, device=A.device)
    ws, wsb = _ws_args(workspace)
    _check(lib().perm_pm1(ctypes.c_void_p(A.data_ptr()), n, B, ctypes.c_void_p(out.data_ptr()), ws, wsb,
                          _stream_ptr(stream)))
    if not as_int:
        return out
    raw = out.cpu().numpy()
    return [(int(hi) << 64) + (int(lo) & ((1 << 64) - 1)) for lo, hi in raw]


def perm_int01_range(A, k_begin: int, k_end: int, *, stream=None) -> int:
    """Raw exact Gray sum of ONE 0-1 matrix (an (n, n) or (1, n, n) uint8 CUDA tensor) over the ranks
    [k_begin, k_end) of perm_int01's walk, as a Python int in [0, 2^128) (two's-complement bits mod
    2^128) -- the unit of sharding one exact permanent across GPUs (perm.h).  Synchronizes."""
    torch = _torch()
    if not (_is_torch(A) and A.is_cuda and A.dtype == torch.uint8):
        raise ValueError("perm_int01_range expects a CUDA uint8 tensor (n, n)")
    A = A.contiguous()
    n = A.shape[-1]
    if A.numel() != n * n:
        raise ValueError("perm_int01_range takes one square matrix")
    out = i128()
    _check(lib().perm_int01_range(ctypes.c_void_p(A.data_ptr()), n, int(k_begin), int(k_end), ctypes.byref(out),
                                  _stream_ptr(stream)))
    return ((int(out.hi) << 64) + int(out.lo)) & ((1 << 128) - 1)


def perm_int01_finalize(partials, n: int) -> int:
    """per(A) from the raw partials (ints mod 2^128) of spans covering the rank space exactly once."""
    parts = list(partials)
    arr = (i128 * max(1, len(parts)))()
    for k, v in enumerate(parts):
        v = int(v) & ((1 << 128) - 1)
        arr[k].lo = v & ((1 << 64) - 1)
        hi = v >> 64
        arr[k].hi = hi - (1 << 64) if hi >= (1 << 63) else hi
    out = i128()
    _check(lib().perm_int01_finalize(arr, len(parts), n, ctypes.byref(out)))
    return (int(out.hi) << 64) + int(out.lo)


def perm_c128_seed(A, ranks) -> np.ndarray:
    """w(r) (App. A steps 2, 5-8) computed by the device seeding code, for each rank r -> (count, n)."""
    ptr, n, keep = _matrix_ptr(A)
    r = np.ascontiguousarray(np.asarray(ranks, dtype=np.uint64))
    out = np.zeros((r.shape[0], n), dtype=np.complex128)
    _check(lib().perm_c128_seed(ptr, n, r.ctypes.data_as(ctypes.c_void_p), r.shape[0],
                                out.ctypes.data_as(ctypes.c_void_p), _stream_ptr(None)))
    del keep
    return out


def perm_fp64_probe(blocks: int, threads: int, iters: int, sink, stream=None):
    """Enqueue the FP64 peak probe: blocks*threads*iters*32 DFMA (64 flops per thread-iteration)."""
    _check(lib().perm_fp64_probe(blocks, threads, iters, ctypes.c_void_p(sink.data_ptr()), _stream_ptr(stream)))


__all__ = ["perm_c128", "perm_c128_range", "perm_c128_finalize", "perm_c128_chunks", "perm_c128_tree",
           "perm_c128_tree_combine", "chunk_log2", "chunk_walkers", "tree_workspace_bytes", "tree_nodes", "make_tree_nodes", "perm_c128_batched", "perm_c128_batched_x", "perm_c128_weighted_batched",
           "perm_int01", "perm_pm1", "perm_int01_range", "perm_int01_finalize", "perm_c128_sparse", "perm_sparse_plan",
           "perm_c128_band_batched", "band_storage",
           "perm_c128_seed", "perm_fp64_probe", "workspace_bytes", "make_workspace", "int01_workspace_bytes",
           "PermError", "DD", "lib", "header_functions", "last_launches"]
