"""Build libperm.so (the C-ABI library of include/perm.h) for sm_100a with nvcc.

    python -m paper_1904_06229_b200.build [-j JOBS] [--force]

Objects go to paper_1904_06229_b200/build/, the library to paper_1904_06229_b200/libperm.so (in-tree,
so it travels with the repo snapshot to the GPU box).  No fast-math: IEEE binary64 round-to-nearest
everywhere (R9); FMA contraction is allowed (products only).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# Development variants: PERM_VARIANT=<name> PERM_EXTRA_FLAGS="-DPERM_WALK_U=2 ..." builds
# build_<name>/ and libperm_<name>.so (loaded when PERM_LIB points at it); the default build has neither.
_VARIANT = os.environ.get("PERM_VARIANT", "")
BUILD = os.path.join(PKG, "build" + (f"_{_VARIANT}" if _VARIANT else ""))
LIB = os.path.join(PKG, "libperm" + (f"_{_VARIANT}" if _VARIANT else "") + ".so")
EXTRA = os.environ.get("PERM_EXTRA_FLAGS", "").split() if _VARIANT else []
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
                f"-I{CSRC}", f"-I{os.path.join(ROOT, 'include')}", "-Xptxas", "-v"]

HEADERS = ["common.cuh", "internal.h", "walk.cuh", "sparse.cuh"]


def units():
    u = [("abi.o", "abi.cu", []), ("reduce.o", "reduce.cu", []), ("tree.o", "tree.cu", []), ("batched.o", "batched.cu", []),
         ("int01.o", "int01.cu", []), ("walk_dispatch.o", "walk_dispatch.cu", []),
         ("weighted.o", "weighted.cu", []), ("band.o", "band.cu", [])]
    for p in range(8):
        u.append((f"walk_inst_{p}.o", "walk_inst.cu", [f"-DPERM_PART={p}"]))
    for p in range(6):
        u.append((f"sparse_inst_{p}.o", "sparse_inst.cu", [f"-DPERM_PART={p}"]))
    return u


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "perm.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(obj, src, extra):
    objp = os.path.join(BUILD, obj)
    srcp = os.path.join(CSRC, src)
    cmd = [NVCC, *FLAGS, *EXTRA, *extra, "-c", srcp, "-o", objp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(objp + ".log", "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src} {extra}:\n{r.stderr[-4000:]}")
    return objp


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    todo = [(o, s, e) for (o, s, e) in units() if force or _stale(os.path.join(BUILD, o), os.path.join(CSRC, s))]
    jobs = jobs or min(len(todo) or 1, os.cpu_count() or 4)
    if todo:
        with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
            futs = [ex.submit(_compile, o, s, e) for (o, s, e) in todo]
            for f in futs:
                p = f.result()
                if verbose:
                    print("built", p, flush=True)
    objs = [os.path.join(BUILD, o) for (o, _, _) in units()]
    if force or todo or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", "--jobs", type=int, default=None)
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, jobs=a.jobs, verbose=True))
    sys.exit(0)
