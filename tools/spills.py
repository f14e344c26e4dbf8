"""List kernels with spill stores in the ptxas logs of the last build (paper_1904_06229_b200/build/*.o.log)."""
from __future__ import annotations

import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def spills(build_dir: str | None = None) -> dict[str, tuple[int, int]]:
    """{mangled kernel name: (spill store bytes, registers)} for every entry function ptxas compiled."""
    build_dir = build_dir or os.path.join(ROOT, "paper_1904_06229_b200", "build")
    out: dict[str, tuple[int, int]] = {}
    for log in sorted(glob.glob(os.path.join(build_dir, "*.o.log"))):
        fn, sp = None, 0
        for line in open(log):
            m = re.search(r"Compiling entry function '(\S+)'", line)
            if m:
                fn, sp = m.group(1), 0
                continue
            m = re.search(r"(\d+) bytes spill stores", line)
            if m and fn:
                sp = int(m.group(1))
            m = re.search(r"Used (\d+) registers", line)
            if m and fn:
                out[fn] = (sp, int(m.group(1)))
                fn = None
    return out


if __name__ == "__main__":
    d = spills(sys.argv[1] if len(sys.argv) > 1 else None)
    names = [k for k, (s, _) in d.items() if s > 0]
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    for k, nm in zip(names, dem):
        print(f"{d[k][0]:5d} B  {d[k][1]:3d} regs  {nm}")
