"""Development tool: SASS listing with decoded control bits (stall, yield, wr/rd barrier, wait mask,
reuse) for sm_100a.   usage: sass_ctrl.py obj func [start_hex end_hex]"""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", "-fun", sys.argv[2], sys.argv[1]], capture_output=True, text=True).stdout
lines = out.splitlines()
res = []
for k, l in enumerate(lines):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/", l)
    if m and k + 1 < len(lines):
        m2 = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[k + 1])
        hi = int(m2.group(1), 16)
        ctrl = hi >> 41
        stall = ctrl & 0xF
        yld = (ctrl >> 4) & 1
        wb = (ctrl >> 5) & 7
        rb = (ctrl >> 8) & 7
        wm = (ctrl >> 11) & 0x3F
        ru = (ctrl >> 17) & 0xF
        res.append((int(m.group(1), 16), stall, yld, wb, rb, wm, ru, m.group(2).strip()))
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else 0
hi_ = int(sys.argv[4], 16) if len(sys.argv) > 4 else 1 << 40
for a, st, y, wb, rb, wm, ru, t in res:
    if lo <= a <= hi_:
        print(f"{a:05x} S{st:2d} Y{y} W{wb if wb != 7 else '-'} R{rb if rb != 7 else '-'} M{wm:02x} U{ru:x}  {t}")
