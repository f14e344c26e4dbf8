"""Development tool: summarise an ncu --page source --csv (SASS) dump: stall samples by opcode class
and by stall reason, plus the hottest instructions.   usage: ncu_src.py src.csv [top]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
byop = collections.Counter()
byop_reason = collections.defaultdict(collections.Counter)
execd = collections.Counter()
insts = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
    base = op.split(".")[0]
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    n = int(r[ix["Instructions Executed"]] or 0)
    execd[base] += n
    byop[base] += s
    for c in stall_cols:
        v = int(r[ix[c]] or 0)
        tot[c] += v
        byop_reason[base][c] += v
    insts.append((s, r[ix["Address"]][-5:], src, n))
S = sum(tot.values())
print("total samples", S)
for c, v in tot.most_common():
    if v:
        print(f"  {c:28s} {v / S:6.3f}")
print("by opcode (samples share, executed warp-instrs):")
for op, v in byop.most_common(14):
    top = ", ".join(f"{k[6:]}={w / max(v, 1):.2f}" for k, w in byop_reason[op].most_common(4) if w)
    print(f"  {op:10s} {v / S:6.3f}  exec={execd[op]:.3e}  [{top}]")
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for s, a, src, n in sorted(insts, reverse=True)[:k]:
    print(f"  {s:8d} {a} {src}")
