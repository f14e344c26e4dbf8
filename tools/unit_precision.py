"""Development tool: accuracy of the walk against the oracle goldens (tests/golden/oracle_values.json, written from
oracle/ only) for the current PERM_UNIT0 setting (unit-column walk on / off): the config-4 permanent (north-star
scaled error) and the chunks44 / chunks32 spans (|gpu - oracle| / max(|oracle|, range scale))."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402
from tests import pins  # noqa: E402

g = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_values.json")))
mode = "unit" if os.environ.get("PERM_UNIT0", "1") != "0" else "plain"


def q(v):
    return complex(v[0] + v[1], v[2] + v[3])


A4 = inputs.cfg4()
ref = q(g["cfg4"]["value"])
got = pb.perm_c128(A4)
floor = 2.0 ** (-16) * float(np.prod(np.linalg.norm(A4, axis=1)))
print(f"{mode} cfg4 per {got} ref {ref} scaled_err {abs(got - ref) / max(abs(ref), floor):.3e} "
      f"rel_to_|per| {abs(got - ref) / abs(ref):.3e}", flush=True)
for key, A in (("chunks44", inputs.cfg5()), ("chunks32", A4)):
    sec = g[key]
    b = sec["chunk_log2"]
    errs = []
    for sp in sec["spans"]:
        parts = pb.perm_c128_chunks(A, sp["c0"], sp["c1"], chunk_log2_=b)
        raw, _ = pb.perm_c128_tree_combine(pb.perm_c128_tree(parts, sp["c0"], sp["c1"]).cpu().numpy())
        r = q(sp["value"])
        scale = max(abs(r), pins.range_scale(A, (sp["c1"] - sp["c0"]) << b))
        errs.append(abs(raw.value - r) / scale)
    print(f"{mode} {key} spans {len(errs)} max_err {max(errs):.3e} mean_err {np.mean(errs):.3e}", flush=True)
