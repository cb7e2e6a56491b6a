"""BASELINE config C2: every d <= 1e8, per-d flags GPU vs the CPU oracle (all host cores)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2507_06579_b200 as eis
from oracle import c_oracle
eis.init(0)
res = {}
for mode, name in [(eis.MODE_HALF, "half"), (eis.MODE_BSGS, "bsgs")]:
    eis.set_option("mode", mode)
    t0 = time.time()
    res[name] = eis.classify_range(0, 10**8)
    res[name + "_s"] = time.time() - t0
t0 = time.time()
want = c_oracle.classify_range(0, 10**8)
ot = time.time() - t0
out = {"candidates": int(want.size), "D": int((want != 255).sum()), "E": int((want == 0).sum()),
       "oracle_s": round(ot, 1), "cores": os.cpu_count()}
for name in ("half", "bsgs"):
    bad = np.flatnonzero(res[name] != want)
    out[name] = {"mismatches": int(bad.size), "first_bad": [int(5 + 8 * i) for i in bad[:5]],
                 "gpu_s": round(res[name + "_s"], 3)}
print(json.dumps(out))
