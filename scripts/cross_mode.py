"""HALF vs BSGS on full windows: every per-d flag compared (two independent
algorithms for t; the oracle is too slow for 1e8 d).  Prints a JSON summary."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_06579_b200 as eis

eis.init(0)
out = []
for lo, hi in [(9 * 10**9, 10**10), (10**11 - 10**9, 10**11)]:
    res = {}
    flags = {}
    for name, mode in (("half", eis.MODE_HALF), ("bsgs", eis.MODE_BSGS)):
        eis.set_option("mode", mode)
        t0 = time.time()
        flags[name] = eis.classify_range(lo, hi)
        res[name + "_s"] = round(time.time() - t0, 2)
    f = flags["half"]
    inD = f != eis.NOT_IN_D
    res.update({"window": [lo, hi], "candidates": int(f.size), "d_in_D": int(inD.sum()),
                "E": int((f == 0).sum()), "t1": int((f == 1).sum()), "t2": int((f == 2).sum()),
                "mismatches": int((flags["half"] != flags["bsgs"]).sum())})
    out.append(res)
    print(json.dumps(res), flush=True)
eis.set_option("mode", eis.MODE_AUTO)
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                 "profiles", os.environ.get("EIS_TAG", "r02") + "_cross_mode.json"), "w"), indent=1)
