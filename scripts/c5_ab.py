"""A/B of AUTO settings on the C5 call shape (count_window_ext at every 1e7):
c5_ab.py TOP key=v[,v...]  -> one JSON line per value."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_06579_b200 as eis
eis.init(0)
top = int(float(sys.argv[1]))
x = np.arange(10**7, top + 1, 10**7, dtype=np.uint64)
for a in sys.argv[2:]:
    k, vs = a.split("=")
    for v in vs.split(","):
        eis.set_option(k, int(float(v)))
        t0 = time.time()
        R = eis.count_window_ext(0, x)
        st = eis.get_stats()
        print(json.dumps({k: v, "top": top, "wall_s": round(time.time() - t0, 2),
                          "total_ms": round(st["total_ms"], 1), "E": int(R["E"][-1])}), flush=True)
