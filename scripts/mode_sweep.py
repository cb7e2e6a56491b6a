"""Time HALF vs BSGS on windows of width W below each scale (device time from
the library's CUDA events), with step statistics.  Used to set the AUTO crossover."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_06579_b200 as eis

eis.init(0)
width = int(sys.argv[1]) if len(sys.argv) > 1 else 10**7
scales = [10**7, 10**8, 10**9, 10**10, 10**11]
alphas = [int(a) for a in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["16"])]
for sc in scales:
    lo = sc - width * (8 if sc >= 10**10 else 1)
    res = {}
    for mode, name in [(eis.MODE_HALF, "half"), (eis.MODE_BSGS, "bsgs")]:
        for a in (alphas if mode == eis.MODE_BSGS else [16]):
            eis.set_option("mode", mode)
            eis.set_option("alpha_x16", a)
            eis.count_window(lo, [sc])          # warm
            cD, cE = eis.count_window(lo, [sc])
            st = eis.get_stats()
            key = name if mode == eis.MODE_HALF else f"bsgs_a{a}"
            res[key] = dict(E=int(cE[0]), D=int(cD[0]), walk_ms=round(st["walk_ms"], 3),
                            rate=st["d_classified"] / (st["total_ms"] / 1e3),
                            baby_per_d=st["baby_steps"] / max(1, st["d_classified"]),
                            giant_per_d=st["giant_steps"] / max(1, st["d_classified"]),
                            fb=st["fallbacks"])
    Es = {v["E"] for v in res.values()}
    print(json.dumps({"scale": sc, "lo": lo, "agree": len(Es) == 1, **res}), flush=True)
eis.set_option("mode", eis.MODE_AUTO)
eis.set_option("alpha_x16", 16)
