import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_06579_b200 as eis
eis.init(0)
eis.set_option("mode", eis.MODE_BSGS)
lo, hi = 9_900_000_000, 10_000_000_000
for mb in [int(v) for v in sys.argv[1].split(",")]:
    eis.set_option("baby_l2_mb", mb)
    eis.count_window(lo, [hi])
    cD, cE = eis.count_window(lo, [hi])
    st = eis.get_stats()
    print(json.dumps({"baby_l2_mb": mb, "E": int(cE[0]), "ms": round(st["total_ms"], 2),
                      "rate_M": round(st["d_classified"] / st["total_ms"] / 1e3, 1)}), flush=True)
