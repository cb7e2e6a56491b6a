"""Sweep library options on the (9.9e9, 1e10] window: opt_sweep.py key=v1,v2 [key2=...]"""
import sys, os, json, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_06579_b200 as eis
eis.init(0)
lo = int(float(os.environ.get("LO", "9.9e9"))); hi = int(float(os.environ.get("HI", "1e10")))
keys, vals = [], []
for a in sys.argv[1:]:
    k, v = a.split("=")
    keys.append(k); vals.append([int(x) for x in v.split(",")])
for combo in itertools.product(*vals):
    for k, v in zip(keys, combo):
        eis.set_option(k, v)
    eis.count_window(lo, [hi])
    cD, cE = eis.count_window(lo, [hi])
    st = eis.get_stats()
    print(json.dumps({**dict(zip(keys, combo)), "E": int(cE[0]), "ms": round(st["total_ms"], 2),
                      "rate_M": round(st["d_classified"] / st["total_ms"] / 1e3, 1),
                      "win": round(st.get("window_ms", 0), 2), "giant": round(st.get("giant_ms", 0), 2),
                      "giant_per_d": round(st["giant_steps"] / max(st["d_classified"], 1), 2),
                      "baby_per_d": round(st["baby_steps"] / max(st["d_classified"], 1), 1),
                      "nw": st.get("window_nw"), "nb": st.get("window_nb"),
                      "fallbacks": st["fallbacks"]}),
          flush=True)
