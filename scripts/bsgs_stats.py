import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_06579_b200 as eis
eis.init(0)
eis.set_option("mode", eis.MODE_BSGS)
for lo, hi in [(9_990_000_000, 10**10), (99_990_000_000, 10**11)]:
    for a in (16, 32, 64):
        eis.set_option("alpha_x16", a)
        eis.count_window(lo, [hi])
        st = eis.get_stats()
        nd = st["d_classified"]
        print(json.dumps({"hi": hi, "alpha_x16": a, "ms": round(st["total_ms"], 2),
                          "baby/d": round(st["baby_steps"] / nd, 1), "giant/d": round(st["giant_steps"] / nd, 1),
                          "red/g": round(st["reduce_steps"] / max(1, st["giant_steps"]), 3),
                          "fallbacks": st["fallbacks"], "sym": st["sym_exits"], "launches": st["kernel_launches"]}))
