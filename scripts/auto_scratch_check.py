"""Per-call host wall and device time of count_window for fixed ranges under two
bsgs_gb settings (scratch reservation behaviour when ranges alternate)."""
import time, os, sys
sys.path.insert(0, os.getcwd())
import paper_2507_06579_b200 as eis
eis.init(0)
for gb in (48, 64):
    eis.set_option("bsgs_gb", gb)
    for lo, hi in [(9875000000, 10**10)] * 3 + [(9 * 10**9, 10**10)] + [(9875000000, 10**10)] * 2 + [(99875000000, 10**11)] * 2:
        t = time.perf_counter(); eis.count_window(lo, [hi]); w = time.perf_counter() - t
        st = eis.get_stats()
        print(gb, lo, round(w * 1e3, 1), "ms wall", round(st["total_ms"], 1), "dev", round(st["walk_ms"], 1), "walk", st["kernel_launches"], "launches", flush=True)
