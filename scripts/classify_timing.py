import time, os, sys
sys.path.insert(0, os.getcwd())
import paper_2507_06579_b200 as eis
eis.init(0)
eis.set_option("mode", eis.MODE_BSGS)
for rep in range(3):
    t = time.perf_counter(); f = eis.classify_range(9 * 10**9, 10**10); w = time.perf_counter() - t
    st = eis.get_stats()
    print("classify", round(w, 3), "s wall", round(st["total_ms"], 1), "ms dev", round(st["walk_ms"], 1), "walk", st["kernel_launches"], "launches", flush=True)
for rep in range(2):
    t = time.perf_counter(); eis.count_window(9 * 10**9, [10**10]); w = time.perf_counter() - t
    st = eis.get_stats()
    print("count", round(w, 3), "s wall", round(st["total_ms"], 1), "ms dev", round(st["walk_ms"], 1), "walk", st["kernel_launches"], "launches", flush=True)
