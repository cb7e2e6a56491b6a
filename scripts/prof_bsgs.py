import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_06579_b200 as eis
eis.init(0)
mode = sys.argv[1] if len(sys.argv) > 1 else "bsgs"
eis.set_option("mode", {"half": eis.MODE_HALF, "bsgs": eis.MODE_BSGS}[mode])
if os.environ.get("EIS_ALPHA_X16"):
    eis.set_option("alpha_x16", int(os.environ["EIS_ALPHA_X16"]))
lo = int(float(sys.argv[2])) if len(sys.argv) > 2 else 9_990_000_000
hi = int(float(sys.argv[3])) if len(sys.argv) > 3 else 10_000_000_000
for _ in range(2):
    cD, cE = eis.count_window(lo, [hi])
print(int(cD[0]), int(cE[0]), eis.get_stats())
