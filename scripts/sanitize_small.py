"""Small end-to-end workload for compute-sanitizer (memcheck): HALF, BSGS and AUTO
classification and counting on small ranges, the device-resident calls and
classify_range over several slices; compared with the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_06579_b200 as eis  # noqa: E402
from oracle import c_oracle  # noqa: E402

eis.init(0)
eis.set_option("segment_log2", 18)
bad = 0
for mode in (eis.MODE_HALF, eis.MODE_BSGS, eis.MODE_AUTO):
    eis.set_option("mode", mode)
    for lo, hi in [(0, 300_000), (10**9 - 40_000, 10**9 + 17), (10**11 - 30_000, 10**11)]:
        f = eis.classify_range(lo, hi)
        bad += int((f != c_oracle.classify_range(lo, hi)).sum())
        x = [lo + (hi - lo) // 2 + 1, hi]
        cD, cE = eis.count_window(lo, x)
        oD, oE = c_oracle.count_window(lo, x)
        bad += int((cD != oD).sum() + (cE != oE).sum())
print("mismatches", bad)
sys.exit(1 if bad else 0)
