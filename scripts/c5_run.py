"""BASELINE config C5 on ONE B200: pi_D, pi_E at every 1e7 up to 1e11.

Checks every Table 1 total as checkpoint differences,
pi_D against the Moebius closed form, and fits eq. (1):
pi_E(x) ~ x/(3 pi^2) + c x^(5/6), the paper reports c ~ -0.024.
Writes profiles/r01_c5_checkpoints.csv and prints a JSON summary."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2507_06579_b200 as eis
from pins import paper_windows, pi_D_closed_form

eis.init(0)
top = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**11
stride = 10**7
x = np.arange(stride, top + 1, stride, dtype=np.uint64)
t0 = time.time()
pD, pE = eis.count(x)
wall = time.time() - t0
st = eis.get_stats()
out = os.path.join(ROOT, "profiles", "r01_c5_checkpoints.csv")
with open(out, "w") as f:
    f.write("x,pi_D,pi_E\n")
    for a, b, c in zip(x, pD, pE):
        f.write(f"{int(a)},{int(b)},{int(c)}\n")
idx = {int(v): i for i, v in enumerate(x)}
def at(arr, v):
    return 0 if v == 0 else int(arr[idx[v]])
table1 = []
for lo, hi, want in paper_windows():
    if hi <= top:
        got = at(pE, hi) - at(pE, lo)
        table1.append({"window": [lo, hi], "E": got, "paper": want, "ok": got == want})
moeb = {str(v): (at(pD, v), pi_D_closed_form(v)) for v in [10**8, 10**9, 10**10, top] if v <= top}
# least-squares fit of pi_E(x) - x/(3 pi^2) = c x^(5/6) on x >= 1e8
xs = x.astype(np.float64)
m = xs >= 1e8
r = pE.astype(np.float64)[m] - xs[m] / (3 * np.pi**2)
b = xs[m] ** (5 / 6)
c = float((b @ r) / (b @ b))
print(json.dumps({"top": top, "checkpoints": len(x), "wall_s": round(wall, 2),
                  "device_ms": round(st["total_ms"], 1), "d_classified": st["d_classified"],
                  "rate_d_per_s": st["d_classified"] / (st["total_ms"] / 1e3),
                  "baby_steps": st["baby_steps"], "giant_steps": st["giant_steps"],
                  "pi_D": at(pD, top), "pi_E": at(pE, top), "table1": table1,
                  "moebius_pi_D": moeb, "fit_c_5_6": c, "paper_c": -0.024,
                  "mode": eis.get_option("mode")}, indent=1))
