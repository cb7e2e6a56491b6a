"""Cost model of per-class baby windows ("Per-class windows",
a design decision that was modelled and not built):

    python scripts/class_window_model.py [LO HI N]

Samples N seeded candidates of (LO, HI], computes each squarefree d's
principal-cycle distance R with bench_tools/regulator_sample.c, and compares the
mean BSGS cost per d of one window W for all d against one window per class,
with the classes cut by quantiles of a predictor of R:

    cost(d; W) = c_b W + [R/2 > D_W] (c_p + c_g max(0, R - D_W) / (2 (D_W - M)))

(D_W = 1.18 W nats: the mean rho-step distance; two-sided stride 2 (D_W - M),
M = 2 ln d + 4).  c_b, c_g, c_p are the bench slab's measured costs per window
entry, per giant step and per windowed d (profiles/r02_bench_n1.json: 15.6 ms /
5.95e9 entries, 10.4 ms / 2.14e8 giant steps, 1.1 ms / 1.18e7 d).
Predictors: the small prime factors of d (genus: 2^(omega-1) | h), the truncated
Euler product L_B (h R ~ sqrt d L(1, chi)), both, and the exact omega and R as
upper bounds.
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402

CB, CG, CP = 2.62, 48.6, 93.0          # ps per entry / giant step / windowed d


def main() -> None:
    lo, hi, n = (int(float(v)) for v in (sys.argv[1:4] if len(sys.argv) > 3
                                         else (9.9e9, 1e10, 3000)))
    exe = os.path.join(tempfile.mkdtemp(), "regulator_sample")
    subprocess.check_call(["gcc", "-O2", "-o", exe,
                           os.path.join(ROOT, "bench_tools", "regulator_sample.c"), "-lm"])
    ds = workloads.sample_candidates(lo, hi, n, seed=3)
    out = subprocess.run([exe, "100"], input="\n".join(str(int(d)) for d in ds),
                         capture_output=True, text=True, check=True).stdout
    A = np.array([[float(x) for x in ln.split()] for ln in out.splitlines()])
    d, R, om, omB, logL = A[:, 0], A[:, 1], A[:, 3], A[:, 4], A[:, 5]
    M = 2 * np.log(d.mean()) + 4
    Ws = np.arange(64, 4000, 8)

    def cost(W, Rv):
        DW = 1.18 * W
        k = np.maximum(0, (Rv - DW) / (2 * (DW - M)))
        return CB * W + np.where(Rv / 2 < DW, 0.0, CP + CG * k)

    def best(Rv):
        return min(Ws, key=lambda W: cost(W, Rv).mean())

    W0 = best(R)
    base = cost(W0, R).mean()
    print(f"{len(R)} squarefree d of {n} sampled in ({lo}, {hi}]: one window W = {W0} "
          f"entries, {base:.0f} ps per d")
    for name, f in [("omega_100", -omB), ("log L_100", logL),
                    ("log L_100 - omega_100 log 2", logL - omB * np.log(2)),
                    ("exact omega (bound)", -om),
                    ("log L_100 - omega log 2 (bound)", logL - om * np.log(2)),
                    ("exact R (bound)", R)]:
        for k in (2, 4, 8):
            qs = np.quantile(f, np.linspace(0, 1, k + 1)[1:-1])
            c = np.searchsorted(qs, f)
            tot = sum(cost(best(R[c == i]), R[c == i]).sum() for i in range(k) if (c == i).any())
            print(f"  {name:34s} {k} classes: {tot / len(R):6.0f} ps per d, "
                  f"{100 * (base * len(R) / tot - 1):+5.1f}%")


if __name__ == "__main__":
    main()
