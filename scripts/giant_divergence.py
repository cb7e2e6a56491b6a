"""Expected SIMT efficiency of the giant step's loops and branches from the CPU
emulation's per-step event counts (tests/emu/giant_profile.cu):

    python scripts/giant_divergence.py [LO HI N ALPHA_X16]

For each counter: the mean per lane-step, the expected maximum over 32 lanes
(what the warp executes when 32 independent steps run together) and their
ratio (lane efficiency inside that loop or branch)."""
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402

NAMES = ["xgcd iters", "F not|s", "euclid iters", "rho steps", "nucomp", "F != 1", "z == 0",
         "bx == 0", "rare path", "key match", "2nd bucket"]


def main() -> None:
    lo, hi, n, ax16 = (int(float(v)) for v in (sys.argv[1:5] if len(sys.argv) > 4
                                               else (9.99e9, 1e10, 3000, 30)))
    exe = os.path.join(tempfile.mkdtemp(), "giant_profile")
    subprocess.check_call(["nvcc", "-x", "cu", "-std=c++17", "-O2", "-gencode",
                           "arch=compute_100a,code=sm_100a", "-o", exe,
                           os.path.join(ROOT, "tests", "emu", "giant_profile.cu")])
    ds = workloads.sample_candidates(lo, hi, n, seed=7)
    out = subprocess.run([exe, str(ax16)], input="\n".join(str(int(d)) for d in ds),
                         capture_output=True, text=True, check=True).stdout
    rows = [ln.split() for ln in out.splitlines()]
    A = np.array([[int(x) for x in r[3:]] for r in rows if r[1] == "S" and r[2] != "0"])
    rng = np.random.default_rng(1)
    print(f"{len(A)} giant steps of {len(ds)} seeded d in [{lo}, {hi}], alpha_x16 {ax16}")
    print(f"{'event':12s} {'mean':>7s} {'E[max32]':>9s} {'eff':>5s} {'P(any)':>7s}")
    for i, nm in enumerate(NAMES):
        v = A[:, i]
        W = v[rng.integers(0, len(v), (20000, 32))].max(1)
        mx = W.mean()
        print(f"{nm:12s} {v.mean():7.3f} {mx:9.3f} {v.mean() / mx if mx else 0:5.2f} "
              f"{(W > 0).mean():7.3f}")


if __name__ == "__main__":
    main()
