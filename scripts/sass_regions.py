"""Per-region dynamic profile of one kernel from an ncu report (source page),
with inline call sites resolved (nvdisasm -gi), so that a helper such as
dfloor_mod is charged to the place that calls it.

    python scripts/sass_regions.py REPORT.ncu-rep KERNEL_REGEX LIB.so [TOP]

For each source site (the call site of an inlined helper, else the line) it
prints the share of warp instructions, threads per instruction, the share of
wasted lane-slots (warp instructions x (32 - threads)) and of stall samples.
"""
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def site_table(lib: str, kernel: str) -> dict[int, str]:
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True,
                   stdout=subprocess.DEVNULL)
    cubin = glob.glob(os.path.join(tmp, "*.cubin"))[0]
    txt = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
    out, inside, cur = {}, False, "?"
    for ln in txt.splitlines():
        if ln.startswith("//---") and ".text." in ln:
            inside = re.search(kernel, ln) is not None
            continue
        if not inside:
            continue
        m = re.match(r'\s*//## File "(.*?)", line (\d+)(?: inlined at "(.*?)", line (\d+))?', ln)
        if m:
            if m.group(3):
                cur = f"{os.path.basename(m.group(1))}:{m.group(2)} @{os.path.basename(m.group(3))}:{m.group(4)}"
            else:
                cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            out[int(m.group(1), 16)] = cur
    return out


def main() -> None:
    rep, kern, lib = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 50
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kern}", "-c", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    h = rows[hi]
    ia, ie = h.index("Address"), h.index("Instructions Executed")
    it, iss = h.index("Thread Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[hi + 1:] if len(r) == len(h) and r[ia].startswith("0x")]
    base = int(body[0][ia], 16)
    sites = site_table(lib, kern)
    agg = defaultdict(lambda: [0, 0, 0])
    for r in body:
        key = sites.get(int(r[ia], 16) - base, "?")
        a = agg[key]
        a[0] += int(r[ie] or 0)
        a[1] += int(r[it] or 0)
        a[2] += int(r[iss] or 0)
    te = sum(a[0] for a in agg.values()) or 1
    tt = sum(a[1] for a in agg.values())
    ts = sum(a[2] for a in agg.values()) or 1
    tw = sum(32 * a[0] - a[1] for a in agg.values()) or 1
    print(f"{kern}: {te:.4g} warp instructions, {tt / te:.2f} threads/inst, {ts} stall samples")
    print(f"{'site (line @ caller)':44s} {'inst%':>6s} {'thr':>5s} {'waste%':>7s} {'stall%':>7s}")
    for k, a in sorted(agg.items(), key=lambda kv: -(32 * kv[1][0] - kv[1][1]))[:top]:
        print(f"{k:44s} {100 * a[0] / te:6.2f} {a[1] / max(a[0], 1):5.1f} "
              f"{100 * (32 * a[0] - a[1]) / tw:7.2f} {100 * a[2] / ts:7.2f}")


if __name__ == "__main__":
    main()
