"""Per-source-line dynamic profile of one kernel from an ncu report.

    python scripts/sass_lines.py REPORT.ncu-rep KERNEL_SUBSTRING [LIB.so] [TOP]

ncu's SASS source page gives per-instruction "Instructions Executed", thread
instructions and stall samples; the line table comes from `nvdisasm -g` of the
library's cubin (built with -lineinfo).  Prints the hottest lines with their
share of warp instructions, threads per instruction and share of stall samples.
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


def line_table(lib: str, kernel: str) -> dict[int, str]:
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True,
                   stdout=subprocess.DEVNULL)
    cubin = glob.glob(os.path.join(tmp, "*.cubin"))[0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    out, inside, cur = {}, False, "?"
    for ln in txt.splitlines():
        if ln.startswith("//---") and ".text." in ln:
            inside = kernel in ln
            continue
        if not inside:
            continue
        m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
        if m:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            out[int(m.group(1), 16)] = cur
    return out


def main() -> None:
    rep, kern = sys.argv[1], sys.argv[2]
    lib = sys.argv[3] if len(sys.argv) > 3 else "paper_2507_06579_b200/libeis.so"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kern}", "-c", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    h = rows[hi]
    ia, isrc = h.index("Address"), h.index("Source")
    ie, it = h.index("Instructions Executed"), h.index("Thread Instructions Executed")
    iss = h.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[hi + 1:] if len(r) == len(h) and r[ia].startswith("0x")]
    base = int(body[0][ia], 16)
    lines = line_table(lib, kern)
    agg = defaultdict(lambda: [0, 0, 0, ""])
    for r in body:
        off = int(r[ia], 16) - base
        key = lines.get(off, "?")
        a = agg[key]
        a[0] += int(r[ie] or 0)
        a[1] += int(r[it] or 0)
        a[2] += int(r[iss] or 0)
        if not a[3]:
            a[3] = r[isrc].strip()[:40]
    te = sum(a[0] for a in agg.values()) or 1
    ts = sum(a[2] for a in agg.values()) or 1
    print(f"{kern}: {te} warp instructions, {ts} stall samples, "
          f"{sum(a[1] for a in agg.values()) / te:.1f} threads/inst")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * a[0] / te:5.1f}% inst  {a[1] / max(a[0], 1):5.1f} thr  "
              f"{100 * a[2] / ts:5.1f}% stall  {k:24s} {a[3]}")


if __name__ == "__main__":
    main()
