"""Stall reasons of one kernel, split by the execution count of its SASS
blocks (instructions with one execution count form a region: the per-step
loop, the per-group build loop, the per-d code ...).

    python scripts/stall_regions.py REPORT.ncu-rep KERNEL_REGEX [TOP]
"""
import collections
import csv
import io
import subprocess
import sys

REASONS = ["stall_long_sb", "stall_short_sb", "stall_wait", "stall_mio", "stall_lg", "stall_math",
           "stall_not_selected", "stall_selected", "stall_branch_resolving", "stall_barrier",
           "stall_membar", "stall_drain", "stall_no_inst", "stall_dispatch", "stall_misc"]


def main() -> None:
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kern}", "-c", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    h = rows[hi]
    ia, ie, isrc = h.index("Address"), h.index("Instructions Executed"), h.index("Source")
    idx = {r: h.index(r) for r in REASONS if r in h}
    seen, body = set(), []
    for r in rows[hi + 1:]:
        if len(r) != len(h) or not r[ia].startswith("0x"):
            continue
        if r[ia] in seen:
            break
        seen.add(r[ia])
        body.append(r)
    reg = collections.defaultdict(lambda: collections.Counter())
    ninst = collections.Counter()
    ops = collections.defaultdict(collections.Counter)
    for r in body:
        e = int(r[ie] or 0)
        ninst[e] += 1
        for nm, i in idx.items():
            reg[e][nm] += int(r[i] or 0)
        op = r[isrc].split()[0] if r[isrc].split() else ""
        if op.startswith("@"):
            op = r[isrc].split()[1]
        ops[e][op.split(".")[0]] += 1
    tot = sum(sum(c.values()) for c in reg.values()) or 1
    print(f"{kern}: {tot} stall samples")
    for e, c in sorted(reg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
        s = sum(c.values())
        parts = ", ".join(f"{k[6:]} {100 * v / s:.0f}%" for k, v in c.most_common(5))
        print(f"exec={e:10d} n={ninst[e]:4d} samples {100 * s / tot:5.1f}%  [{parts}]  "
              f"ops: {' '.join(o for o, _ in ops[e].most_common(6))}")


if __name__ == "__main__":
    main()
