"""Merge a pipe_peaks run (gpurun_out/pipe_peaks.json), the ncu pipe counters
of its kernels (gpurun_out/pipe_map.csv: which pipe each op issues to) and the
clocks sampled during it (gpurun_out/pipe_clocks.csv) into
profiles/r02_pipe_peaks.json, the per-pipe denominators bench.py uses."""
import collections
import csv
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
KERNEL_OF = {"IADD3": "k_iadd3", "LOP3": "k_lop3", "SHF": "k_shf", "IMAD": "k_imad",
             "FFMA": "k_ffma", "FADD": "k_fadd", "DFMA": "k_dfma", "MUFU.RCP": "k_rcp",
             "MUFU.LG2": "k_lg2", "I2FP+F2I": "k_cvt", "I2F.F64+F2I.F64": "k_cvt64",
             "F2F.F32.F64+F2F.F64.F32": "k_f2f", "IADD3+FFMA": "k_mix"}


def main() -> None:
    out = json.load(open(os.path.join(G, "pipe_peaks.json")))
    rows = [r for r in csv.reader(open(os.path.join(G, "pipe_map.csv"))) if len(r) > 10]
    h = rows[0]
    k, m, v = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(dict)
    for r in rows[1:]:
        agg[r[k].split("(")[0]][r[m]] = float(r[v].replace(",", ""))
    for op, kern in KERNEL_OF.items():
        d = agg.get(kern)
        if not d or op not in out["ops"]:
            continue
        tot = d.get("smsp__inst_executed.sum", 0) or 1
        out["ops"][op]["ncu_pipes"] = {
            key.replace("sm__inst_executed_pipe_", "").replace(".sum", ""): round(val / tot, 3)
            for key, val in d.items() if key != "smsp__inst_executed.sum" and val / tot > 0.01}
    sm = []
    for ln in open(os.path.join(G, "pipe_clocks.csv")):
        p = ln.strip().split(",")
        try:
            sm.append(float(p[0].split()[0]))
        except (ValueError, IndexError):
            pass
    out["nvidia_smi_sm_mhz_median"] = statistics.median(sm) if sm else None
    out["source"] = ("bench_tools/pipe_peaks.cu under scripts/gpu_pipe_peaks.sh on one B200; "
                     "ncu_pipes = share of the kernel's warp-instructions per ncu pipe counter")
    dst = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02_pipe_peaks.json")
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps({op: (e["warp_inst_per_clk_per_sm"], e.get("ncu_pipes")) for op, e in
                      out["ops"].items()}, indent=0))


if __name__ == "__main__":
    main()
