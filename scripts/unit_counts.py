"""Per-unit instruction and byte counts of the walk kernels, measured (run on a
GPU box; writes gpurun_out/):

    python scripts/unit_counts.py run  [LO HI]   # one count_window call: stats JSON
    ncu --metrics <METRICS> --csv --log-file gpurun_out/unit_ncu.csv python scripts/unit_counts.py run
    python scripts/unit_counts.py combine        # (here) -> profiles/r02_unit_counts.json

The range defaults to (9.95e9, 1e10]: one BSGS segment at the bench's scale
(d ~ 1e10), so every kernel launches once.  Per unit: thread- and
warp-instructions (all and per pipe) and DRAM bytes per d, per baby step
(window kernel) and per giant step (giant kernel).  bench.py reads the
committed JSON for its roofline numerators.
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
METRICS = ("smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__inst_executed_pipe_alu.sum,"
           "sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,"
           "sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_xu.sum,"
           "sm__inst_executed_pipe_lsu.sum,sm__inst_executed_pipe_uniform.sum,"
           "sm__inst_executed_pipe_cbu.sum,sm__inst_executed_pipe_adu.sum,dram__bytes_read.sum,"
           "dram__bytes_write.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,"
           "smsp__thread_inst_executed_per_inst_executed.ratio,sm__cycles_elapsed.avg.per_second")


def run() -> None:
    import paper_2507_06579_b200 as eis

    lo = int(float(sys.argv[2])) if len(sys.argv) > 3 else 9_950_000_000
    hi = int(float(sys.argv[3])) if len(sys.argv) > 3 else 10_000_000_000
    eis.init(0)
    D, E = eis.count_window(lo, [hi])
    st = eis.get_stats()
    # the HALF walk's per-step count, on (9.9e8, 1e9] (AUTO's HALF region)
    eis.set_option("mode", eis.MODE_HALF)
    eis.count_window(990_000_000, [1_000_000_000])
    sh = eis.get_stats()
    eis.set_option("mode", eis.MODE_AUTO)
    out = {"lo": lo, "hi": hi, "D": int(D[0]), "E": int(E[0]), **st,
           "half": {"lo": 990_000_000, "hi": 1_000_000_000, "d": sh["d_classified"],
                    "baby_steps": sh["baby_steps"]}}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "unit_stats.json"), "w") as f:
        json.dump(out, f)
    print(json.dumps(out))


def combine(csv_path: str, stats_path: str, out_path: str) -> None:
    st = json.load(open(stats_path))
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    h = rows[0]
    k, m, v = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    kern = collections.defaultdict(lambda: collections.defaultdict(float))
    launches = collections.Counter()
    seen = set()
    second_call, prefix_id = False, None
    for r in rows[1:]:
        name = r[k].split("(")[0].split("::")[-1].replace("<unnamed>", "").strip()
        name = name[5:] if name.startswith("void ") else name
        if prefix_id is not None and r[h.index("ID")] != prefix_id:
            second_call = True                 # past the first call's prefix kernel
        if name.startswith("bsgs_"):                         # (templates on the list layout)
            name = name.split("<")[0]
        elif name.startswith("walk_half_kernel"):
            name = "walk_half_kernel"
        elif second_call:                      # kernels of the HALF call
            name += " (HALF call)"
        elif name.startswith("prefix_kernel"):
            prefix_id = r[h.index("ID")]
        kern[name][r[m]] += float(r[v].replace(",", ""))
        if (r[h.index("ID")], name) not in seen:
            seen.add((r[h.index("ID")], name))
            launches[name] += 1
    nd = st["d_classified"]
    out = {"source": "ncu --metrics (counters summed over the call's launches) of one "
                     f"count_window({st['lo']}, [{st['hi']}]) call; stats from eis_get_stats",
           "d": nd, "baby_steps": st["baby_steps"], "giant_steps": st["giant_steps"],
           "reduce_steps": st["reduce_steps"], "half_call": st.get("half"), "kernels": {}}
    pipes = ("alu", "fma", "fmaheavy", "fp64", "xu", "lsu", "uniform", "cbu", "adu")
    for name, d in kern.items():
        w = d["smsp__inst_executed.sum"]
        e = {"launches": launches[name],
             "warp_inst": w, "thread_inst": d["smsp__thread_inst_executed.sum"],
             "threads_per_inst": d["smsp__thread_inst_executed.sum"] / w if w else None,
             "warp_inst_per_d": w / nd, "thread_inst_per_d": d["smsp__thread_inst_executed.sum"] / nd,
             "pipe_warp_inst_per_d": {p: d[f"sm__inst_executed_pipe_{p}.sum"] / nd for p in pipes},
             "dram_bytes_per_d": (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / nd,
             "dram_read_per_d": d["dram__bytes_read.sum"] / nd,
             "dram_write_per_d": d["dram__bytes_write.sum"] / nd,
             "ncu_ms": d["gpu__time_duration.sum"] / 1e6}
        if name == "bsgs_window_kernel":
            e["thread_inst_per_baby_step"] = e["thread_inst"] / st["baby_steps"]
        if name == "bsgs_giant_kernel":
            e["thread_inst_per_giant_step"] = e["thread_inst"] / st["giant_steps"]
        if name.startswith("walk_half_kernel") and st.get("half"):
            e["thread_inst_per_baby_step"] = e["thread_inst"] / st["half"]["baby_steps"]
            for key in ("warp_inst_per_d", "thread_inst_per_d", "dram_bytes_per_d",
                        "dram_read_per_d", "dram_write_per_d"):
                e[key] = e[key] * nd / st["half"]["d"]
            e["pipe_warp_inst_per_d"] = {p: v * nd / st["half"]["d"]
                                         for p, v in e["pipe_warp_inst_per_d"].items()}
            e["per_d_basis"] = "d of the HALF call"
        out["kernels"][name] = e
    json.dump(out, open(out_path, "w"), indent=1)
    print(json.dumps({n: {kk: e[kk] for kk in ("warp_inst_per_d", "thread_inst_per_d",
                                                 "threads_per_inst", "dram_bytes_per_d")}
                      for n, e in out["kernels"].items()}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    elif sys.argv[1] == "metrics":
        print(METRICS)
    else:
        combine(os.path.join(ROOT, "gpurun_out", "unit_ncu.csv"),
                os.path.join(ROOT, "gpurun_out", "unit_stats.json"),
                sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles",
                                                                   "r02_unit_counts.json"))
