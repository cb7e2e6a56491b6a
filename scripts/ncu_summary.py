"""Summarise an ncu report (--set full) and a launch-list CSV into a text file for profiles/."""
import csv, subprocess, sys, io, collections
rep, launches, out, title = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "smsp__thread_inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "sm__cycles_elapsed.avg.per_second"]
lines = [f"# {title}", f"# source: {rep} (ncu --set full --clock-control none), {launches}", ""]
for r in rows[2:]:
    for n in want:
        if n in h:
            i = h.index(n)
            lines.append(f"{n:70s} {r[i]:>22s} {units[i]}")
    stalls = [(h[i], float(r[i])) for i in range(len(h))
              if h[i].startswith("smsp__average_warps_issue_stalled") and h[i].endswith("per_issue_active.ratio")
              and r[i] not in ("", "n/a")]
    stalls.sort(key=lambda t: -t[1])
    lines.append("top stall reasons (warps per issue-active cycle):")
    for n, v in stalls[:8]:
        lines.append(f"  {n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {v:8.3f}")
    lines.append("")
# launch list
import os
if not os.path.exists(launches):
    open(out, "w").write("\n".join(lines) + "\n"); print("\n".join(lines)); sys.exit(0)
lr = list(csv.reader(open(launches)))
hi = [i for i, r in enumerate(lr) if r and r[0] == "ID"][0]
H = lr[hi]
ki, mi = H.index("Kernel Name"), H.index("Metric Value")
tot = collections.Counter(); cnt = collections.Counter()
for r in lr[hi + 1:]:
    k = r[ki].split("(")[0][:60]
    tot[k] += float(r[mi].replace(",", "")); cnt[k] += 1
allns = sum(tot.values())
lines.append("launch list (gpu__time_duration.sum, cold-cache, serialised):")
for k, v in tot.most_common():
    lines.append(f"  {k:62s} n={cnt[k]:3d} total={v/1e6:9.3f} ms share={v/allns*100:6.2f}%")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
