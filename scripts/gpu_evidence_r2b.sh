# Round-2 evidence on one GPU, self-consistent in one call (run from the repo
# root on a GPU box; the shipped libeis.so is measured, no rebuild):
#  1) per-unit counts of the walk kernels -> profiles/r02_unit_counts.json (combined
#     on the box, so that the bench line below reads the counts of this build)
#  2) the bench line (N=1, with cpu_baseline)
#  3) the launch list of the bench command and one ncu --set full capture of the
#     BSGS walk kernels
# Outputs under gpurun_out/ (copy the profiles/ files back from gpurun_out/).
mkdir -p gpurun_out
bash scripts/gpu_unit_counts.sh
python scripts/unit_counts.py combine > gpurun_out/unit_combine.log 2>&1; echo "combine exit $?"
cp profiles/r02_unit_counts.json gpurun_out/r02_unit_counts.json
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo "bench exit $?"
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --window-calls 0"
$B > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv $B > /dev/null 2> gpurun_out/ev_ncu_launch.err; echo "ncu launches exit $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"bsgs_(giant|window|prep)" -s 3 -c 3 -o gpurun_out/ev_prof $B > /dev/null 2> gpurun_out/ev_ncu_full.err; echo "ncu full exit $?"
