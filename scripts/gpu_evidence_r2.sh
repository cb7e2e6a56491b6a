# Round-2 evidence on one GPU (run from the repo root on a GPU box; no rebuild, so
# the shipped libeis.so is what is measured and profiled):
#  bench line (N=1, with cpu_baseline), launch list of the bench command, one
#  ncu --set full capture of the BSGS walk kernels, per-unit counts, pipe peaks
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo "bench exit $?"
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --window-calls 0"
$B > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv $B > /dev/null 2> gpurun_out/ev_ncu_launch.err; echo "ncu launches exit $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"bsgs_(giant|window|prep)" -s 3 -c 3 -o gpurun_out/ev_prof $B > /dev/null 2> gpurun_out/ev_ncu_full.err; echo "ncu full exit $?"
bash scripts/gpu_unit_counts.sh
bash scripts/gpu_pipe_peaks.sh
