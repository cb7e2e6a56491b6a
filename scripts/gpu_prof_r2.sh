# ncu evidence of the bench command (run on a GPU box from the repo root):
#   TAG=... bash scripts/gpu_prof_r2.sh
# 1) the launch list (gpu__time_duration, --clock-control none) of the bench command
# 2) one --set full capture (with source) of each BSGS walk kernel, on the 3rd segment
# The in-tree libeis.so is used as shipped (no rebuild), so its line table matches.
mkdir -p gpurun_out
TAG=${TAG:-cur}
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 600 $B > gpurun_out/pb_$TAG.json 2> gpurun_out/pb_$TAG.err; echo "bench exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $B > /dev/null 2> gpurun_out/ncu_launch_$TAG.err; echo "ncu launches exit $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-bsgs_(giant|window|prep)}" -s ${SKIP:-6} -c ${COUNT:-3} -o gpurun_out/prof_$TAG $B > /dev/null 2> gpurun_out/ncu_full_$TAG.err; echo "ncu full exit $?"
tail -2 gpurun_out/ncu_full_$TAG.err
