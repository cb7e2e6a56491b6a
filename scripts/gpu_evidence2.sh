mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench exit $?"
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bsgs.csv $B > /dev/null 2> gpurun_out/ncu_launch.err; echo "ncu launches exit $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"bsgs_(giant|window|prep)" -s 12 -c 3 -o gpurun_out/prof_bench_bsgs $B > /dev/null 2> gpurun_out/ncu_full.err; echo "ncu full exit $?"
