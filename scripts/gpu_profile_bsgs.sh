mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 600 $B > gpurun_out/pb_bench.json 2> gpurun_out/pb_bench.err; echo "bench exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bsgs.csv $B > /dev/null 2> gpurun_out/ncu_launch.err; echo "ncu launches exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"bsgs_(giant|window|prep)" -s 30 -c 3 -o gpurun_out/prof_bench_bsgs $B > /dev/null 2> gpurun_out/ncu_full.err; echo "ncu full exit $?"
tail -2 gpurun_out/ncu_full.err
