# ncu evidence for the bench command (one GPU). Plain run first, then ncu.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?"
$CMD > gpurun_out/prof_plain2.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:walk -s 1 -c 1 -o gpurun_out/prof_walk $CMD > gpurun_out/ncu_full.log 2>&1
echo "full exit $?"
