# ncu --set full of the three BSGS kernels on one 1e7-wide window at 1e10 (default options)
mkdir -p gpurun_out
TAG=${TAG:-cur}
CMD="python scripts/prof_bsgs.py bsgs 9990000000 10000000000"
timeout 120 $CMD > gpurun_out/pg_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bsgs_(giant|window|prep)" -s 0 -c 3 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu exit $?"; cat gpurun_out/pg_$TAG.log
