mkdir -p gpurun_out
CMD="python scripts/prof_bsgs.py bsgs 9900000000 10000000000"
$CMD > gpurun_out/pb3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bsgs -s 3 -c 3 -o gpurun_out/prof_v3 $CMD > gpurun_out/ncu_v3.log 2>&1
echo "ncu exit $?"; cat gpurun_out/pb3.log
