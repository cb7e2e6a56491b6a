mkdir -p gpurun_out
CMD="python scripts/prof_bsgs.py bsgs 9900000000 10000000000"
$CMD > gpurun_out/pb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bsgs -s 2 -c 2 -o gpurun_out/prof_bsgs2 $CMD > gpurun_out/ncu_bsgs.log 2>&1
echo "exit $?"; cat gpurun_out/pb_plain.log; tail -3 gpurun_out/ncu_bsgs.log
