mkdir -p gpurun_out
export EIS_ALPHA_X16=64
CMD="python scripts/prof_bsgs.py bsgs 99990000000 100000000000"
$CMD > gpurun_out/pb.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:build -s 0 -c 1 -o gpurun_out/prof_build $CMD > gpurun_out/ncu_b.log 2>&1
echo "exit $?"
