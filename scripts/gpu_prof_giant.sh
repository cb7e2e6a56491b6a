mkdir -p gpurun_out
export EIS_ALPHA_X16=${EIS_ALPHA_X16:-24}
for R in "99995000000 100000000000 e11" "9990000000 10000000000 e10"; do
set -- $R
CMD="python scripts/prof_bsgs.py bsgs $1 $2"
timeout 120 $CMD > gpurun_out/pg_$3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bsgs_(giant|baby|build)" -s 0 -c 3 -o gpurun_out/prof_giant_$3 $CMD > gpurun_out/ncu_g_$3.log 2>&1
echo "ncu exit $?"; cat gpurun_out/pg_$3.log; tail -1 gpurun_out/ncu_g_$3.log
done
