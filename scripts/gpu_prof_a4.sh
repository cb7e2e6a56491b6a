mkdir -p gpurun_out
export EIS_ALPHA_X16=64
CMD="python scripts/prof_bsgs.py bsgs 99990000000 100000000000"
$CMD > gpurun_out/pa4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/pa4.csv $CMD > gpurun_out/ncu_pa4.log 2>&1
echo "exit $?"; cat gpurun_out/pa4.log
