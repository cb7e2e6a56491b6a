mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu13.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_gpu13.log
timeout 300 python scripts/opt_sweep.py mode=2 alpha_x16=16,20,24,28,32
LO=99900000000 HI=100000000000 timeout 300 python scripts/opt_sweep.py mode=2 alpha_x16=16,24,32,40
export EIS_ALPHA_X16=24
CMD="python scripts/prof_bsgs.py bsgs 9990000000 10000000000"
timeout 120 $CMD > gpurun_out/pg14.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bsgs_(giant|window|prep)" -s 0 -c 3 -o gpurun_out/prof_v6 $CMD > gpurun_out/ncu_v6.log 2>&1
echo "ncu exit $?"; cat gpurun_out/pg14.log; tail -1 gpurun_out/ncu_v6.log
