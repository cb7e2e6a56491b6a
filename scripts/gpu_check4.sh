mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu4.log
timeout 600 python scripts/mode_sweep.py 1000000 16,32,48 > gpurun_out/sweep4.log 2>&1; echo "sweep exit $?"
python -c "
import json
for l in open('gpurun_out/sweep4.log'):
    r=json.loads(l); print(r['scale'], r['agree'], {k:(round(v['rate']/1e6,1), round(v['walk_ms'],2)) for k,v in r.items() if isinstance(v,dict)})
"
CMD="python scripts/prof_bsgs.py bsgs 9900000000 10000000000"
$CMD > gpurun_out/pb_plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bsgs -s 2 -c 2 -o gpurun_out/prof_bsgs4 $CMD > gpurun_out/ncu_bsgs4.log 2>&1
echo "ncu exit $?"; cat gpurun_out/pb_plain4.log
