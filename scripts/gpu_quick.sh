mkdir -p gpurun_out
timeout 600 python scripts/mode_sweep.py 1000000 16,32 > gpurun_out/sweepq.log 2>&1; echo "sweep exit $?"
python -c "
import json
for l in open('gpurun_out/sweepq.log'):
    r=json.loads(l); print(r['scale'], r['agree'], {k:(round(v['rate']/1e6,1), round(v['walk_ms'],2)) for k,v in r.items() if isinstance(v,dict)})
"
CMD="python scripts/prof_bsgs.py bsgs 9900000000 10000000000"
$CMD > gpurun_out/pbq.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bsgs -s 2 -c 2 -o gpurun_out/prof_q $CMD > gpurun_out/ncu_q.log 2>&1
echo "ncu exit $?"; cat gpurun_out/pbq.log
