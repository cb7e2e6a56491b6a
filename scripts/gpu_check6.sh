mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_gpu6.log
python scripts/l2_sweep.py 40,64,72,80
for m in half bsgs; do timeout 300 python bench.py --steps 10 --warmup 3 --mode $m --no-cpu-baseline > gpurun_out/bench6_$m.json 2> gpurun_out/bench6_$m.err; echo "bench $m exit $?"; python -c "
import json; r=json.load(open('gpurun_out/bench6_$m.json')); print(r['value']/1e6, r['ms_per_step'], r['config']['verified'], r['roofline']['frac'], r['clocks'])"; done
