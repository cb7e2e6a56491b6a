mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu7.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_gpu7.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo "bench exit $?"
python -c "
import json; r=json.load(open('gpurun_out/bench7.json')); print(r['value']/1e6, r['ms_per_step'], r['config']['verified'], r['roofline']['frac'], r['clocks'])"
bash scripts/crossover.sh
