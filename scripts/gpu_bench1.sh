mkdir -p gpurun_out
true
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_auto.json 2> gpurun_out/bench_auto.err; echo "bench exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --mode half --no-cpu-baseline > gpurun_out/bench_half.json 2> gpurun_out/bench_half.err; echo "bench half exit $?"
python -c "
import json
for f in ['gpurun_out/bench_auto.json','gpurun_out/bench_half.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f, round(d['value']/1e6,1), 'M d/s', d['ms_per_step'], d['roofline']['kernel'], round(d['roofline']['frac'],3), json.dumps(d['roofline']['per_kernel']), d['e2e']['value']/1e6, d['clocks'])
"
