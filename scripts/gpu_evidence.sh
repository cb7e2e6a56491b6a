mkdir -p gpurun_out profiles
nproc
timeout 900 python scripts/c5_run.py > gpurun_out/c5.json 2> gpurun_out/c5.err; echo "c5 exit $?"
cp profiles/r01_c5_checkpoints.csv gpurun_out/ 2>/dev/null
cat gpurun_out/c5.json | head -60
timeout 900 python scripts/c2_full.py > gpurun_out/c2_full.json 2> gpurun_out/c2_full.err; echo "c2 exit $?"
cat gpurun_out/c2_full.json
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo "bench exit $?"
cat gpurun_out/bench_r01.json
