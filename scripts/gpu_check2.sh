mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest exit $?"
tail -30 gpurun_out/pytest_gpu2.log
timeout 600 python scripts/mode_sweep.py 1000000 8,16,32 > gpurun_out/sweep2.log 2>&1; echo "sweep exit $?"
cat gpurun_out/sweep2.log
for m in half bsgs; do timeout 300 python bench.py --steps 10 --warmup 3 --mode $m --no-cpu-baseline > gpurun_out/bench2_$m.json 2> gpurun_out/bench2_$m.err; echo "bench $m exit $?"; cut -c1-400 gpurun_out/bench2_$m.json; tail -3 gpurun_out/bench2_$m.err; done
