mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu17.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu17.log
timeout 900 python scripts/c5_run.py > gpurun_out/c5_summary.json 2> gpurun_out/c5.err; echo "c5 exit $?"
cp profiles/r01_c5_checkpoints.csv gpurun_out/c5_checkpoints.csv
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench exit $?"
