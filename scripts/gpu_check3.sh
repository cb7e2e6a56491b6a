mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest exit $?"
tail -15 gpurun_out/pytest_gpu3.log
timeout 600 python scripts/mode_sweep.py 1000000 8,16,32 > gpurun_out/sweep3.log 2>&1; echo "sweep exit $?"
cat gpurun_out/sweep3.log | cut -c1-600
