mkdir -p gpurun_out
timeout 120 python scripts/bsgs_stats.py; echo "stats exit $?"
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu9.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_gpu9.log
timeout 300 python scripts/opt_sweep.py mode=2 alpha_x16=16,24,32,48
LO=99900000000 HI=100000000000 timeout 300 python scripts/opt_sweep.py mode=2 alpha_x16=16,24,32,48
