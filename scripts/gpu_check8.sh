mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu8.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu8.log
python scripts/opt_sweep.py mode=2 alpha_x16=16,24,32,48,64
LO=99900000000 HI=100000000000 python scripts/opt_sweep.py mode=1,2 alpha_x16=16,32,48,64
