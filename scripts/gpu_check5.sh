mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_gpu5.log
bash scripts/gpu_quick.sh
