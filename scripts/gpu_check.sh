set -x
mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|^CPU\(s\)"; nvidia-smi -L; free -g | head -2
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench exit $?"
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
