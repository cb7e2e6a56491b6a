mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_final.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_final.log
timeout 900 python scripts/c5_run.py > gpurun_out/c5_summary.json 2> gpurun_out/c5.err; echo "c5 exit $?"
cp profiles/r01_c5_checkpoints.csv gpurun_out/c5_checkpoints.csv
timeout 600 python scripts/cross_mode.py > gpurun_out/cross.log 2>&1; echo "cross exit $?"; cat gpurun_out/cross.log; cp profiles/r01_cross_mode.json gpurun_out/
bash scripts/gpu_multirank.sh > gpurun_out/mr.log 2>&1; grep -o "multirank exit [0-9]*" gpurun_out/mr.log; grep -o '"verified[^}]*' gpurun_out/mr2.json
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
