# End-of-round checks on one GPU: pytest -m gpu, smoke(), C5 (with the Table 1
# totals and the checkpoint hash), the HALF/BSGS cross-check, the 2-rank
# orchestration run and the reference arm.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/final_smoke.log
timeout 900 python scripts/c5_run.py > gpurun_out/r02_c5_summary.json 2> gpurun_out/c5.err; echo "c5 exit $?"; cp profiles/r02_c5_checkpoints.csv gpurun_out/
timeout 600 python scripts/cross_mode.py > gpurun_out/cross.log 2>&1; echo "cross exit $?"; cp profiles/r02_cross_mode.json gpurun_out/
bash scripts/gpu_multirank.sh > gpurun_out/mr.log 2>&1; grep -o "multirank exit [0-9]*\|ref exit [0-9]*\|ref2 exit [0-9]*" gpurun_out/mr.log
