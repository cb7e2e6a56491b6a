# Change check on one GPU: pytest -m gpu, smoke(), C5 (checkpoints + Table 1), the
# HALF/BSGS cross-check and the bench line, into gpurun_out/$TAG/
mkdir -p gpurun_out/${TAG:-chk}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG:-chk}/pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/${TAG:-chk}/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-chk}/smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/${TAG:-chk}/smoke.log
timeout 900 python scripts/c5_run.py > gpurun_out/${TAG:-chk}/c5_summary.json 2> gpurun_out/${TAG:-chk}/c5.err; echo "c5 exit $?"; cp profiles/r02_c5_checkpoints.csv gpurun_out/${TAG:-chk}/c5_checkpoints.csv
timeout 600 python scripts/cross_mode.py > gpurun_out/${TAG:-chk}/cross.log 2>&1; echo "cross exit $?"; cp profiles/r02_cross_mode.json gpurun_out/${TAG:-chk}/cross_mode.json
timeout 300 python bench.py > gpurun_out/${TAG:-chk}/bench.json 2> gpurun_out/${TAG:-chk}/bench.err; echo "bench exit $?"; cut -c1-300 gpurun_out/${TAG:-chk}/bench.json
