# per-unit counts of the walk kernels (scripts/unit_counts.py) + pipe peaks
mkdir -p gpurun_out
python scripts/unit_counts.py run > gpurun_out/unit_run.log 2>&1 && echo "plain ok" && \
timeout 900 ncu --metrics $(python scripts/unit_counts.py metrics) --clock-control none --csv --log-file gpurun_out/unit_ncu.csv python scripts/unit_counts.py run > /dev/null 2> gpurun_out/unit_ncu.err; echo "ncu exit $?"
