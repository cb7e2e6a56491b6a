# Per-kernel device time (ncu gpu__time_duration, launch list) of one count_window
# call on the bench slab for every build_variants/*.so:  bash scripts/variant_kernel_times.sh
# (for A/B of kernels whose variants break results, e.g. traffic experiments)
log=${VLOG:-gpurun_out/vktimes.log}
: > $log
for lib in build_variants/*.so; do
  n=$(basename $lib .so)
  EIS_LIB=$lib LO=${LO:-9875000000} HI=${HI:-10000000000} timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"${KREGEX:-bsgs}" --log-file gpurun_out/vk_$n.csv python scripts/opt_sweep.py ${ARGS:-giant_cap=0} > /dev/null 2>&1
  python - gpurun_out/vk_$n.csv $n >> $log <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; k = h.index("Kernel Name"); m = h.index("Metric Name"); v = h.index("Metric Value")
agg = collections.defaultdict(lambda: collections.defaultdict(float))
for r in rows[1:]:
    agg[r[k].split("(")[0]][r[m]] += float(r[v].replace(",", ""))
for kn, d in agg.items():
    print(sys.argv[2], kn, {m: round(x, 3) for m, x in d.items()})
PY
done
cat $log
