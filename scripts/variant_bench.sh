# A/B of builds: opt_sweep.py on the bench slab for every build_variants/*.so
# (EIS_LIB selects the library), two passes, then the rates per build.
# Extra opt_sweep arguments may be passed (default: mode=2 alpha_x16=0,0).
args=${*:-"mode=2 alpha_x16=0,0"}
log=${VLOG:-gpurun_out/variants.log}
: > $log
for pass in 1 2; do
  for lib in build_variants/*.so; do
    echo "== $lib" >> $log
    EIS_LIB=$lib LO=${LO:-9875000000} HI=${HI:-10000000000} timeout 120 python scripts/opt_sweep.py $args >> $log 2>&1
  done
done
python - "$log" <<'PY'
import collections, json, sys
cur, r = None, collections.defaultdict(list)
for l in open(sys.argv[1]):
    if l.startswith("=="):
        cur = l.split()[-1]
    elif l.startswith("{"):
        j = json.loads(l)
        r[cur].append((j["rate_M"], j.get("E")))
for k, v in r.items():
    print(k, [x[0] for x in v], sorted({x[1] for x in v}))
PY
