# time library variants in build_variants/ on the metric windows
for lib in build_variants/*.so; do
  echo "== $lib"
  EIS_LIB=$lib timeout 120 python scripts/opt_sweep.py mode=2 alpha_x16=24,28
  EIS_LIB=$lib LO=99900000000 HI=100000000000 timeout 120 python scripts/opt_sweep.py mode=2 alpha_x16=24
done
