for lib in build_variants/*.so build_variants/*.so; do
  echo "== $lib"
  EIS_LIB=$lib LO=9875000000 HI=10000000000 timeout 120 python scripts/opt_sweep.py mode=2 alpha_x16=0,0
done
