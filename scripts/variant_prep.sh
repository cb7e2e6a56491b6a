for lib in build_variants/*.so build_variants/*.so; do
  echo "== $lib"
  EIS_LIB=$lib python scripts/prof_bsgs.py bsgs 9990000000 10000000000 | tail -1 | grep -o "'window_ms.*"
  EIS_LIB=$lib LO=9875000000 HI=10000000000 timeout 120 python scripts/opt_sweep.py mode=2 alpha_x16=0
done
