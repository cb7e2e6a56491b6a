for lib in build_variants/libeis_head.so build_variants/libeis_new.so build_variants/libeis_head.so build_variants/libeis_new.so; do
  echo "== $lib"
  EIS_LIB=$lib python scripts/prof_bsgs.py bsgs 9990000000 10000000000 | tail -1 | grep -o "'window_ms.*"
  EIS_LIB=$lib timeout 120 python scripts/opt_sweep.py mode=2 alpha_x16=28,36
done
EIS_LIB=build_variants/libeis_new.so timeout 120 python scripts/opt_sweep.py mode=2 sparse=0 alpha_x16=28
