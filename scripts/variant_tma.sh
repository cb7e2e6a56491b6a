for lib in build_variants/*.so build_variants/*.so; do
  echo "== $lib"
  EIS_LIB=$lib LO=9875000000 HI=10000000000 timeout 120 python scripts/opt_sweep.py mode=2 alpha_x16=0,0
done
EIS_LIB=build_variants/libeis_tma.so python -m pytest tests/test_gpu_parity.py -x -q -k "bsgs or auto or options or large" -p no:cacheprovider 2>&1 | tail -1
