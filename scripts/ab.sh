for lib in build_variants/libeis_head.so build_variants/libeis_new.so build_variants/libeis_head.so build_variants/libeis_new.so; do
  echo "== $lib"; EIS_LIB=$lib LO=9875000000 HI=10000000000 timeout 300 python scripts/opt_sweep.py mode=2 bsgs_gb=32,32,32
done
nvidia-smi --query-gpu=name,memory.used,memory.total,clocks.sm,power.draw,temperature.gpu --format=csv
