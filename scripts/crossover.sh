for c in 1000000000 3000000000 10000000000 30000000000 100000000000; do
  LO=$((c-100000000)) HI=$c python scripts/opt_sweep.py mode=1,2 | sed "s/^/$c /"
done
