# fine alpha sweep (alpha_x16 22..40) of BSGS, and HALF, on (c - 1e8, c] windows
for c in 1200000000 1400000000 1600000000 1800000000 2000000000 3000000000 5000000000 7000000000 10000000000 20000000000 30000000000 50000000000 100000000000; do
  LO=$((c-100000000)) HI=$c timeout 300 python scripts/opt_sweep.py mode=1 | sed "s/^/$c /"
  LO=$((c-100000000)) HI=$c timeout 300 python scripts/opt_sweep.py mode=2 alpha_x16=0,22,24,26,28,30,32,34,36,38,40 | sed "s/^/$c /"
done
