# HALF vs BSGS (several alpha, and the default schedule) on (c - 1e8, c] windows
for c in 1000000000 1600000000 2000000000 3000000000 4000000000 5000000000 7000000000 10000000000 30000000000 100000000000; do
  LO=$((c-100000000)) HI=$c timeout 300 python scripts/opt_sweep.py mode=1 | sed "s/^/$c /"
  LO=$((c-100000000)) HI=$c timeout 300 python scripts/opt_sweep.py mode=2 alpha_x16=0,24,26,28,30,32,34,36,38 | sed "s/^/$c /"
done
