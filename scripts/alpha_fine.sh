# fine alpha sweep (alpha_x16 22..40) of BSGS, and HALF, on (c - 1e8, c] windows
# (C: the window ends; default: around the HALF/BSGS crossover)
for c in ${C:-1100000000 1200000000 1300000000 1400000000 1500000000 1600000000}; do
  LO=$((c-100000000)) HI=$c timeout 300 python scripts/opt_sweep.py mode=1 | sed "s/^/$c /"
  LO=$((c-100000000)) HI=$c timeout 300 python scripts/opt_sweep.py mode=2 alpha_x16=0,22,24,26,28,30,32,34,36,38,40 | sed "s/^/$c /"
done
