# HALF (mode 1) vs BSGS (mode 2, several alpha) on 1e8-wide windows below each scale
for c in 100000000 300000000 1000000000 3000000000 10000000000 30000000000 100000000000; do
  LO=$((c-100000000)) HI=$c timeout 300 python scripts/opt_sweep.py mode=1 | sed "s/^/$c /"
  LO=$((c-100000000)) HI=$c timeout 300 python scripts/opt_sweep.py mode=2 alpha_x16=16,24,32,40 | sed "s/^/$c /"
done
