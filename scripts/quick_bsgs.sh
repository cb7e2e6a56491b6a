# quick BSGS timing on the two metric windows
timeout 120 python scripts/opt_sweep.py mode=2 alpha_x16=24,28,32
LO=99900000000 HI=100000000000 timeout 120 python scripts/opt_sweep.py mode=2 alpha_x16=20,24,28
