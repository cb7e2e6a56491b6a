LO=900000000 HI=1000000000 timeout 300 python scripts/opt_sweep.py mode=1 blocks_per_sm=4,5,6,8
timeout 300 python scripts/opt_sweep.py mode=1 blocks_per_sm=4,5,6,8
