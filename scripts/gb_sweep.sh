LO=9875000000 HI=10000000000 timeout 600 python scripts/opt_sweep.py mode=2 bsgs_gb=12,20,30,40
LO=9875000000 HI=10000000000 timeout 600 python scripts/opt_sweep.py mode=2 bsgs_gb=30 segment_log2=25,26
