timeout 600 python scripts/opt_sweep.py mode=2 window_ctas=0,3,4 giant_ctas=0,1,2,3
