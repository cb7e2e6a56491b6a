# alpha_x16 around alpha_for()'s schedule at five d (two passes each): opt_sweep.py
# rates on 1e8-wide windows (1e9-wide at 1e11), into gpurun_out/alpha_sweep.log
log=gpurun_out/alpha_sweep.log; : > $log
run() { for pass in 1 2; do LO=$1 HI=$2 timeout 300 python scripts/opt_sweep.py alpha_x16=$3 >> $log 2>&1; done; }
run 1900000000 2000000000 30,33,36,39,42
run 4900000000 5000000000 28,30,32,34,36
run 9900000000 10000000000 26,28,30,32,34
run 29900000000 30000000000 24,26,28,30,32
run 99000000000 100000000000 22,24,26,28,30
cat $log
