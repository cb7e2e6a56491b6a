# the default alpha (alpha_x16 = 0) at the points of gpu_alpha_sweep.sh, two passes
log=gpurun_out/alpha_default.log; : > $log
for pass in 1 2; do
  for w in "1900000000 2000000000" "4900000000 5000000000" "9900000000 10000000000" "29900000000 30000000000" "99000000000 100000000000"; do
    set -- $w; LO=$1 HI=$2 timeout 300 python scripts/opt_sweep.py alpha_x16=0 >> $log 2>&1
  done
done
cat $log
