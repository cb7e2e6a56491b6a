# co-residency of the window kernel (segment i+1) and the giant kernel (segment i)
# on the one-call window (9e9, 1e10]: window_ctas x giant_ctas, two passes
log=gpurun_out/overlap.log; : > $log
for pass in 1 2; do
  LO=9000000000 HI=10000000000 timeout 600 python scripts/opt_sweep.py window_ctas=0,3,2 giant_ctas=0,4,3,2 >> $log 2>&1
done
cat $log
