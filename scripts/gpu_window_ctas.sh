set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export LO=9875000000 HI=10000000000
for pass in 1 2; do
  timeout 300 python scripts/opt_sweep.py window_ctas=4,3,2,1 2>&1
done > gpurun_out/wctas.log
for c in 1 2 4; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv -k regex:bsgs_window --log-file gpurun_out/wc_$c.csv python scripts/opt_sweep.py window_ctas=$c > /dev/null 2>&1
done
cat gpurun_out/wctas.log
grep -h "bsgs_window" gpurun_out/wc_*.csv | awk -F'","' '{print FILENAME, $(NF-2), $NF}' 
for c in 1 2 4; do echo "== $c"; grep bsgs_window gpurun_out/wc_$c.csv | awk -F'","' '{print $(NF-2), $NF}'; done
