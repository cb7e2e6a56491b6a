# Measured per-pipe peaks (bench_tools/pipe_peaks.cu) and which ncu pipe counter
# each op lands in; output gpurun_out/pipe_peaks.json, gpurun_out/pipe_map.csv
mkdir -p gpurun_out
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -diag-suppress 177 -o gpurun_out/pipe_peaks bench_tools/pipe_peaks.cu || exit 1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/pipe_clocks.csv &
SMI=$!
./gpurun_out/pipe_peaks > gpurun_out/pipe_peaks.json; echo "pipe_peaks exit $?"
kill $SMI
./gpurun_out/pipe_peaks > /dev/null && timeout 600 ncu --metrics smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_uniform.sum,sm__inst_executed_pipe_cbu.sum,sm__inst_executed_pipe_lsu.sum,sm__inst_executed_pipe_adu.sum --csv --log-file gpurun_out/pipe_map.csv --kernel-id :::1 ./gpurun_out/pipe_peaks > /dev/null; echo "ncu exit $?"
